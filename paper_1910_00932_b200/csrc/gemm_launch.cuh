// Host-side launch of the tcgen05 GEMM template (tc_gemm.cuh), shared by
// the translation units that instantiate it (gemm_inst_*.cu: the kernel
// instantiations are spread over several files so they compile in parallel)
// and by conv_ops.cu, which plans the convolutions.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <utility>

#include "common.cuh"
#include "tc_gemm.cuh"

namespace tsm {
namespace gemm_host {

// Programmatic dependent launch for the persistent tcgen05 kernels (see
// tc::pdl_wait): the next kernel's prologue overlaps this one's tail.  Off by
// default (TSM_PDL=1 enables): measured on one box, 2943-2950 clips/s with
// against 2961-2974 without — the side stream already fills the tails.
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("TSM_PDL");
    return e && atoi(e) != 0;
  }();
  return on;
}

template <class Kern, class... Args>
inline tsm_status launch_maybe_pdl(Kern kern, dim3 grid, dim3 block, int smem,
                                   cudaStream_t stream, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cuda_status(cudaLaunchKernelEx(&cfg, kern, args...), "cudaLaunchKernelEx");
}

using gemm::BK;
using gemm::BM;
using gemm::Params;

inline int num_sms() {
  constexpr int kMaxDev = 64;
  static std::atomic<int> n[kMaxDev] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDev) dev = 0;
  int v = n[dev].load(std::memory_order_relaxed);
  if (!v) {
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    if (v <= 0) v = 148;
    n[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

// Dynamic shared memory available to `kern` (`cap` minus its static smem),
// with the opt-in attribute set.  The attribute is per device, so the result
// is cached per (kernel, device): a second GPU in the same process sets it on
// its first launch too.
template <class Kern>
inline tsm_status dyn_smem_limit(Kern kern, int cap, int* limit) {
  // keyed by (kernel, device): every instantiation shares this function's
  // signature type, so the cache cannot be per template instance
  static std::map<std::pair<const void*, int>, int> cached;
  static std::mutex mu;
  int dev = 0;
  TSM_CUDA_TRY(cudaGetDevice(&dev));
  const auto key = std::make_pair(reinterpret_cast<const void*>(kern), dev);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cached.find(key);
  if (it == cached.end()) {
    cudaFuncAttributes fa{};
    TSM_CUDA_TRY(cudaFuncGetAttributes(&fa, kern));  // static smem counts against the cap
    const int l = cap - (int)fa.sharedSizeBytes;
    TSM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, l));
    it = cached.emplace(key, l).first;
  }
  *limit = it->second;
  return TSM_OK;
}

struct Maps {
  CUtensorMap a, b, out, res, mask;  // out/res/mask only for the TMA epilogue
};

inline bool out_slot_rule() {  // TSM_RES_SLOT1=0: two slots for the skip-gradient dgrad (A/B)
  static const bool on = [] {
    const char* e = getenv("TSM_RES_SLOT1");
    return !e || atoi(e) != 0;
  }();
  return on;
}

template <int BN, int KCA, int KCB, bool AMN, bool BMN, int CG = 1, int BKT = BK>
inline tsm_status launch_gemm(const Maps& m, Params p, cudaStream_t stream) {
  using C = gemm::Cfg<BN, KCA, KCB, AMN, BMN, CG, BKT>;
  auto kern = gemm::tc_gemm_kernel<BN, KCA, KCB, AMN, BMN, CG, BKT>;
  int limit = 0;  // dynamic shared memory available to this instantiation
  TSM_TRY(dyn_smem_limit(kern, gemm::kSmemLimit, &limit));
  const bool tma = p.epi == gemm::EPI_BF16 && p.tma_out;
  // K-heavy GEMMs are tensor-bound: one staging buffer per epilogue group
  // keeps their operand ring one stage deeper; short-K (epilogue-bound) ones
  // double-buffer the staging
  // one staging slot (a deeper operand ring) for K-heavy GEMMs and for the
  // skip-gradient dgrad (adjoint shift + identity-residual k-blocks): its
  // residual stream gains more from the extra stage than the epilogue loses
  // (res2-res5 dgrad conv1 + skip -25 us per step; conv3 + skip, whose
  // epilogue is busier, keeps two slots)
  p.out_slots = (p.k_blocks >= 8 || (p.res_kb && p.shift_out && out_slot_rule())) ? 1 : 2;
  {  // TSM_OUT_SLOTS=1|2 forces the epilogue staging depth (A/B experiments)
    static const int os = [] {
      const char* e = getenv("TSM_OUT_SLOTS");
      return e ? atoi(e) : 0;
    }();
    if (os == 1 || os == 2) p.out_slots = os;
  }
  const int epi = C::epi_bytes(p.residual != nullptr, p.mask != nullptr, tma, p.out_slots);
  const int extra = ((tma && p.bias) ? p.n_tiles * BN * 4 : 0)  // staged bias
                    + (p.res_kb ? gemm::kIdentBytes : 0);            // identity operand
  p.stages = C::stages_for_limit(limit, epi, extra);
  {  // TSM_MAX_STAGES=n caps the operand ring (A/B experiments)
    static const int cap = [] {
      const char* e = getenv("TSM_MAX_STAGES");
      return e ? atoi(e) : 0;
    }();
    if (cap > 0 && p.stages > cap) p.stages = cap;
  }
  if (p.stages < 1) return fail(TSM_ERR_UNSUPPORTED, "tc_gemm: no room for an operand stage");
  const int smem = C::smem_bytes(p.stages, epi, extra);
  if constexpr (CG == 1) {
    const int tiles = p.m_tiles * p.n_tiles * p.splits * (p.cls_n ? p.cls_n : 1);
    const int grid = std::max(1, std::min(tiles, num_sms()));
    TSM_TRY(launch_maybe_pdl(kern, dim3(grid), dim3(gemm::kThreads), smem, stream, m.a, m.b,
                             m.out, m.res, m.mask, p));
  } else {
    // CTA pairs: 2-CTA clusters, one pair per TPC, a persistent grid of
    // pairs over the (m pair, n, split) tiles
    if (p.res_kb || p.db_mode == 2 || (p.epi == gemm::EPI_BF16 && !tma))
      return fail(TSM_ERR_UNSUPPORTED, "tc_gemm pair: no fused residual / B-side bias grad");
    const int pair_tiles = (p.m_tiles + 1) / 2 * p.n_tiles * p.splits * (p.cls_n ? p.cls_n : 1);
    const int pairs = std::max(1, std::min(pair_tiles, num_sms() / 2));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(gemm::kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    TSM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, m.a, m.b, m.out, m.res, m.mask, p));
  }
  count_launches();
  return cuda_status(cudaGetLastError(), "tc_gemm_kernel launch");
}


constexpr int kWgradPairBK = 128;

// Per-group dispatchers (gemm_inst_*.cu).  fwd: K-major A (slab width kca)
// x K-major B; wgrad: MN-major A (dY, 64 channels) x MN-major B (X, kcb);
// swapped wgrad: MN-major A (X, kca) x MN-major B (dY).
tsm_status dispatch_fwd_kc64(int bn, const Maps& m, const Params& p, cudaStream_t s);
tsm_status dispatch_fwd_kc32(int bn, const Maps& m, const Params& p, cudaStream_t s);
tsm_status dispatch_fwd_kc16(int bn, const Maps& m, const Params& p, cudaStream_t s);
tsm_status dispatch_fwd_kc8(int bn, const Maps& m, const Params& p, cudaStream_t s);
tsm_status dispatch_fwd_pair(int bn, const Maps& m, const Params& p, cudaStream_t s);
tsm_status dispatch_wgrad_kc64(int bn, const Maps& m, const Params& p, cudaStream_t s);
tsm_status dispatch_wgrad_kc32(int bn, const Maps& m, const Params& p, cudaStream_t s);
tsm_status dispatch_wgrad_kc8(int bn, const Maps& m, const Params& p, cudaStream_t s);
tsm_status dispatch_wgrad_pair(const Maps& m, const Params& p, cudaStream_t s);
tsm_status dispatch_wgrad_swapped(int kca, const Maps& m, const Params& p, cudaStream_t s);
tsm_status dispatch_wgrad_bk128(int bn, int kcb, const Maps& m, const Params& p, cudaStream_t s);
tsm_status dispatch_wgrad_swapped_bk128(int kca, const Maps& m, const Params& p, cudaStream_t s);
bool wgrad_bk128_ok(bool swap, int bn, int kcx);

}  // namespace gemm_host
}  // namespace tsm
