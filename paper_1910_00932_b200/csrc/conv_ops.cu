// Host side of the tcgen05 conv engine: TMA tensor-map construction, tile
// planning and launches for every convolution of the TSM bottleneck and the
// TSM-R50 stem (NTHWC bf16 activations, fp32 accumulation).
//
// Mapping to the reference (kernels.cpp):
//   conv_fwd    <- conv_forward, frame-local path (kernels.cpp:171-200)
//   conv_dgrad  <- conv_backward, grad_x gather  (kernels.cpp:246-280)
//   conv_wgrad  <- conv_backward, grad_w          (kernels.cpp:282-310)
// The reference's fp64 fixed-order sums become bf16 x bf16 -> fp32 tensor-core
// sums; wgrad is split over K deterministically (fixed partition, ordered
// reduction) so results are bitwise reproducible run to run.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <string>

#include "aux_kernels.cuh"
#include "common.cuh"
#include "conv_ops.h"
#include "halo128.cuh"
#include "shift_conv.cuh"
#include "fused_block.cuh"
#include "halo_conv.cuh"
#include "head_kernels.cuh"
#include "gemm_launch.cuh"
#include "tc_gemm.cuh"

namespace tsm {
namespace {

using gemm::BK;
using gemm::BM;
using gemm::Params;
using gemm_host::dyn_smem_limit;
using gemm_host::Maps;
using gemm_host::num_sms;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
typedef CUresult (*EncodeIm2colFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const int*, const int*,
                                   cuuint32_t, cuuint32_t, const cuuint32_t*,
                                   CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct Driver {
  EncodeTiledFn tiled = nullptr;
  EncodeIm2colFn im2col = nullptr;
  int version = 0;
};

const Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      d.tiled = reinterpret_cast<EncodeTiledFn>(fn);
    fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      d.im2col = reinterpret_cast<EncodeIm2colFn>(fn);
    cudaDriverGetVersion(&d.version);
  });
  return d;
}

CUtensorMapSwizzle swizzle_of(int row_bytes) {
  switch (row_bytes) {
    case 128: return CU_TENSOR_MAP_SWIZZLE_128B;
    case 64: return CU_TENSOR_MAP_SWIZZLE_64B;
    case 32: return CU_TENSOR_MAP_SWIZZLE_32B;
    default: return CU_TENSOR_MAP_SWIZZLE_NONE;
  }
}

// L2 promotion of the TMA maps (A/B: TSM_L2_PROMO = 0 / 64 / 128 / 256 for
// every map; TSM_L2_PROMO_NARROW for maps whose box rows are narrower than
// 128 B).  256-byte promotion is the measured best for full-width rows; for
// the 16- / 32-channel shift slabs it pulls in the neighbouring channels of
// the neighbouring frame, which other tiles read much later (res2 conv1
// weight gradient 229 -> 207 us without promotion).
static CUtensorMapL2promotion promo_of(int bytes) {
  switch (bytes) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 64: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 128: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
}

static CUtensorMapL2promotion l2_promo(uint32_t row_bytes = 128) {
  static const int wide = [] {
    const char* e = getenv("TSM_L2_PROMO");
    return e ? atoi(e) : 256;
  }();
  static const int narrow = [] {
    const char* e = getenv("TSM_L2_PROMO_NARROW");
    return e ? atoi(e) : 0;
  }();
  return promo_of(row_bytes < 128 ? narrow : wide);
}

tsm_status encode_tiled(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                        const uint64_t* strides_bytes, const uint32_t* box,
                        bool no_swizzle = false) {
  const Driver& d = driver();
  if (!d.tiled) return fail(TSM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = d.tiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base),
                       dims, strides_bytes, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       no_swizzle ? CU_TENSOR_MAP_SWIZZLE_NONE : swizzle_of(box[0] * 2),
                       l2_promo(box[0] * 2),
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(TSM_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return TSM_OK;
}

// 3-D activation map: (C, rows_per_clip, clips), box {kc, rows, 1}.
tsm_status map_act3d(CUtensorMap* map, const void* base, int64_t c, int64_t rows_per_clip,
                     int64_t clips, int kc, int box_rows, int box_clips = 1) {
  uint64_t dims[3] = {(uint64_t)c, (uint64_t)rows_per_clip, (uint64_t)clips};
  uint64_t strides[2] = {(uint64_t)c * 2, (uint64_t)(rows_per_clip * c * 2)};
  uint32_t box[3] = {(uint32_t)kc, (uint32_t)box_rows, (uint32_t)box_clips};
  return encode_tiled(map, base, 3, dims, strides, box);
}

// 2-D matrix map: row-major [rows][k], box {kc, box_rows}.
tsm_status map_w2d(CUtensorMap* map, const void* base, int64_t k, int64_t rows, int kc,
                   int box_rows);

// The B (weights) map of a CTA-pair launch: each CTA loads half the N tile.
struct PairB {
  CUtensorMap map;
  bool ok = false;
  const CUtensorMap* get() const { return ok ? &map : nullptr; }
  tsm_status make(const void* w, int64_t k, int64_t rows, int bn) {
    if (bn != 256 && bn != 128) return TSM_OK;
    TSM_TRY(map_w2d(&map, w, k, rows, 64, bn / 2));
    ok = true;
    return TSM_OK;
  }
};

tsm_status map_w2d(CUtensorMap* map, const void* base, int64_t k, int64_t rows, int kc,
                   int box_rows) {
  uint64_t dims[2] = {(uint64_t)k, (uint64_t)rows};
  uint64_t strides[1] = {(uint64_t)k * 2};
  uint32_t box[2] = {(uint32_t)kc, (uint32_t)box_rows};
  return encode_tiled(map, base, 2, dims, strides, box);
}

// 4-D im2col map over NTHWC activations (C, W, H, frames) for a kxk conv
// with the given stride and padding; box = kc channels x `pixels` pixels.
// Window origins per axis (W, H) span [lo, dim-1 + hi].
tsm_status map_im2col_box(CUtensorMap* map, const void* base, int64_t c, int64_t w, int64_t h,
                          int64_t frames, int lo, int hi, int stride, int kc, int pixels) {
  const Driver& d = driver();
  if (!d.im2col) return fail(TSM_ERR_CUDA, "cuTensorMapEncodeIm2col unavailable");
  cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)frames};
  cuuint64_t strides[3] = {(cuuint64_t)c * 2, (cuuint64_t)(w * c * 2),
                           (cuuint64_t)(h * w * c * 2)};
  int lower[2] = {lo, lo};
  int upper[2] = {hi, hi};
  cuuint32_t es[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
  CUresult r = d.im2col(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims,
                        strides, lower, upper, (cuuint32_t)kc, (cuuint32_t)pixels, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_of(kc * 2),
                        l2_promo(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(TSM_ERR_CUDA, "cuTensorMapEncodeIm2col failed (" + std::to_string(r) + ")");
  // Same driver workaround CUTLASS applies to im2col maps of tensors under
  // 128 KiB on drivers <= 13.1 (cute/atom/copy_traits_sm90_im2col.hpp).
  if (d.version <= 13010 && frames * h * w * c * 2 < 131072)
    reinterpret_cast<uint64_t*>(map)[1] &= ~(1ull << 21);
  return TSM_OK;
}

// kxk conv with the given stride and symmetric padding: origins span
// [-pad, dim-1 + pad-(k-1)].
tsm_status map_im2col(CUtensorMap* map, const void* base, int64_t c, int64_t w, int64_t h,
                      int64_t frames, int ksize, int stride, int pad, int kc, int pixels) {
  return map_im2col_box(map, base, c, w, h, frames, -pad, pad - (ksize - 1), stride, kc, pixels);
}

// CTA pairs (cta_group::2, M = 256 per MMA) for the compute-bound K-major
// GEMMs: long K, a 256-wide N tile, the TMA epilogue without the fused
// residual.  Each CTA of the pair stages half the B tile, so the operand
// bytes per MMA flop halve and the smem ring gets deeper.  TSM_PAIR=0
// disables (A/B).
static bool pair_enabled() {
  static const bool on = [] {
    const char* e = getenv("TSM_PAIR");
    return !e || atoi(e) != 0;
  }();
  return on;
}

// (Measured, tools/bench_gemms.py: 5-12% faster on the long-K fused shift +
// conv1, 3x3 fwd/dgrad, conv3 dgrad and strided projection; slower on the
// epilogue-bound conv3 with its residual streamed in the epilogue, which
// stays single-CTA.)
static bool pair128_enabled() {  // TSM_PAIR128=0: 128-wide N tiles stay single-CTA (A/B)
  static const bool on = [] {
    const char* e = getenv("TSM_PAIR128");
    return !e || atoi(e) != 0;
  }();
  return on;
}

// 128-wide N tiles: pairs only on the long-K (3x3) GEMMs — fwd / dgrad
// conv2 at res3 127 -> 117 / 138 -> 129 us; the HBM-bound 8-k-block 1x1s
// (shift + conv1, conv3 dgrad) measured 12-15 % slower as pairs.
static bool use_pair(int bn, int kca, const Params& p) {
  return pair_enabled() &&
         (bn == 256 || (bn == 128 && pair128_enabled() && p.k_blocks >= 16)) && kca == 64 && p.k_blocks >= 8 && !p.res_kb &&
         !p.residual && p.tma_out && p.epi == gemm::EPI_BF16 && p.m_tiles >= 2;
}

gemm::OpLoad act_load(int rows_per_clip, int g0 = 0, int g1 = 0, int off0 = 0, int off1 = 0) {
  gemm::OpLoad l{};
  l.mode = gemm::LOAD_ACT3D;
  l.rows_per_clip = rows_per_clip;
  l.g0 = g0;
  l.g1 = g1;
  l.off0 = off0;
  l.off1 = off1;
  return l;
}

gemm::OpLoad w_load() {
  gemm::OpLoad l{};
  l.mode = gemm::LOAD_W2D;
  return l;
}

gemm::OpLoad im2col_load(int ho, int wo, int stride, int pad, int c_in, int k,
                         int rows_per_clip) {
  gemm::OpLoad l{};
  l.mode = gemm::LOAD_IM2COL;
  l.h_out = ho;
  l.w_out = wo;
  l.stride = stride;
  l.pad = pad;
  l.c_in = c_in;
  l.taps_w = k;
  l.rows_per_clip = rows_per_clip;
  return l;
}

// Largest slab width (channels) that keeps every shift-group boundary inside
// one slab: 64 (128B swizzle), 32 (64B), 8 (no swizzle).
int shift_kc(int64_t f) {
  if (f % 64 == 0) return 64;
  if (f % 32 == 0) return 32;
  if (f % 8 == 0) return 8;
  return 0;
}

int pick_bn(int64_t n) {
  if (n <= 64) return 64;
  if (n <= 128) return 128;
  return 256;
}

// K-major A (KC = kca) x K-major B (KC = 64): forward and dgrad.  `b_pair`
// is the B map with a half-height box for the pair kernel.
tsm_status dispatch_fwd(int bn, int kca, const Maps& m, const Params& p, cudaStream_t s,
                        const CUtensorMap* b_pair = nullptr) {
  if (b_pair && use_pair(bn, kca, p)) {
    Maps mp = m;
    mp.b = *b_pair;
    return gemm_host::dispatch_fwd_pair(bn, mp, p, s);
  }
  switch (kca) {
    case 64: return gemm_host::dispatch_fwd_kc64(bn, m, p, s);
    case 32: return gemm_host::dispatch_fwd_kc32(bn, m, p, s);
    case 16: return gemm_host::dispatch_fwd_kc16(bn, m, p, s);
    case 8: return gemm_host::dispatch_fwd_kc8(bn, m, p, s);
  }
  return fail(TSM_ERR_UNSUPPORTED, "no forward GEMM for KC=" + std::to_string(kca));
}

using gemm_host::kWgradPairBK;

// MN-major A (KC = 64) x MN-major B (KC = kcb): wgrad.  Long pixel ranges
// with 256-wide N tiles and a dY (A-side) bias gradient run as CTA pairs
// with 128 pixel rows per stage (Cfg's BKT; conv_wgrad builds the maps and
// k-block counts to match).
static bool use_pair_wgrad(int bn, int kcb, const ConvShape& s, int64_t m_tiles) {
  return pair_enabled() && bn == 256 && kcb == 64 && m_tiles >= 2 &&
         s.clips * s.T * s.h_out() * s.w_out() >= 16 * kWgradPairBK;
}

tsm_status dispatch_wgrad(int bn, int kcb, const Maps& m, const Params& p, cudaStream_t s,
                          bool pair) {
  if (pair) return gemm_host::dispatch_wgrad_pair(m, p, s);
  switch (kcb) {
    case 64: return gemm_host::dispatch_wgrad_kc64(bn, m, p, s);
    case 32: return gemm_host::dispatch_wgrad_kc32(bn, m, p, s);
    case 8: return gemm_host::dispatch_wgrad_kc8(bn, m, p, s);
  }
  return fail(TSM_ERR_UNSUPPORTED, "no wgrad GEMM for KC=" + std::to_string(kcb));
}

using gemm_host::dispatch_wgrad_swapped;

Params base_params() {
  Params p{};
  p.splits = 1;
  p.epi = gemm::EPI_BF16;
  return p;
}

// Switch a bf16 epilogue to the TMA path when its geometry allows: 32-column
// sub-tiles, no row scatter, shift groups aligned to sub-tiles.  Builds the
// out / residual / mask maps: 3-D (C, rows_per_clip, clips) for MAP_CLIP
// tiles (needed for the adjoint-shift row offsets), 2-D (C, rows) otherwise.
tsm_status setup_epilogue(Params& p, Maps& m, int64_t clips) {
  if (p.epi != gemm::EPI_BF16 || p.n_total % gemm::EC || p.ldo % gemm::EC) return TSM_OK;
  if (p.scatter) {
    // staged sub-tiles stored by the epilogue threads (no output map)
    if (!p.residual && !p.mask && !p.shift_out) p.tma_out = 1;
    return TSM_OK;
  }
  if (p.shift_out && (p.sg0 % gemm::EC || p.sg1 % gemm::EC || p.map_mode != gemm::MAP_CLIP))
    return TSM_OK;
  auto make = [&](CUtensorMap* map, const void* base) -> tsm_status {
    if (p.map_mode == gemm::MAP_CLIP)
      return map_act3d(map, base, p.ldo, p.rows_per_clip, clips, gemm::EC, BM);
    return map_w2d(map, base, p.ldo, p.m_total, gemm::EC, BM);
  };
  TSM_TRY(make(&m.out, p.out));
  if (p.residual) TSM_TRY(make(&m.res, p.residual));
  if (p.mask) TSM_TRY(make(&m.mask, p.mask));
  p.tma_out = 1;
  return TSM_OK;
}

// ---------------------------------------------------------------------------
// Halo-tile 3x3 path (halo_conv.cuh): 64 -> 64 channels, stride 1, no shift.
bool halo_ok(const ConvShape& s) {
  return s.k == 3 && s.stride == 1 && s.c_in == 64 && s.c_out == 64 && !s.F && !s.B;
}

// 4-D NTHWC map (C, W, H, frames), box {bc, bw, bh, 1}.
tsm_status map_act4d(CUtensorMap* map, const void* base, int64_t c, int64_t w, int64_t h,
                     int64_t frames, int bc, int bw, int bh) {
  uint64_t dims[4] = {(uint64_t)c, (uint64_t)w, (uint64_t)h, (uint64_t)frames};
  uint64_t strides[3] = {(uint64_t)c * 2, (uint64_t)(w * c * 2), (uint64_t)(h * w * c * 2)};
  uint32_t box[4] = {(uint32_t)bc, (uint32_t)bw, (uint32_t)bh, 1};
  return encode_tiled(map, base, 4, dims, strides, box);
}


// A persistent grid of 2-CTA clusters (CTA pairs) of the halo kernels.
template <class Kern, class... Args>
static tsm_status launch_pair(Kern kern, int pairs, int smem, cudaStream_t stream,
                              Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(halo::kThreads);
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
  cfg.numAttrs = gemm_host::pdl_enabled() ? 2 : 1;
  return cuda_status(cudaLaunchKernelEx(&cfg, kern, args...), "cudaLaunchKernelEx (pair)");
}

// 3x3 / stride 1, 128 -> 128 channels (res3 conv2 and its input gradient)
// on the halo-tile kernel with streamed weights (halo128.cuh).
// TSM_HALO128: 2 = CTA pairs (default), 1 = single CTAs, 0 = the im2col GEMM.
static int halo128_mode() {
  static const int mode = [] {
    const char* e = getenv("TSM_HALO128");
    return e ? atoi(e) : 2;
  }();
  return mode;
}

static bool halo128_ok(const ConvShape& s) {
  return halo128_mode() > 0 && s.k == 3 && s.stride == 1 && s.c_in == 128 && s.c_out == 128 &&
         !s.F && !s.B;
}

static tsm_status halo128_conv(const ConvShape& s, const void* x, const void* w,
                               const float* bias, void* y, int relu, cudaStream_t stream,
                               uint32_t* bits_out, const uint32_t* mask_bits) {
  using namespace halo;
  const int64_t frames = s.clips * s.T;
  const int cg = halo128_mode() == 1 ? 1 : 2;
  auto kern = cg == 2 ? halo128_kernel<2> : halo128_kernel<1>;
  int limit = 0;
  TSM_TRY(dyn_smem_limit(kern, halo::kSmemLimit, &limit));
  CUtensorMap mx, mw, mo;
  TSM_TRY(map_act4d(&mx, x, 128, s.W, s.H, frames, 64, kH128HP, kH128HR));
  TSM_TRY(map_w2d(&mw, w, 9 * 128, 128, 64, 128 / cg));
  TSM_TRY(map_act4d(&mo, y, 128, s.W, s.H, frames, 32, kTW, kTH));
  Halo128Params p{};
  p.tiles_y = (int)((s.H + kTH - 1) / kTH);
  p.tiles_x = (int)((s.W + kTW - 1) / kTW);
  p.total = (int)(frames * p.tiles_y * p.tiles_x);
  p.bias = bias;
  p.relu = relu;
  p.H = (int)s.H;
  p.W = (int)s.W;
  p.bits_out = bits_out;
  p.mask_bits = mask_bits;
  const int fixed = 1024 + 2 * kH128HaloStride + 4 * kSub;
  const int bbytes = kH128BBytes / cg;
  p.bstages = std::min(kH128MaxBs, (limit - fixed) / bbytes);
  if (p.bstages < 2) return fail(TSM_ERR_UNSUPPORTED, "halo128: shared memory");
  const int smem = fixed + p.bstages * bbytes;
  if (cg == 1) {
    const int grid = std::max(1, std::min(p.total, num_sms()));
    TSM_TRY(gemm_host::launch_maybe_pdl(kern, dim3(grid), dim3(kThreads), smem, stream, mx, mw,
                                        mo, p));
  } else {
    const int pairs = std::max(1, std::min((p.total + 1) / 2, num_sms() / 2));
    TSM_TRY(launch_pair(kern, pairs, smem, stream, mx, mw, mo, p));
  }
  count_launches();
  return cuda_status(cudaGetLastError(), "halo128_kernel launch");
}

// Fused shift + 1x1 conv, 64 -> 64 channels, shift groups F, B multiples of
// 8 with F + B <= 16 (res2.0 conv1) on the three-frame tile kernel
// (shift_conv.cuh).  TSM_SHIFT1=0: the generic GEMM with 8-channel slabs.
static bool shift1_ok(const ConvShape& s) {
  static const bool on = [] {
    const char* e = getenv("TSM_SHIFT1");
    return !e || atoi(e) != 0;
  }();
  return on && s.k == 1 && s.stride == 1 && s.c_in == 64 && s.c_out == 64 && (s.F || s.B) &&
         s.F % 8 == 0 && s.B % 8 == 0 && s.F + s.B <= 16;
}

// forward (dg = 0): y = act(conv1x1(shift(x), w) + bias), bits_out;
// input gradient (dg = 1): dx = mask_bits * (adjshift(conv1x1(dy, wt)) + skip)
static tsm_status shift1x1_conv(const ConvShape& s, const void* x, const void* w,
                                const float* bias, const void* skip, void* y, int relu,
                                cudaStream_t stream, uint32_t* bits_out,
                                const uint32_t* mask_bits, bool dg) {
  using namespace halo;
  const int64_t frames = s.clips * s.T;
  auto kern = dg ? shift1x1_kernel<true> : shift1x1_kernel<false>;
  int limit = 0;
  TSM_TRY(dyn_smem_limit(kern, halo::kSmemLimit, &limit));
  CUtensorMap mx, mw, mo, mr;
  {
    const uint64_t c2 = 64 * 2;
    uint64_t dims[5] = {64, (uint64_t)s.W, (uint64_t)s.H, (uint64_t)s.T, (uint64_t)s.clips};
    uint64_t strides[4] = {c2, (uint64_t)s.W * c2, (uint64_t)(s.H * s.W) * c2,
                           (uint64_t)(s.T * s.H * s.W) * c2};
    uint32_t box[5] = {64, (uint32_t)kTW, (uint32_t)kTH, 1, 1};
    TSM_TRY(encode_tiled(&mx, x, 5, dims, strides, box));
  }
  TSM_TRY(map_w2d(&mw, w, 64, 64, 64, 64));
  TSM_TRY(map_act4d(&mo, y, 64, s.W, s.H, frames, 32, kTW, kTH));
  if (skip) TSM_TRY(map_act4d(&mr, skip, 64, s.W, s.H, frames, 32, kTW, kTH));
  else mr = mo;
  Shift1Params p{};
  p.tiles_y = (int)((s.H + kTH - 1) / kTH);
  p.tiles_x = (int)((s.W + kTW - 1) / kTW);
  p.total = (int)(frames * p.tiles_y * p.tiles_x);
  p.T = (int)s.T;
  p.F = (int)s.F;
  p.B = (int)s.B;
  p.bias = bias;
  p.relu = relu;
  p.H = (int)s.H;
  p.W = (int)s.W;
  p.bits_out = bits_out;
  p.mask_bits = mask_bits;
  p.has_res = skip != nullptr;
  // weights (+ variants) and 2 groups x (2 staging (+ 2 skip)) sub-tiles
  const int fixed = 1024 + (dg ? 4 : 2) * 64 * kRowB + (dg ? 8 : 4) * kSub;
  p.stages = std::min(kMaxStages, (limit - fixed) / kS1Stage);
  if (p.stages < 2) return fail(TSM_ERR_UNSUPPORTED, "shift1x1: shared memory");
  const int smem = fixed + p.stages * kS1Stage;
  const int grid = std::max(1, std::min(p.total, num_sms()));
  TSM_TRY(gemm_host::launch_maybe_pdl(kern, dim3(grid), dim3(kThreads), smem, stream, mx, mw, mo,
                                      mr, p));
  count_launches();
  return cuda_status(cudaGetLastError(), "shift1x1_kernel launch");
}

static int shift1_wgrad_ctas(const ConvShape& s) {
  const int64_t patches = s.clips * s.T * ((s.H + halo::kPW - 1) / halo::kPW) *
                          ((s.W + halo::kPW - 1) / halo::kPW);
  return (int)std::max<int64_t>(1, std::min<int64_t>(patches, num_sms()));
}

static size_t shift1_wgrad_workspace_bytes(const ConvShape& s) {
  return (size_t)shift1_wgrad_ctas(s) * 256 * 64 * 4;
}

// dw [64][64] fp32 (and db [64]) of the narrow-split shifted 1x1 conv:
// per-CTA partials of wgrad_shift1_kernel + ordered reduction.
static tsm_status shift1_wgrad(const ConvShape& s, const void* x, const void* dy, float* dw,
                               float* db, float* ws, cudaStream_t stream) {
  using namespace halo;
  const int grid = shift1_wgrad_ctas(s);
  int limit = 0;
  TSM_TRY(dyn_smem_limit(wgrad_shift1_kernel, halo::kSmemLimit, &limit));
  CUtensorMap mx, mdy;
  const uint64_t c2 = 64 * 2;
  uint64_t dims[5] = {64, (uint64_t)s.W, (uint64_t)s.H, (uint64_t)s.T, (uint64_t)s.clips};
  uint64_t strides[4] = {c2, (uint64_t)s.W * c2, (uint64_t)(s.H * s.W) * c2,
                         (uint64_t)(s.T * s.H * s.W) * c2};
  uint32_t box[5] = {64, (uint32_t)kPW, (uint32_t)kPW, 1, 1};
  TSM_TRY(encode_tiled(&mx, x, 5, dims, strides, box));
  TSM_TRY(encode_tiled(&mdy, dy, 5, dims, strides, box));
  Shift1WgradParams p{};
  p.patches_y = (int)((s.H + kPW - 1) / kPW);
  p.patches_x = (int)((s.W + kPW - 1) / kPW);
  p.total = (int)(s.clips * s.T * p.patches_y * p.patches_x);
  p.T = (int)s.T;
  p.ws = ws;
  const int fixed = 1024 + kS1Patch;  // + the all-ones tile
  p.stages = std::min(kMaxStages, (limit - fixed) / kS1WStage);
  const int smem = fixed + p.stages * kS1WStage;
  TSM_TRY(gemm_host::launch_maybe_pdl(wgrad_shift1_kernel, dim3(grid), dim3(kThreads), smem,
                                      stream, mx, mdy, p));
  count_launches();
  TSM_CUDA_TRY(cudaGetLastError());
  wgrad_shift1_reduce_kernel<<<(64 * 64 + 64) / 32, 256, 0, stream>>>(
      ws, dw, db, grid, (int)s.F, (int)s.B);
  count_launches();
  return cuda_status(cudaGetLastError(), "wgrad_shift1_reduce_kernel launch");
}

// Weight gradient of the 3x3 / 128-channel conv on the halo window kernel
// (wgrad_halo128_kernel; res3 conv2 151 -> 139 us in the step;
// TSM_HALO128_WGRAD=0: the im2col pair GEMM, A/B).
static bool halo128_wgrad_ok(const ConvShape& s) {
  static const bool on = [] {
    const char* e = getenv("TSM_HALO128_WGRAD");
    return !e || atoi(e) != 0;
  }();
  return on && s.k == 3 && s.stride == 1 && s.c_in == 128 && s.c_out == 128 && !s.F && !s.B;
}

static int halo128_wgrad_gctas() { return std::max(1, num_sms() / 3); }

static size_t halo128_wgrad_workspace_bytes() {
  return (size_t)3 * halo128_wgrad_gctas() * halo::kW128Rows * 128 * 4;
}

static tsm_status halo128_wgrad(const ConvShape& s, const void* x, const void* dy, float* dw,
                                float* db, float* ws, cudaStream_t stream) {
  using namespace halo;
  const int gctas = halo128_wgrad_gctas();
  int limit = 0;
  TSM_TRY(dyn_smem_limit(wgrad_halo128_kernel, halo::kSmemLimit, &limit));
  const int64_t frames = s.clips * s.T;
  CUtensorMap mx, mdy;
  TSM_TRY(map_act4d(&mx, x, 128, s.W, s.H, frames, 64, kW128P, kPW));
  TSM_TRY(map_act4d(&mdy, dy, 128, s.W, s.H, frames, 64, kPW, kPW));
  Wgrad128Params p{};
  p.patches_y = (int)((s.H + kPW - 1) / kPW);
  p.patches_x = (int)((s.W + kPW - 1) / kPW);
  p.total = (int)(frames * p.patches_y * p.patches_x);
  p.gctas = gctas;
  p.ws = ws;
  const int fixed = 1024 + 2 * kDyBytes;  // + the all-ones tile (two atoms)
  p.stages = std::min(kMaxStages, (limit - fixed) / kW128Stage);
  const int smem = fixed + p.stages * kW128Stage;
  TSM_TRY(gemm_host::launch_maybe_pdl(wgrad_halo128_kernel, dim3(3 * gctas), dim3(kThreads),
                                      smem, stream, mx, mdy, p));
  count_launches();
  TSM_CUDA_TRY(cudaGetLastError());
  const int n = 9 * 128 * 128 + 128;
  wgrad_halo128_reduce_kernel<<<(n + 255) / 256, 256, 0, stream>>>(ws, dw, db, gctas);
  count_launches();
  return cuda_status(cudaGetLastError(), "wgrad_halo128_reduce_kernel launch");
}

// y = act(conv_KHxKH(x, w) + bias) [* mask]; w K-major [64][KH*KH][C]; x
// [frames][H][W][C], window offsets -KH/2 .. KH-1-KH/2, 64 output channels.
template <int KH, int C>
tsm_status halo_conv_t(const void* x, const void* w, const float* bias, const void* mask,
                       void* y, int relu, int64_t frames, int64_t H, int64_t W,
                       cudaStream_t stream, uint32_t* bits_out, const uint32_t* mask_bits) {
  using namespace halo;
  using HC = HaloCfg<KH, C>;
  int limit = 0;
  TSM_TRY(dyn_smem_limit(halo_conv_kernel<KH, C>, halo::kSmemLimit, &limit));
  CUtensorMap mx, mw, mo, mm;
  TSM_TRY(map_act4d(&mx, x, C, W, H, frames, C, HC::HP, HC::HR));
  TSM_TRY(map_w2d(&mw, w, KH * KH * C, 64, C, 64));
  TSM_TRY(map_act4d(&mo, y, 64, W, H, frames, 32, kTW, kTH));
  if (mask) TSM_TRY(map_act4d(&mm, mask, 64, W, H, frames, 32, kTW, kTH));
  else mm = mo;
  FwdParams p{};
  p.tiles_y = (int)((H + kTH - 1) / kTH);
  p.tiles_x = (int)((W + kTW - 1) / kTW);
  p.total = (int)(frames * p.tiles_y * p.tiles_x);
  p.bias = bias;
  p.relu = relu;
  p.has_mask = mask != nullptr;
  p.H = (int)H;
  p.W = (int)W;
  p.bits_out = bits_out;
  p.mask_bits = mask_bits;
  const int fixed = 1024 + HC::WBYTES + 6 * kSub;  // 2 groups x (2 out + 1 mask) sub-tiles
  p.stages = std::min(kMaxStages, (limit - fixed) / HC::STRIDE);
  const int smem = fixed + p.stages * HC::STRIDE;
  const int grid = std::max(1, std::min(p.total, num_sms()));
  TSM_TRY(gemm_host::launch_maybe_pdl(halo_conv_kernel<KH, C>, dim3(grid), dim3(kThreads), smem,
                                      stream, mx, mw, mo, mm, p));
  count_launches();
  return cuda_status(cudaGetLastError(), "halo_conv_kernel launch");
}

tsm_status halo_conv(const ConvShape& s, const void* x, const void* w, const float* bias,
                     const void* mask, void* y, int relu, cudaStream_t stream,
                     uint32_t* bits_out = nullptr, const uint32_t* mask_bits = nullptr) {
  return halo_conv_t<3, 64>(x, w, bias, mask, y, relu, s.clips * s.T, s.H, s.W, stream,
                            bits_out, mask_bits);
}

int halo_wgrad_ctas(const ConvShape& s) {
  const int64_t patches = s.clips * s.T * ((s.H + halo::kPW - 1) / halo::kPW) *
                          ((s.W + halo::kPW - 1) / halo::kPW);
  return (int)std::max<int64_t>(1, std::min<int64_t>(patches, num_sms()));
}

size_t halo_wgrad_workspace_bytes(const ConvShape& s) {
  return (size_t)halo_wgrad_ctas(s) * (576 * 64 + 64) * 4;
}

// Launch wgrad_halo_kernel<KH, KW> over x [frames][H][W][64] and dy
// [frames][H][W][64]: per-CTA partials ws[grid][KH*KW*64][64] (+ db_ws).
template <int KH, int KW>
tsm_status halo_wgrad_launch(const void* x, const void* dy, float* ws, float* db_ws,
                             int64_t frames, int64_t H, int64_t W, int grid, cudaStream_t stream) {
  using namespace halo;
  using WC = WgradCfg<KH, KW>;
  int limit = 0;
  TSM_TRY(dyn_smem_limit(wgrad_halo_kernel<KH, KW>, halo::kSmemLimit, &limit));
  CUtensorMap mx, mdy;
  TSM_TRY(map_act4d(&mx, x, 64, W, H, frames, 64, WC::P, WC::R));
  TSM_TRY(map_act4d(&mdy, dy, 64, W, H, frames, 64, kPW, kPW));
  WgradParams p{};
  p.patches_y = (int)((H + kPW - 1) / kPW);
  p.patches_x = (int)((W + kPW - 1) / kPW);
  p.total = (int)(frames * p.patches_y * p.patches_x);
  p.ws = ws;
  p.db_ws = db_ws;
  const int fixed = 1024 + (WC::ONES ? kOnesBytes : 0);
  p.stages = std::min(kMaxStages, (limit - fixed) / WC::STAGE);
  const int smem = fixed + p.stages * WC::STAGE;
  TSM_TRY(gemm_host::launch_maybe_pdl(wgrad_halo_kernel<KH, KW>, dim3(grid), dim3(kThreads), smem,
                                      stream, mx, mdy, p));
  count_launches();
  return cuda_status(cudaGetLastError(), "wgrad_halo_kernel launch");
}

// dw [64][9][64] fp32 (and db [64]) via per-CTA partials + ordered reduction.
tsm_status halo_wgrad(const ConvShape& s, const void* x, const void* dy, float* dw, float* db,
                      float* ws, cudaStream_t stream) {
  const int grid = halo_wgrad_ctas(s);
  float* db_ws = db ? ws + (size_t)grid * 576 * 64 : nullptr;
  TSM_TRY((halo_wgrad_launch<3, 3>(x, dy, ws, db_ws, s.clips * s.T, s.H, s.W, grid, stream)));
  TSM_TRY(splitk_reduce_transpose(ws, dw, grid, 576, 64, stream));
  return db ? splitk_reduce(db_ws, db, grid, 64, stream) : TSM_OK;
}

}  // namespace

// ---------------------------------------------------------------------------
// Forward:  y = act( conv_kxk(shift(x)) + bias (+ residual) ).
// Largest main-loop length (k-blocks) whose residual goes through the MMA
// (TSM_FUSE_RES=0 disables, TSM_FUSE_RES=n sets the limit; default 4).
static int fuse_res_kb() {
  static const int kb = [] {
    const char* e = getenv("TSM_FUSE_RES");
    return e ? atoi(e) : 4;
  }();
  return kb;
}

static bool rem_gather_enabled() {
  static const bool on = [] {
    const char* e = getenv("TSM_REM_GATHER");
    return !e || atoi(e) != 0;
  }();
  return on;
}

tsm_status conv_fwd(const ConvShape& s, const void* x, const void* w, const float* bias,
                    const void* residual, void* y, int relu, cudaStream_t stream,
                    uint32_t* bits_out) {
  const int64_t frames = s.clips * s.T;
  const int64_t ho = s.h_out(), wo = s.w_out();
  const int kk = s.k * s.k;
  if (s.c_out % 16 != 0) return fail(TSM_ERR_UNSUPPORTED, "conv: c_out must be a multiple of 16");
  if ((s.F || s.B) && (s.k != 1 || s.stride != 1))
    return fail(TSM_ERR_INVALID, "conv: the temporal shift only precedes a 1x1 stride-1 conv");
  if (bits_out && s.c_out % 32) return fail(TSM_ERR_UNSUPPORTED, "conv: bitmask needs c_out % 32");
  if (halo_ok(s) && !residual)
    return halo_conv(s, x, w, bias, nullptr, y, relu, stream, bits_out, nullptr);
  if (halo128_ok(s) && !residual)
    return halo128_conv(s, x, w, bias, y, relu, stream, bits_out, nullptr);
  if (shift1_ok(s) && !residual)
    return shift1x1_conv(s, x, w, bias, nullptr, y, relu, stream, bits_out, nullptr, false);
  const int bn = pick_bn(s.c_out);
  Maps mp{};
  CUtensorMap &ma = mp.a, &mb = mp.b;
  Params p = base_params();
  PairB pb;
  p.n_tiles = (int)((s.c_out + bn - 1) / bn);
  p.n_total = (int)s.c_out;
  p.bias = bias;
  p.residual = static_cast<const __nv_bfloat16*>(residual);
  p.out = static_cast<__nv_bfloat16*>(y);
  p.ldo = (int)s.c_out;
  p.relu = relu;
  int kca;
  if (s.k == 1 && s.stride == 1) {
    if (s.c_in % 64 != 0) return fail(TSM_ERR_UNSUPPORTED, "conv1x1: c_in % 64 != 0");
    if (s.F < 0 || s.B < 0 || s.F + s.B > s.c_in)
      return fail(TSM_ERR_INVALID, "conv1x1: bad shift split");
    kca = std::min(shift_kc(s.F), shift_kc(s.F + s.B));
    if (!kca) return fail(TSM_ERR_UNSUPPORTED, "conv1x1: shift split must be a multiple of 8");
    const int64_t rows = s.T * s.H * s.W;
    TSM_TRY(map_act3d(&ma, x, s.c_in, rows, s.clips, kca, BM));
    TSM_TRY(map_w2d(&mb, w, s.c_in, s.c_out, 64, bn));
    TSM_TRY(pb.make(w, s.c_in, s.c_out, bn));
    p.tiles_per_clip = (int)((rows + BM - 1) / BM);
    p.m_tiles = (int)(s.clips * p.tiles_per_clip);
    p.k_blocks = (int)(s.c_in / BK);
    p.map_mode = gemm::MAP_CLIP;
    p.rows_per_clip = (int)rows;
    p.a = act_load((int)rows, (int)s.F, (int)(s.F + s.B), (int)(-s.H * s.W), (int)(s.H * s.W));
  } else {
    // im2col path (3x3, strided 1x1, 7x7 stem); K = k*k*c_in, zero-padded
    // to a multiple of 64 in the weights when c_in < 64.
    kca = s.c_in >= 64 ? 64 : (int)s.c_in;
    if (s.c_in % kca != 0 || (kca != 64 && kca != 32 && kca != 8))
      return fail(TSM_ERR_UNSUPPORTED, "conv: c_in must be 8, 32 or a multiple of 64");
    const int64_t k_real = kk * s.c_in, k_pad = (k_real + BK - 1) / BK * BK;
    TSM_TRY(map_im2col(&ma, x, s.c_in, s.W, s.H, frames, s.k, s.stride, s.k / 2, kca, BM));
    TSM_TRY(map_w2d(&mb, w, k_pad, s.c_out, 64, bn));
    TSM_TRY(pb.make(w, k_pad, s.c_out, bn));
    p.m_total = (int)(frames * ho * wo);
    p.m_tiles = (p.m_total + BM - 1) / BM;
    p.k_blocks = (int)(k_pad / BK);
    p.map_mode = gemm::MAP_LINEAR;
    p.a = im2col_load((int)ho, (int)wo, s.stride, s.k / 2, (int)s.c_in, s.k, 0);
  }
  p.b = w_load();
  TSM_TRY(setup_epilogue(p, mp, s.clips));
  // Residual through the MMA (unshifted 1x1 convs, i.e. conv3 + skip): the
  // residual's 64-channel slabs become extra k-blocks against an identity
  // operand, so the epilogue has no residual stream to wait on (the
  // epilogue-bound part of these memory-bound GEMMs).
  // (short K only: with 8+ k-blocks the GEMM is tensor-bound and the N = 64
  // identity MMAs cost more than the epilogue stream they replace)
  if (residual && p.tma_out && s.k == 1 && s.stride == 1 && !s.F && !s.B && kca == 64 &&
      bn % 64 == 0 && s.c_out % bn == 0 && p.k_blocks <= fuse_res_kb()) {
    const int64_t rows = s.T * s.H * s.W;
    TSM_TRY(map_act3d(&mp.res, residual, s.c_out, rows, s.clips, 64, BM));
    p.r = act_load((int)rows);
    p.res_kb = bn / 64;
    p.residual = nullptr;
  }
  if (bits_out) {
    if (!p.tma_out) return fail(TSM_ERR_UNSUPPORTED, "conv: bitmask output needs the TMA epilogue");
    p.bits_out = bits_out;
    p.bits_ld = (int)(s.c_out / 32);
  }
  // Clip remainders gathered (fused shift): when a clip's rows leave a
  // short last tile (res5: 392 = 3 x 128 + 8, res4: 1568 = 12 x 128 + 32),
  // the remainder rows of BM / rem clips share one tile through a
  // {KC, rem, BM / rem} box of the same 3-D map (each clip's rows keep their
  // own frame offsets and out-of-clip zero fill): 196 M tiles instead of 256
  // at res5.  The output uses the same box shape.  TSM_REM_GATHER=0: off.
  if (p.map_mode == gemm::MAP_CLIP && (s.F || s.B) && s.k == 1 && p.tma_out && !p.residual &&
      !p.res_kb && rem_gather_enabled()) {
    const int64_t rows = s.T * s.H * s.W, rem = rows % BM;
    if (rem && BM % rem == 0 && rem <= 32) {
      const int rc = (int)(BM / rem);
      p.tiles_per_clip = (int)(rows / BM);
      p.rem_tiles0 = (int)(s.clips * p.tiles_per_clip);
      p.rem_rows = (int)rem;
      p.rem_clips = rc;
      p.n_clips = (int)s.clips;
      p.m_tiles = p.rem_tiles0 + (int)((s.clips + rc - 1) / rc);
      TSM_TRY(map_act3d(&mp.res, x, s.c_in, rows, s.clips, kca, (int)rem, rc));
      TSM_TRY(map_act3d(&mp.mask, y, s.c_out, rows, s.clips, gemm::EC, (int)rem, rc));
    }
  }
  return dispatch_fwd(bn, kca, mp, p, stream, pb.get());
}

// ---------------------------------------------------------------------------
// Narrow shift splits in virtual channels (F + B <= 32, e.g. res2.0's 8 + 8
// of 64 channels): instead of 8-channel slabs (16-byte TMA rows), the
// shifted x operand of the weight gradient becomes 64 + c_in virtual
// channels — 32 channels at frame t-1, 32 at t+1, all c_in at t, each a
// 64-byte-row slab read through TMA row offsets — and the reduction keeps
// only each channel's live copy.  (The same expansion for the forward, with
// zero-masked weights, measured slower than the 8-channel slabs: 126.6 vs
// 118.1 µs at res2.0, profiles/r02/README.md.)
bool vshift_ok(const ConvShape& s) {
  return s.k == 1 && s.stride == 1 && (s.F || s.B) && s.F % 8 == 0 && s.B % 8 == 0 &&
         s.F + s.B <= kVShift && (s.F % 32 || s.B % 32) && s.c_in % 64 == 0;
}

// ---------------------------------------------------------------------------
// Input gradient.  `wt` is the dgrad weight: for 1x1 W^T [c_in][c_out]; for
// kxk the tap-flipped transpose [c_in][k][k][c_out] (weights_for_dgrad).
// out = mask? * ( adjshift(dgrad(dy)) + residual ).  For stride 2:
//   1x1: rows scattered to (2ho, 2wo), dx pre-zeroed here;
//   3x3: dy is zero-inserted into `scratch` (frames*H*W*c_out bf16) first.
static bool subpix_merged() {
  static const bool on = [] {
    const char* e = getenv("TSM_SUBPIX_MERGED");
    return !e || atoi(e) != 0;
  }();
  return on;
}

// TSM_SUBPIX_TMA=0: the merged sub-pixel dgrad stores its scattered rows per
// thread instead of through row-aligned tiles and the 5-D class map (A/B).
static bool subpix_tma_enabled() {
  static const bool on = [] {
    const char* e = getenv("TSM_SUBPIX_TMA");
    return !e || atoi(e) != 0;
  }();
  return on;
}

tsm_status conv_dgrad(const ConvShape& s, const void* dy, const void* wt, const void* residual,
                      const void* mask, void* dx, void* scratch, cudaStream_t stream,
                      const uint32_t* mask_bits, int accumulate) {
  const int64_t frames = s.clips * s.T;
  if (accumulate && (s.k != 1 || s.stride == 1))
    return fail(TSM_ERR_INVALID, "dgrad: accumulate is for strided 1x1 only");
  const int64_t ho = s.h_out(), wo = s.w_out();
  if (s.c_in % 16 != 0 || s.c_out % 64 != 0)
    return fail(TSM_ERR_UNSUPPORTED, "dgrad: c_in % 16 or c_out % 64");
  if (mask_bits && (mask || s.c_in % 32))
    return fail(TSM_ERR_INVALID, "dgrad: one mask kind; bitmask needs c_in % 32");
  if (halo_ok(s) && !residual)  // stride-1 3x3 dgrad = 3x3 conv of dy with flipped W^T
    return halo_conv(s, dy, wt, nullptr, mask, dx, 0, stream, nullptr, mask_bits);
  if (halo128_ok(s) && !residual && !mask)
    return halo128_conv(s, dy, wt, nullptr, dx, 0, stream, nullptr, mask_bits);
  if (shift1_ok(s) && !mask && !accumulate)  // adjoint shift + skip, 64 channels
    return shift1x1_conv(s, dy, wt, nullptr, residual, dx, 0, stream, nullptr, mask_bits, true);
  const int bn = pick_bn(s.c_in);
  Maps mp{};
  CUtensorMap &ma = mp.a, &mb = mp.b;
  Params p = base_params();
  PairB pb;
  p.n_tiles = (int)((s.c_in + bn - 1) / bn);
  p.n_total = (int)s.c_in;
  p.residual = static_cast<const __nv_bfloat16*>(residual);
  p.mask = static_cast<const __nv_bfloat16*>(mask);
  p.mask_bits = mask_bits;
  p.bits_ld = (int)(s.c_in / 32);
  p.out = static_cast<__nv_bfloat16*>(dx);
  p.ldo = (int)s.c_in;
  p.map_mode = gemm::MAP_LINEAR;
  p.b = w_load();
  if (s.k == 1) {
    const int64_t rows_out = frames * ho * wo;
    TSM_TRY(map_w2d(&mb, wt, s.c_out, s.c_in, 64, bn));
    TSM_TRY(pb.make(wt, s.c_out, s.c_in, bn));
    p.k_blocks = (int)(s.c_out / BK);
    // The skip-gradient residual can enter the MMA as identity k-blocks (see
    // conv_fwd); its slabs are loaded at the adjoint-shift row offsets of
    // their channel group, so the slab width follows the shift split.
    const int kcr = (s.F || s.B) ? std::min(shift_kc(s.F), shift_kc(s.F + s.B)) : 64;
    const bool fused = residual && s.stride == 1 && kcr >= 32 && bn % 64 == 0 &&
                       s.c_in % bn == 0 && s.c_in % gemm::EC == 0 && s.c_out / BK <= fuse_res_kb();
    int kca_dg = fused ? kcr : 64;
    if (s.stride == 1) {
      // clip-structured tiles so the adjoint shift is a row offset per clip
      const int64_t rows = s.T * s.H * s.W;
      TSM_TRY(map_act3d(&ma, dy, s.c_out, rows, s.clips, kca_dg, BM));
      p.map_mode = gemm::MAP_CLIP;
      p.rows_per_clip = (int)rows;
      p.tiles_per_clip = (int)((rows + BM - 1) / BM);
      p.m_tiles = (int)(s.clips * p.tiles_per_clip);
      p.a = act_load((int)rows);
    } else {
      TSM_TRY(map_w2d(&ma, dy, s.c_out, rows_out, 64, BM));
      p.m_total = (int)rows_out;
      p.m_tiles = (p.m_total + BM - 1) / BM;
      p.a = w_load();
    }
    if (s.F || s.B) {
      if (s.stride != 1) return fail(TSM_ERR_INVALID, "dgrad: shift with stride");
      if (s.F % 8 || s.B % 8) return fail(TSM_ERR_UNSUPPORTED, "dgrad: shift split % 8");
      p.shift_out = 1;
      p.sg0 = (int)s.F;
      p.sg1 = (int)(s.F + s.B);
      p.hw = (int)(s.H * s.W);
      p.frames = (int)s.T;
    }
    if (s.stride != 1) {
      if (residual || mask) return fail(TSM_ERR_UNSUPPORTED, "dgrad: strided 1x1 epilogue");
      if (!accumulate)
        TSM_CUDA_TRY(cudaMemsetAsync(dx, 0, (size_t)(frames * s.H * s.W * s.c_in * 2), stream));
      p.scatter = 1;
      p.acc_out = accumulate;
      p.sc_wo = (int)wo;
      p.sc_ho = (int)ho;
      p.sc_stride = s.stride;
      p.sc_wi = (int)s.W;
      p.sc_hi = (int)s.H;
    }
    TSM_TRY(setup_epilogue(p, mp, s.clips));
    if (p.acc_out && !p.tma_out)
      return fail(TSM_ERR_UNSUPPORTED, "dgrad: accumulate needs c_in % 32");
    if (fused && p.tma_out) {
      const int64_t rows = s.T * s.H * s.W;
      TSM_TRY(map_act3d(&mp.res, residual, s.c_in, rows, s.clips, kcr, BM));
      p.r = act_load((int)rows, (int)s.F, (int)(s.F + s.B), (int)(-s.H * s.W), (int)(s.H * s.W));
      p.res_kb = bn / 64;
      p.residual = nullptr;
    } else if (kca_dg != 64) {  // epilogue path after all: plain 64-channel A slabs
      kca_dg = 64;
      TSM_TRY(map_act3d(&ma, dy, s.c_out, s.T * s.H * s.W, s.clips, 64, BM));
    }
    TSM_TRY(dispatch_fwd(bn, kca_dg, mp, p, stream, pb.get()));
    // TMA path: rows leaving the clip were clipped; fill the vacated frames
    if (p.shift_out && p.tma_out)
      TSM_TRY(shift_out_boundary(dx, residual, mask, s.clips, s.T, s.H * s.W, s.c_in, s.F, s.B,
                                 stream, mask_bits));
    return TSM_OK;
  }
  if (s.k == 3 && s.stride == 2 && s.H == 2 * ho && s.W == 2 * wo) {
    // Sub-pixel decomposition.  dx(2a+p, 2b+q) only meets the taps whose
    // parity matches (p, q): row tap r reads dy row a+d with (p=0: r=1, d=0),
    // (p=1: r=2, d=0 | r=0, d=1), the same for columns.  Each parity class
    // is a stride-1 conv over dy with 1, 2, 2 or 4 taps at offsets {0, 1}
    // (9 taps in total, against 36 over a zero-inserted dy), scattered to
    // its quarter of dx.  Every dx row is written by exactly one class.
    TSM_TRY(map_im2col_box(&ma, dy, s.c_out, wo, ho, frames, 0, 0, 1, 64, BM));
    TSM_TRY(map_w2d(&mb, wt, 9 * s.c_out, s.c_in, 64, bn));
    TSM_TRY(pb.make(wt, 9 * s.c_out, s.c_in, bn));
    p.m_total = (int)(frames * ho * wo);
    p.m_tiles = (p.m_total + BM - 1) / BM;
    p.scatter = 1;
    p.sc_wo = (int)wo;
    p.sc_ho = (int)ho;
    p.sc_stride = 2;
    p.sc_wi = (int)s.W;
    p.sc_hi = (int)s.H;
    auto tap_of = [](int par, int d) { return par == 0 ? 1 : (d == 0 ? 2 : 0); };
    // All four classes in one launch: their taps are listed as 9 virtual
    // taps (A: dy offsets (dr, ds); B: the flipped weight tap), class c
    // owning k-blocks [cls_kb[c], cls_kb[c + 1]).  The tile walk visits the
    // four classes of an M tile on neighbouring CTAs, so dy is read from HBM
    // once and every dx pixel pair is written in the same window.
    // (TSM_SUBPIX_MERGED=0: one launch per class, A/B)
    const bool merged = subpix_merged();
    unsigned long long tmap = 0;
    int vrs = 0, vt = 0;
    p.cls_kb[0] = 0;
    for (int cls = 0; cls < 4; ++cls) {
      const int ph = cls >> 1, pw = cls & 1;
      const int th = ph + 1, tw = pw + 1;  // taps per axis in this class
      int map = 0;
      for (int dr = 0; dr < th; ++dr)
        for (int ds = 0; ds < tw; ++ds) {
          // w_dgrad holds tap (r, s) at the flipped index (2-r)*3 + (2-s)
          const int r = tap_of(ph, dr), c = tap_of(pw, ds);
          const int wt_tap = (2 - r) * 3 + (2 - c);
          map |= wt_tap << (4 * (dr * tw + ds));
          tmap |= (unsigned long long)wt_tap << (4 * vt);
          vrs |= (dr | (ds << 1)) << (2 * vt);
          ++vt;
        }
      p.cls_kb[cls + 1] = p.cls_kb[cls] + (int)(th * tw * s.c_out / BK);
      p.cls_oh[cls] = ph;
      p.cls_ow[cls] = pw;
      if (merged) continue;
      p.k_blocks = (int)(th * tw * s.c_out / BK);
      p.a = im2col_load((int)ho, (int)wo, 1, 0, (int)s.c_out, tw, 0);
      p.b.tap_map = (unsigned long long)map;
      p.b.c_in = (int)s.c_out;
      p.sc_oh = ph;
      p.sc_ow = pw;
      if (cls == 0) TSM_TRY(setup_epilogue(p, mp, s.clips));
      TSM_TRY(dispatch_fwd(bn, 64, mp, p, stream, pb.get()));
    }
    if (merged) {
      p.cls_n = 4;
      p.k_blocks = (int)(4 * s.c_out / BK);  // the longest class (pair choice)
      p.a = im2col_load((int)ho, (int)wo, 1, 0, (int)s.c_out, 2, 0);
      p.a.vtaps = 9;
      p.a.vtap_rs = vrs;
      p.b.tap_map = tmap;
      p.b.c_in = (int)s.c_out;
      TSM_TRY(setup_epilogue(p, mp, s.clips));
      if (p.tma_out && !p.acc_out && subpix_tma_enabled() && wo <= BM &&
          (BM / wo) * wo >= 120) {
        // row-aligned M tiles of R whole class rows; dx viewed as (C, q, Wo,
        // p, frames * Ho): class (p, q) row (f, ho) is index f * Ho + ho of
        // the last dimension (stride two dx rows).  Only where the tiles
        // lose little of the MMA's 128 rows: 126 at 14 / 7 wide (res4.0
        // 139 -> 125 us); 112 at 28 wide lost more than the TMA store saves
        // (res3.0 238 -> 251 us).
        const int R = (int)(BM / wo);
        p.m_rows = (int)(R * wo);
        p.sc_rows = R;
        p.sc_tma = 1;
        p.m_tiles = (int)((frames * ho + R - 1) / R);
        const uint64_t c2 = (uint64_t)s.c_in * 2;
        uint64_t dims[5] = {(uint64_t)s.c_in, 2, (uint64_t)wo, 2, (uint64_t)(frames * ho)};
        uint64_t strides[4] = {c2, 2 * c2, (uint64_t)s.W * c2, 2 * (uint64_t)s.W * c2};
        uint32_t box[5] = {(uint32_t)gemm::EC, 1, (uint32_t)wo, 1, (uint32_t)R};
        TSM_TRY(encode_tiled(&mp.out, dx, 5, dims, strides, box));
      }
      TSM_TRY(dispatch_fwd(bn, 64, mp, p, stream, pb.get()));
    }
    return TSM_OK;
  }
  // kxk: dgrad = conv_kxk(dy (zero-inserted if strided), flipped W^T), pad k/2.
  const void* src = dy;
  if (s.stride != 1) {
    if (s.stride != 2 || s.H != 2 * ho || s.W != 2 * wo)
      return fail(TSM_ERR_UNSUPPORTED, "dgrad: strided kxk needs stride 2 and even extents");
    if (!scratch) return fail(TSM_ERR_INVALID, "dgrad: strided kxk needs scratch");
    TSM_TRY(zero_insert(dy, scratch, frames, ho, wo, s.c_out, stream));
    src = scratch;
  }
  const int kk = s.k * s.k;
  TSM_TRY(map_im2col(&ma, src, s.c_out, s.W, s.H, frames, s.k, 1, s.k / 2, 64, BM));
  TSM_TRY(map_w2d(&mb, wt, kk * s.c_out, s.c_in, 64, bn));
  TSM_TRY(pb.make(wt, kk * s.c_out, s.c_in, bn));
  p.m_total = (int)(frames * s.H * s.W);
  p.m_tiles = (p.m_total + BM - 1) / BM;
  p.k_blocks = (int)(kk * s.c_out / BK);
  p.a = im2col_load((int)s.H, (int)s.W, 1, s.k / 2, (int)s.c_out, s.k, 0);
  TSM_TRY(setup_epilogue(p, mp, s.clips));
  return dispatch_fwd(bn, 64, mp, p, stream, pb.get());
}

// ---------------------------------------------------------------------------
// Weight gradient: dw[c_out][k*k*c_in] (fp32) = sum_p dy[p, co] * im2col(shift(x))[p, :]
// Split over K (pixels) into `splits` fixed ranges; partials go to `ws`
// (splits * c_out * N fp32) and are summed in split order.
// c_out < 128 (the 64-wide res2 convs): put the wide side on M instead of
// padding M = c_out to 128 — D[k*k*c_in][c_out], transposed on reduction.
static bool wgrad_swapped(const ConvShape& s) {
  return s.c_out < BM && s.k * s.k * s.c_in >= BM;
}

int splits_for(int64_t tiles, int64_t kb);

// The X operand's slab width: the shift split picks it for the shifted 1x1
// (shift_kc), 64 channels otherwise.
static int wgrad_kcx(const ConvShape& s) {
  if (s.k == 1 && s.stride == 1) return std::min(shift_kc(s.F), shift_kc(s.F + s.B));
  return 64;
}

// Tiling of one weight gradient (kept in one place: the workspace size
// depends on the split count).
struct WgradPlan {
  bool swap, pair;
  int bn, bk;            // N tile, pixels (K) per stage
  int64_t tiles;         // single-CTA tiles before the K split
  int kb_per_clip;
  int64_t k_blocks;
  int splits;
  int krem_rows, krem_clips;  // > 0: gathered clip remainders (see wgrad_plan)
};

// Pixel rows per box / stage of the single-CTA weight gradients
// (TSM_WGRAD_BK=64|128).  128 measured (tools/bench_gemms.py, 64 -> 128):
// res2 conv3 233 -> 181 us, res3.0 conv1 282 -> 265, res3 conv3 117 -> 105,
// res2 conv1 239 -> 234 / 159 -> 151 (virtual channels), res3 conv2 155 -> 151.
static int wgrad_single_bk() {
  static const int bk = [] {
    const char* e = getenv("TSM_WGRAD_BK");
    return e ? atoi(e) : 128;
  }();
  return bk;
}

static bool krem_enabled() {  // TSM_KREM_GATHER=0: padded last K block per clip (A/B)
  static const bool on = [] {
    const char* e = getenv("TSM_KREM_GATHER");
    return !e || atoi(e) != 0;
  }();
  return on;
}

static WgradPlan wgrad_plan(const ConvShape& s) {
  WgradPlan w{};
  const int64_t n = s.k * s.k * s.c_in;
  w.swap = wgrad_swapped(s);
  int64_t m_tiles;
  if (w.swap) {
    w.bn = 64;
    m_tiles = (n + BM - 1) / BM;
    w.tiles = m_tiles;
  } else {
    w.bn = pick_bn(n);
    m_tiles = (s.c_out + BM - 1) / BM;
    w.tiles = m_tiles * ((n + w.bn - 1) / w.bn);
  }
  w.pair = !w.swap && use_pair_wgrad(w.bn, wgrad_kcx(s), s, m_tiles);
  w.bk = w.pair ? kWgradPairBK
                : (wgrad_single_bk() == 128 &&
                           gemm_host::wgrad_bk128_ok(w.swap, w.bn, wgrad_kcx(s))
                       ? 128
                       : BK);
  const int64_t rows_per_clip = s.T * s.h_out() * s.w_out();
  if (s.F || s.B) {
    // shifted x: K blocks stay inside a clip (frame offsets, zero fill).
    // A short last block per clip (res5: 392 = 3 x 128 + 8 rows) is gathered
    // with those of bk / rem clips into one block ({KC, rem, bk / rem}
    // boxes of the same 3-D maps; rows keep their clip's offsets).
    // (clips shorter than one block stay padded: gathering every block of
    // such a GEMM faulted on B200 — an unexplained TMA exception; the tiny
    // shapes it would serve do not occur at the benchmark extent)
    const int64_t rem = rows_per_clip % w.bk;
    if (rem && w.bk % rem == 0 && rem * 4 <= w.bk && rows_per_clip >= w.bk && krem_enabled()) {
      w.kb_per_clip = (int)(rows_per_clip / w.bk);
      w.krem_rows = (int)rem;
      w.krem_clips = (int)(w.bk / rem);
      w.k_blocks = s.clips * w.kb_per_clip + (s.clips + w.krem_clips - 1) / w.krem_clips;
    } else {
      w.kb_per_clip = (int)((rows_per_clip + w.bk - 1) / w.bk);
      w.k_blocks = s.clips * w.kb_per_clip;
    }
  } else {
    // K = all pixels, linear: no padded last block per clip (res5: 392
    // rows per clip = 3 x 128 + 8, a third of the K work)
    w.kb_per_clip = 0;
    w.k_blocks = (s.clips * rows_per_clip + w.bk - 1) / w.bk;
  }
  w.splits = splits_for(w.tiles, w.k_blocks);
  return w;
}

int wgrad_splits(const ConvShape& s) { return wgrad_plan(s).splits; }

int splits_for(int64_t tiles, int64_t kb) {
  // Split K so tiles * splits fills whole waves of the persistent grid (a
  // wave a few tiles over, e.g. 5 x 60 = 300 on 148 SMs, costs a whole
  // extra tile time).  Cost in k-block units: waves x (k-blocks per tile +
  // ~5 for the fp32 partial-tile epilogue) + the reduction's partial reads.
  const int64_t sms = num_sms(), smax = std::max<int64_t>(1, kb / 4);
  int64_t best = 1;
  double best_cost = 1e30;
  for (int64_t sp = 1; sp <= std::min<int64_t>(smax, 4 * sms); ++sp) {
    const int64_t t = tiles * sp, waves = (t + sms - 1) / sms;
    const double cost = (double)waves * (double)((kb + sp - 1) / sp + 5) +
                        0.5 * (double)t / (double)sms;
    if (cost < best_cost) {
      best_cost = cost;
      best = sp;
    }
  }
  return (int)best;
}

static bool use_vshift_wgrad(const ConvShape& s) {
  static const int on = [] {  // TSM_VSHIFT=0: 8-channel slabs instead (A/B)
    const char* e = getenv("TSM_VSHIFT");
    return e ? atoi(e) : 1;
  }();
  return on && s.c_out == 64 && vshift_ok(s);
}

static size_t wgrad_vshift_workspace_bytes(const ConvShape& s);

// Bias gradient of a CTA-pair 3x3 weight gradient as a separate column sum
// over dY (TSM_DB_APART = the largest c_out for which it applies; 0 =
// always fused).  The fused sum makes each pair stage wait for the bias
// warps after the MMA consumed it; measured at TSM-R50 shapes
// (tools/bench_gemms.py, with / without the fused sum): res4 conv2 128 /
// 100 us, res5 conv2 150 / 111 against a ~10-13 us column sum; the 1x1s
// (res4 conv1 78 / 67, res5 conv1 84 / 72, conv3) keep it fused.
static bool db_apart(const ConvShape& s, bool pair) {
  static const int cmax = [] {
    const char* e = getenv("TSM_DB_APART");
    return e ? atoi(e) : 512;
  }();
  return pair && s.k == 3 && s.c_out <= cmax;
}

// Interleaved split-K chunk (k-blocks) for the weight gradients of shifted
// operands (TSM_WGRAD_ILV, 0: contiguous K range per split).
static int wgrad_ilv() {
  static const int q = [] {
    const char* e = getenv("TSM_WGRAD_ILV");
    return e ? atoi(e) : 4;
  }();
  return q;
}

size_t wgrad_workspace_bytes(const ConvShape& s) {
  // weight-gradient partials + bias-gradient partials (or the column sum's)
  if (halo_ok(s)) return halo_wgrad_workspace_bytes(s);
  if (halo128_wgrad_ok(s)) return halo128_wgrad_workspace_bytes();
  if (shift1_ok(s)) return shift1_wgrad_workspace_bytes(s);
  if (use_vshift_wgrad(s)) return wgrad_vshift_workspace_bytes(s);
  const size_t b = (size_t)wgrad_splits(s) * (size_t)s.c_out * (size_t)(s.k * s.k * s.c_in + 1) * 4;
  const size_t cs = (size_t)colsum_workspace_floats(s.clips * s.T * s.h_out() * s.w_out(), s.c_out) * 4;
  return std::max(b, cs);
}

// Weight gradient of a narrow-split shifted 1x1 (see vshift_ok), c_out
// = 64: the X side in virtual channels on M (64 + c_in rows, 64-byte slab
// rows), partials reduced with the virtual -> real row map.
static int vshift_bk() { return wgrad_single_bk() == 128 ? 128 : BK; }

static int64_t vshift_splits(const ConvShape& s) {
  const int64_t rows_out = s.T * s.H * s.W, bk = vshift_bk();
  return splits_for(((2 * kVShift + s.c_in) + BM - 1) / BM, s.clips * ((rows_out + bk - 1) / bk));
}

static size_t wgrad_vshift_workspace_bytes(const ConvShape& s) {
  return (size_t)vshift_splits(s) * (size_t)s.c_out * (size_t)(2 * kVShift + s.c_in + 1) * 4;
}

static tsm_status conv_wgrad_vshift(const ConvShape& s, const void* x, const void* dy, float* dw,
                                    float* db, float* ws, cudaStream_t stream) {
  const int64_t rows = s.T * s.H * s.W, mv = 2 * kVShift + s.c_in;
  Maps mp{};
  Params p = base_params();
  const int bk = vshift_bk();
  TSM_TRY(map_act3d(&mp.b, dy, s.c_out, rows, s.clips, 64, bk));
  TSM_TRY(map_act3d(&mp.a, x, s.c_in, rows, s.clips, kVShift, bk));
  p.a = act_load((int)rows, 0, 0, (int)(-s.H * s.W), (int)(s.H * s.W));
  p.a.vg = kVShift;
  p.b = act_load((int)rows);
  p.kb_per_clip = (int)((rows + bk - 1) / bk);
  p.k_blocks = (int)(s.clips * p.kb_per_clip);
  p.splits = (int)vshift_splits(s);
  p.epi = gemm::EPI_F32;
  p.m_total = (int)mv;
  p.m_tiles = (int)((mv + BM - 1) / BM);
  p.n_total = (int)s.c_out;
  p.n_tiles = 1;
  p.out_f32 = ws;
  float* db_part = ws + (size_t)p.splits * s.c_out * mv;
  if (db) {
    p.db_mode = 2;
    p.db_part = db_part;
    p.db_c = (int)s.c_out;
  }
  TSM_TRY(bk == 128 ? gemm_host::dispatch_wgrad_swapped_bk128(kVShift, mp, p, stream)
                    : dispatch_wgrad_swapped(kVShift, mp, p, stream));
  TSM_TRY(splitk_reduce_transpose_vmap(ws, dw, p.splits, mv, s.c_in, s.c_out, s.F, s.B, kVShift,
                                       stream));
  return db ? splitk_reduce(db_part, db, p.splits, s.c_out, stream) : TSM_OK;
}

tsm_status conv_wgrad(const ConvShape& s, const void* x, const void* dy, float* dw, float* db, float* ws,
                      cudaStream_t stream) {
  const int64_t ho = s.h_out(), wo = s.w_out();
  const int64_t n = s.k * s.k * s.c_in;
  const int64_t rows_out = s.T * ho * wo;  // pixels per clip of dy
  if (s.c_out % 64 != 0) return fail(TSM_ERR_UNSUPPORTED, "wgrad: c_out % 64");
  if (halo_ok(s)) return halo_wgrad(s, x, dy, dw, db, ws, stream);
  if (halo128_wgrad_ok(s)) return halo128_wgrad(s, x, dy, dw, db, ws, stream);
  if (shift1_ok(s)) return shift1_wgrad(s, x, dy, dw, db, ws, stream);
  if (use_vshift_wgrad(s)) return conv_wgrad_vshift(s, x, dy, dw, db, ws, stream);
  const WgradPlan plan = wgrad_plan(s);
  const bool swap = plan.swap;
  const int bk = plan.bk;
  Maps mp{};
  // the dY operand and the X (im2col / shifted) operand; swap decides which
  // is A (M side) and which is B (N side)
  CUtensorMap& m_dy = swap ? mp.b : mp.a;
  CUtensorMap& m_x = swap ? mp.a : mp.b;
  Params p = base_params();
  const bool lin_k = plan.kb_per_clip == 0;  // unshifted: K over all pixels
  gemm::OpLoad l_x, l_dy;
  if (lin_k) {
    TSM_TRY(map_w2d(&m_dy, dy, s.c_out, s.clips * rows_out, 64, bk));
    l_dy = w_load();
  } else {
    TSM_TRY(map_act3d(&m_dy, dy, s.c_out, rows_out, s.clips, 64, bk));
    l_dy = act_load((int)rows_out);
  }
  int kcx;
  if (s.k == 1 && s.stride == 1) {
    kcx = wgrad_kcx(s);
    if (!kcx || s.c_in % 64) return fail(TSM_ERR_UNSUPPORTED, "wgrad1x1: split/c_in");
    if (lin_k) {
      TSM_TRY(map_w2d(&m_x, x, s.c_in, s.clips * rows_out, kcx, bk));
      l_x = w_load();
    } else {
      TSM_TRY(map_act3d(&m_x, x, s.c_in, s.T * s.H * s.W, s.clips, kcx, bk));
      l_x = act_load((int)rows_out, (int)s.F, (int)(s.F + s.B), (int)(-s.H * s.W),
                     (int)(s.H * s.W));
    }
  } else {
    if (s.F || s.B) return fail(TSM_ERR_INVALID, "wgrad: shift only before 1x1 stride 1");
    if (s.c_in % 64)
      return fail(TSM_ERR_UNSUPPORTED, "wgrad: im2col operand needs c_in % 64 == 0");
    kcx = 64;
    TSM_TRY(map_im2col(&m_x, x, s.c_in, s.W, s.H, s.clips * s.T, s.k, s.stride, s.k / 2, kcx, bk));
    l_x = im2col_load((int)ho, (int)wo, s.stride, s.k / 2, (int)s.c_in, s.k, (int)rows_out);
  }
  p.kb_per_clip = plan.kb_per_clip;
  p.k_blocks = (int)plan.k_blocks;
  p.splits = plan.splits;
  p.epi = gemm::EPI_F32;
  if ((s.F || s.B) && p.splits > 1) p.k_ilv = wgrad_ilv();
  if (plan.krem_rows) {  // gathered clip remainders: the A / B maps boxed {KC, rem, clips}
    p.krem_rows = plan.krem_rows;
    p.krem_clips = plan.krem_clips;
    p.krem0 = (int)(s.clips * plan.kb_per_clip);
    const int64_t rows_x = s.T * s.H * s.W;
    CUtensorMap& r_dy = swap ? mp.mask : mp.res;
    CUtensorMap& r_x = swap ? mp.res : mp.mask;
    TSM_TRY(map_act3d(&r_dy, dy, s.c_out, rows_out, s.clips, 64, plan.krem_rows,
                      plan.krem_clips));
    TSM_TRY(map_act3d(&r_x, x, s.c_in, rows_x, s.clips, kcx, plan.krem_rows, plan.krem_clips));
  }
  // (pairs: the bias gradient as a column sum after the GEMM, see db_apart)
  float* const db_sep = db && !swap && db_apart(s, plan.pair) ? db : nullptr;
  if (db_sep) db = nullptr;
  // bias gradient fused into the same pass over dY (partials after the
  // weight-gradient partials in the workspace)
  float* db_part = ws + (size_t)p.splits * s.c_out * n;
  if (db) {
    p.db_mode = swap ? 2 : 1;
    p.db_part = db_part;
    p.db_c = (int)s.c_out;
  }
  auto finish_db = [&]() -> tsm_status {
    return db ? splitk_reduce(db_part, db, p.splits, s.c_out, stream) : TSM_OK;
  };
  if (swap) {
    p.a = l_x;
    p.b = l_dy;
    p.m_total = (int)n;
    p.m_tiles = (int)((n + BM - 1) / BM);
    p.n_total = (int)s.c_out;
    p.n_tiles = 1;
    p.out_f32 = ws;
    TSM_TRY(bk == 128 ? gemm_host::dispatch_wgrad_swapped_bk128(kcx, mp, p, stream)
                      : dispatch_wgrad_swapped(kcx, mp, p, stream));
    TSM_TRY(splitk_reduce_transpose(ws, dw, p.splits, n, s.c_out, stream));
    return finish_db();
  }
  const int bn = plan.bn;
  p.a = l_dy;
  p.b = l_x;
  p.m_total = (int)s.c_out;
  p.m_tiles = (int)((s.c_out + BM - 1) / BM);
  p.n_total = (int)n;
  p.n_tiles = (int)((n + bn - 1) / bn);
  p.out_f32 = p.splits == 1 ? dw : ws;
  TSM_TRY(bk == 128 && !plan.pair ? gemm_host::dispatch_wgrad_bk128(bn, kcx, mp, p, stream)
                                  : dispatch_wgrad(bn, kcx, mp, p, stream, plan.pair));
  if (p.splits > 1)  // weight and bias partials reduced by one launch
    TSM_TRY(splitk_reduce2(ws, dw, (int64_t)s.c_out * n, db_part, db, db ? s.c_out : 0, p.splits,
                           stream));
  else
    TSM_TRY(finish_db());
  // the partials are consumed: the column sum reuses the workspace
  return db_sep ? colsum_bf16(dy, db_sep, ws, s.clips * rows_out, s.c_out, stream) : TSM_OK;
}


// ---------------------------------------------------------------------------
// Whole-bottleneck fusion of the res2 identity unit (fused_block.cuh).
tsm_status bottleneck_fused_fwd(const void* x, const void* w1f, const void* w2f, const void* w3f,
                                const float* b1, const float* b2, const float* b3, void* y,
                                void* r1, void* r2, uint32_t* r1_bits, uint32_t* r2_bits,
                                uint32_t* y_bits, int64_t clips, int64_t T, int64_t H, int64_t W,
                                cudaStream_t stream) {
  using namespace fused;
  int limit = 0;
  TSM_TRY(dyn_smem_limit(bottleneck_fwd_kernel, kSmemLimit, &limit));
  int slots = kMaxSlots;
  while (slots > 2 && Layout::bytes(slots) > limit) --slots;
  if (Layout::bytes(slots) > limit) return fail(TSM_ERR_UNSUPPORTED, "fused block: smem");
  const int64_t frames = clips * T;
  CUtensorMap mx5, mxc5, mw1, mw2, mw3, mr2, my;
  {
    uint64_t dims[5] = {(uint64_t)kC, (uint64_t)W, (uint64_t)H, (uint64_t)T, (uint64_t)clips};
    uint64_t strides[4] = {(uint64_t)kC * 2, (uint64_t)(W * kC * 2), (uint64_t)(H * W * kC * 2),
                           (uint64_t)(T * H * W * kC * 2)};
    uint32_t box[5] = {32, (uint32_t)kHP, (uint32_t)kHR, 1, 1};
    TSM_TRY(encode_tiled(&mx5, x, 5, dims, strides, box));
    uint32_t boxc[5] = {32, (uint32_t)kTW, (uint32_t)kTH, 1, 1};
    TSM_TRY(encode_tiled(&mxc5, x, 5, dims, strides, boxc));
  }
  TSM_TRY(map_w2d(&mw1, w1f, kC, kWd, 64, 64));
  TSM_TRY(map_w2d(&mw2, w2f, 9 * kWd, kWd, 64, 64));
  TSM_TRY(map_w2d(&mw3, w3f, kWd, kC, 64, 256));
  TSM_TRY(map_act4d(&mr2, r2, kWd, W, H, frames, 64, kTW, kTH));
  TSM_TRY(map_act4d(&my, y, kC, W, H, frames, 32, kTW, kTH));
  fused::Params p{};
  p.tiles_y = (int)((H + kTH - 1) / kTH);
  p.tiles_x = (int)((W + kTW - 1) / kTW);
  p.total = (int)(frames * p.tiles_y * p.tiles_x);
  p.T = (int)T;
  p.H = (int)H;
  p.W = (int)W;
  p.b1 = b1;
  p.b2 = b2;
  p.b3 = b3;
  p.r1 = static_cast<__nv_bfloat16*>(r1);
  p.r1_bits = r1_bits;
  p.r2_bits = r2_bits;
  p.y_bits = y_bits;
  p.slots = slots;
  const int grid = std::max(1, std::min(p.total, num_sms()));
  TSM_TRY(gemm_host::launch_maybe_pdl(bottleneck_fwd_kernel, dim3(grid), dim3(kThreads),
                                      Layout::bytes(slots), stream, mx5, mxc5, mw1, mw2, mw3, mr2,
                                      my, p));
  count_launches();
  return cuda_status(cudaGetLastError(), "bottleneck_fwd_kernel launch");
}

// ---------------------------------------------------------------------------
// Space-to-depth stem (head_kernels.cu: stem_s2d): the 7x7/s2 conv1 as a 4x4
// stride-1 conv over xs [frames][H2][W2][16] bf16, window offsets -2..+1
// (im2col origins span [-2, dim-3]), K = 16 taps x 16 channels = 256, 32-byte
// (SW32) K slabs.  Replaces the materialised 2.5 GB im2col matrix.
tsm_status stem_s2d_fwd(const void* xs, const void* wf, const float* bias, void* y,
                        int64_t frames, int64_t H2, int64_t W2, cudaStream_t stream) {
  // halo-tile kernel: one TMA box of 19 x 11 s2d pixels per 16 x 8 outputs,
  // the 16 taps as descriptor offsets (im2col would issue 16 32-byte row
  // requests per output pixel); linear (expand_layer keeps conv1 linear)
  return halo_conv_t<4, 16>(xs, wf, bias, nullptr, y, 0, frames, H2, W2, stream, nullptr,
                            nullptr);
}

// Stem conv + max pool in one kernel (halo_conv.cuh stem_pool_kernel): y
// [frames][Ho][Wo][64] bf16 and the argmax bytes, bitwise those of
// stem_s2d_fwd followed by maxpool_fwd; the stem output is never stored.
bool stem_pool_enabled() {  // TSM_STEM_POOL=0: the two-kernel path (A/B)
  static const bool on = [] {
    const char* e = getenv("TSM_STEM_POOL");
    return !e || atoi(e) != 0;
  }();
  return on;
}

tsm_status stem_pool_fwd(const void* xs, const void* wf, const float* bias, void* y,
                         uint8_t* arg, int64_t frames, int64_t H2, int64_t W2,
                         cudaStream_t stream) {
  using namespace halo;
  int limit = 0;
  TSM_TRY(dyn_smem_limit(stem_pool_kernel, halo::kSmemLimit, &limit));
  CUtensorMap mx, mw;
  TSM_TRY(map_act4d(&mx, xs, 16, W2, H2, frames, 16, kSPHP, kSPHP));
  TSM_TRY(map_w2d(&mw, wf, 16 * 16, 64, 16, 64));
  StemPoolParams p{};
  p.H = (int)H2;
  p.W = (int)W2;
  p.Ho = (int)((H2 + 2 - 3) / 2 + 1);
  p.Wo = (int)((W2 + 2 - 3) / 2 + 1);
  p.tiles_y = (p.Ho + 6) / 7;
  p.tiles_x = (p.Wo + 6) / 7;
  p.total = (int)(frames * p.tiles_y * p.tiles_x);
  p.bias = bias;
  p.y = static_cast<uint4*>(y);
  p.arg = reinterpret_cast<uint2*>(arg);
  const int fixed = 1024 + kSPW + 2 * kSPTile;
  p.stages = std::min(kMaxStages, (limit - fixed) / kSPStride);
  if (p.stages < 2) return fail(TSM_ERR_UNSUPPORTED, "stem_pool: shared memory");
  const int smem = fixed + p.stages * kSPStride;
  const int grid = std::max(1, std::min(p.total, num_sms()));
  TSM_TRY(gemm_host::launch_maybe_pdl(stem_pool_kernel, dim3(grid), dim3(kSPThreads), smem,
                                      stream, mx, mw, p));
  count_launches();
  return cuda_status(cudaGetLastError(), "stem_pool_kernel launch");
}

// Stem weight gradient: the 4 horizontal taps folded into 64 channels
// (stem_x4), the 4 vertical taps as halo descriptor offsets
// (wgrad_halo_kernel<4, 1>: two tap-pair M tiles, 8 x 8 output patches),
// per-CTA partials reduced in a fixed order.  db = the weight-gradient row of
// the all-ones s2d channel at the centre tap (row 2*64 + 2*16 + 3).
static int stem_grid(int64_t clips, int64_t T, int64_t H2, int64_t W2) {
  const int64_t patches = clips * T * ((H2 + 7) / 8) * ((W2 + 7) / 8);
  return (int)std::max<int64_t>(1, std::min<int64_t>(patches, num_sms()));
}

static size_t stem_x4_bytes(int64_t clips, int64_t T, int64_t H2, int64_t W2) {
  return ((size_t)(clips * T * H2 * W2 * 64 * 2) + 255) / 256 * 256;
}

size_t stem_s2d_wgrad_workspace_bytes(int64_t clips, int64_t T, int64_t H2, int64_t W2) {
  return stem_x4_bytes(clips, T, H2, W2) + (size_t)stem_grid(clips, T, H2, W2) * 256 * 64 * 4;
}

// The same with the max-pool backward gathered into the dY operand (halo_conv.cuh
// stem_wgrad_pool_kernel): gy / arg are the pooled gradient and argmax bytes.
bool stem_pool_bwd_enabled() {  // TSM_STEM_POOL_BWD=0: pool backward kernel + stem wgrad (A/B)
  static const bool on = [] {
    const char* e = getenv("TSM_STEM_POOL_BWD");
    return !e || atoi(e) != 0;
  }();
  return on;
}

tsm_status stem_s2d_wgrad_pool(const void* xs, const void* gy, const uint8_t* arg, float* dw,
                               float* db, float* ws, int64_t clips, int64_t T, int64_t H2,
                               int64_t W2, cudaStream_t stream) {
  using namespace halo;
  using WC = WgradCfg<4, 1>;
  if (H2 % 2 || W2 % 2) return fail(TSM_ERR_UNSUPPORTED, "stem_wgrad_pool: odd stem extent");
  const int64_t frames = clips * T;
  const int grid = stem_grid(clips, T, H2, W2);
  float* part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) +
                                         stem_x4_bytes(clips, T, H2, W2));
  int limit = 0;
  TSM_TRY(dyn_smem_limit(stem_wgrad_pool_kernel, halo::kSmemLimit, &limit));
  // the raw s2d halo (the x4 fold of the 4 horizontal taps is built in
  // shared memory): 11 x 11 pixels of 16 channels, unswizzled
  CUtensorMap mx;
  {
    uint64_t dims[4] = {16, (uint64_t)W2, (uint64_t)H2, (uint64_t)frames};
    uint64_t strides[3] = {32, (uint64_t)(W2 * 32), (uint64_t)(H2 * W2 * 32)};
    uint32_t box[4] = {16, (uint32_t)(kPW + 3), (uint32_t)WC::R, 1};
    TSM_TRY(encode_tiled(&mx, xs, 4, dims, strides, box, true));
  }
  // the pooled gradient and the argmax bytes (as bf16 pairs) per patch: 5 x 5
  // pool windows, unswizzled
  CUtensorMap mgy, marg;
  {
    const uint64_t ho = H2 / 2, wo = W2 / 2;
    uint64_t dims[4] = {64, wo, ho, (uint64_t)frames};
    uint64_t strides[3] = {128, wo * 128, ho * wo * 128};
    uint32_t box[4] = {64, 5, 5, 1};
    TSM_TRY(encode_tiled(&mgy, gy, 4, dims, strides, box, true));
    uint64_t adims[4] = {32, wo, ho, (uint64_t)frames};
    uint64_t astrides[3] = {64, wo * 64, ho * wo * 64};
    uint32_t abox[4] = {32, 5, 5, 1};
    TSM_TRY(encode_tiled(&marg, arg, 4, adims, astrides, abox, true));
  }
  StemWgradPoolParams sp{};
  sp.w.patches_y = (int)((H2 + kPW - 1) / kPW);
  sp.w.patches_x = (int)((W2 + kPW - 1) / kPW);
  sp.w.total = (int)(frames * sp.w.patches_y * sp.w.patches_x);
  sp.w.ws = part;
  constexpr int kStage = WC::STAGE + 9216;  // + raw s2d halo and the pool windows
  sp.w.stages = std::min(kMaxStages, (limit - 1024) / kStage);
  sp.gy = static_cast<const uint4*>(gy);
  sp.arg = reinterpret_cast<const uint2*>(arg);
  sp.Ho = (int)(H2 / 2);
  sp.Wo = (int)(W2 / 2);
  sp.H = (int)H2;
  sp.W = (int)W2;
  const int smem = 1024 + sp.w.stages * kStage;
  TSM_TRY(gemm_host::launch_maybe_pdl(stem_wgrad_pool_kernel, dim3(grid), dim3(kSWThreads), smem,
                                      stream, mx, mgy, marg, sp));
  count_launches();
  TSM_TRY(cuda_status(cudaGetLastError(), "stem_wgrad_pool_kernel launch"));
  TSM_TRY(splitk_reduce_transpose(part, dw, grid, 256, 64, stream));
  if (db)
    TSM_CUDA_TRY(cudaMemcpy2DAsync(db, sizeof(float), dw + 2 * 64 + 2 * 16 + 3, 256 * sizeof(float),
                                   sizeof(float), 64, cudaMemcpyDeviceToDevice, stream));
  return TSM_OK;
}

tsm_status stem_s2d_wgrad(const void* xs, const void* dy, float* dw, float* db, float* ws,
                          int64_t clips, int64_t T, int64_t H2, int64_t W2, cudaStream_t stream) {
  const int64_t frames = clips * T;
  const int grid = stem_grid(clips, T, H2, W2);
  void* x4 = ws;
  float* part = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(ws) +
                                         stem_x4_bytes(clips, T, H2, W2));
  TSM_TRY(stem_x4(xs, x4, frames, H2, W2, stream));
  TSM_TRY((halo_wgrad_launch<4, 1>(x4, dy, part, nullptr, frames, H2, W2, grid, stream)));
  TSM_TRY(splitk_reduce_transpose(part, dw, grid, 256, 64, stream));
  if (db)
    TSM_CUDA_TRY(cudaMemcpy2DAsync(db, sizeof(float), dw + 2 * 64 + 2 * 16 + 3, 256 * sizeof(float),
                                   sizeof(float), 64, cudaMemcpyDeviceToDevice, stream));
  return TSM_OK;
}

}  // namespace tsm
