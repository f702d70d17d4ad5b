// Host side of the tcgen05 conv engine: TMA tensor-map construction, tile
// planning and launches for the bottleneck's convolutions (NTHWC bf16
// activations, fp32 accumulation, bf16 outputs).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <string>

#include "common.cuh"
#include "conv_ops.h"
#include "tc_gemm.cuh"

namespace tsm {
namespace {

using gemm::BK;
using gemm::BM;
using gemm::Params;

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

tsm_status encode_tiled(CUtensorMap* map, const void* base, int rank, const uint64_t* dims,
                        const uint64_t* strides_bytes, const uint32_t* box) {
  const Driver& d = driver();
  if (!d.tiled) return fail(TSM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = d.tiled(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(base),
                       dims, strides_bytes, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       swizzle_of(box[0] * 2), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(TSM_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return TSM_OK;
}

// 3-D activation map: (C, rows_per_clip, clips), box {kc, rows, 1}.
tsm_status map_act3d(CUtensorMap* map, const void* base, int64_t c, int64_t rows_per_clip,
                     int64_t clips, int kc, int box_rows) {
  uint64_t dims[3] = {(uint64_t)c, (uint64_t)rows_per_clip, (uint64_t)clips};
  uint64_t strides[2] = {(uint64_t)c * 2, (uint64_t)(rows_per_clip * c * 2)};
  uint32_t box[3] = {(uint32_t)kc, (uint32_t)box_rows, 1};
  return encode_tiled(map, base, 3, dims, strides, box);
}

// 2-D matrix map: row-major [rows][k], box {kc, box_rows}.
tsm_status map_w2d(CUtensorMap* map, const void* base, int64_t k, int64_t rows, int kc,
                   int box_rows) {
  uint64_t dims[2] = {(uint64_t)k, (uint64_t)rows};
  uint64_t strides[1] = {(uint64_t)k * 2};
  uint32_t box[2] = {(uint32_t)kc, (uint32_t)box_rows};
  return encode_tiled(map, base, 2, dims, strides, box);
}

// 4-D im2col map over NTHWC activations (C, W, H, frames) for a kxk conv
// with the given stride and padding; box = kc channels x `pixels` pixels.
tsm_status map_im2col(CUtensorMap* map, const void* base, int64_t c, int64_t w, int64_t h,
                      int64_t frames, int ksize, int stride, int pad, int kc, int pixels) {
  const Driver& d = driver();
  if (!d.im2col) return fail(TSM_ERR_CUDA, "cuTensorMapEncodeIm2col unavailable");
  cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)frames};
  cuuint64_t strides[3] = {(cuuint64_t)c * 2, (cuuint64_t)(w * c * 2), (cuuint64_t)(h * w * c * 2)};
  // Bounding box of window origins: [-pad, dim - 1 + pad - (k - 1)] per axis.
  int lower[2] = {-pad, -pad};
  int upper[2] = {pad - (ksize - 1), pad - (ksize - 1)};
  cuuint32_t es[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
  CUresult r = d.im2col(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims,
                        strides, lower, upper, (cuuint32_t)kc, (cuuint32_t)pixels, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle_of(kc * 2),
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(TSM_ERR_CUDA, "cuTensorMapEncodeIm2col failed (" + std::to_string(r) + ")");
  // Same driver workaround CUTLASS applies for im2col maps of tensors under
  // 128 KiB on drivers <= 13.1 (copy_traits_sm90_im2col.hpp).
  if (d.version <= 13010 && frames * h * w * c * 2 < 131072)
    reinterpret_cast<uint64_t*>(map)[1] &= ~(1ull << 21);
  return TSM_OK;
}

int num_sms() {
  static int n = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  return n;
}

template <int BN, int KCA, int KCB, bool AMN, bool BMN>
tsm_status launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, const Params& p,
                       cudaStream_t stream) {
  using C = gemm::Cfg<BN, KCA, KCB, AMN, BMN>;
  auto kern = gemm::tc_gemm_kernel<BN, KCA, KCB, AMN, BMN>;
  static bool configured = false;
  if (!configured) {
    TSM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      C::SMEM_BYTES));
    configured = true;
  }
  const int tiles = p.m_tiles * p.n_tiles * p.splits;
  const int grid = std::max(1, std::min(tiles, num_sms()));
  kern<<<grid, gemm::kThreads, C::SMEM_BYTES, stream>>>(ma, mb, p);
  count_launches();
  return cuda_status(cudaGetLastError(), "tc_gemm_kernel launch");
}

gemm::OpLoad act_load(int g0 = 0, int g1 = 0, int off0 = 0, int off1 = 0) {
  gemm::OpLoad l{};
  l.mode = gemm::LOAD_ACT3D;
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

int shift_kc(int64_t f) {
  if (f == 0) return 64;
  if (f % 64 == 0) return 64;
  if (f % 32 == 0) return 32;
  if (f % 8 == 0) return 8;
  return 0;
}

// dispatch on (BN, KCA) for K-major x K-major GEMMs
template <bool AMN, bool BMN, int KCB>
tsm_status dispatch_kk(int bn, int kca, const CUtensorMap& ma, const CUtensorMap& mb,
                       const Params& p, cudaStream_t s) {
#define TSM_CASE(BN_, KC_) \
  if (bn == BN_ && kca == KC_) return launch_gemm<BN_, KC_, KCB, AMN, BMN>(ma, mb, p, s);
  TSM_CASE(64, 64) TSM_CASE(128, 64) TSM_CASE(256, 64)
  TSM_CASE(64, 32) TSM_CASE(128, 32) TSM_CASE(256, 32)
  TSM_CASE(64, 8) TSM_CASE(128, 8) TSM_CASE(256, 8)
#undef TSM_CASE
  return fail(TSM_ERR_UNSUPPORTED, "no GEMM instantiation for BN=" + std::to_string(bn) +
                                       " KC=" + std::to_string(kca));
}

int pick_bn(int64_t n) {
  if (n <= 64) return 64;
  if (n <= 128) return 128;
  return 256;
}

}  // namespace

// ---------------------------------------------------------------------------
// 1x1 conv forward with the temporal shift fused into the A loads.
//   x: [clips][T][HW][c_in] bf16, w: [c_out][c_in] bf16, bias fp32[c_out],
//   residual (optional) like y, y: [clips][T][HW][c_out] bf16.
//   y = act(shift(x) . w^T + bias (+ residual))  where act = relu if relu.
tsm_status conv1x1_fwd(const void* x, const void* w, const float* bias, const void* residual,
                       void* y, int64_t clips, int64_t T, int64_t HW, int64_t c_in,
                       int64_t c_out, int64_t F, int64_t B, int relu, cudaStream_t stream) {
  if (c_in % 64 != 0 || c_out % 16 != 0)
    return fail(TSM_ERR_UNSUPPORTED, "conv1x1: c_in must be a multiple of 64, c_out of 16");
  if (F < 0 || B < 0 || F + B > c_in) return fail(TSM_ERR_INVALID, "conv1x1: bad shift split");
  const int kca = shift_kc(F) && shift_kc(F + B) ? std::min(shift_kc(F), shift_kc(F + B)) : 0;
  if (!kca) return fail(TSM_ERR_UNSUPPORTED, "conv1x1: shift split must be a multiple of 8");
  const int64_t rows = T * HW;
  const int bn = pick_bn(c_out);
  CUtensorMap ma, mb;
  TSM_TRY(map_act3d(&ma, x, c_in, rows, clips, kca, BM));
  TSM_TRY(map_w2d(&mb, w, c_in, c_out, 64, bn));
  Params p{};
  p.tiles_per_clip = (int)((rows + BM - 1) / BM);
  p.m_tiles = (int)(clips * p.tiles_per_clip);
  p.n_tiles = (int)((c_out + bn - 1) / bn);
  p.k_blocks = (int)(c_in / BK);
  p.splits = 1;
  p.map_mode = gemm::MAP_CLIP;
  p.rows_per_clip = (int)rows;
  p.a = act_load((int)F, (int)(F + B), (int)-HW, (int)HW);
  p.a.rows_per_clip = (int)rows;
  p.b = w_load();
  p.epi = gemm::EPI_BF16;
  p.n_total = (int)c_out;
  p.bias = bias;
  p.residual = static_cast<const __nv_bfloat16*>(residual);
  p.out = static_cast<__nv_bfloat16*>(y);
  p.ldo = (int)c_out;
  p.relu = relu;
  return dispatch_kk<false, false, 64>(bn, kca, ma, mb, p, stream);
}

}  // namespace tsm
