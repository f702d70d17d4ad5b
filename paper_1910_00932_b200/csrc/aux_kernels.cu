// Helper kernels (see aux_kernels.cuh).  All bandwidth-bound; 16-byte
// vector accesses wherever the layout allows.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "aux_kernels.cuh"
#include "common.cuh"

namespace tsm {
namespace {

constexpr int kT = 256;

inline unsigned grid_for(int64_t n, int per_thread = 1) {
  int64_t b = (n + (int64_t)kT * per_thread - 1) / ((int64_t)kT * per_thread);
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16));
}

// sum_{s < splits} p[s * stride] in split order (fixed -> deterministic),
// eight independent loads in flight: a one-load-at-a-time loop over up to
// ~100 splits is latency-bound.
__device__ __forceinline__ float ordered_sum(const float* __restrict__ p, int splits,
                                             int64_t stride) {
  float a = __ldg(p);
  int s = 1;
  for (; s + 8 <= splits; s += 8) {
    float b[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) b[u] = __ldg(p + (int64_t)(s + u) * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) a += b[u];
  }
  for (; s < splits; ++s) a += __ldg(p + (int64_t)s * stride);
  return a;
}

// Split-K reduction with the splits themselves spread over threads: a
// block holds E = 256 / G float4 output vectors x G split groups; group g
// sums splits [g S / G, (g + 1) S / G) in order, then the G partials are
// added in group order — a fixed order (deterministic) with short chains
// (a thread per output summing ~100-150 splits serially is latency-bound:
// up to 20 us for a 64-element bias gradient).  Two jobs per launch (weight
// and bias partials); `transpose`: out[j * m + i] for element t = i * n + j.
struct RedJob {
  const float4* ws;
  float* out;
  int64_t n4, m, n, blocks;
  int G, transpose;
};

__global__ void __launch_bounds__(256)
    ordered_reduce_kernel(RedJob j0, RedJob j1, int splits) {
  const bool first = blockIdx.x < j0.blocks;
  const RedJob& J = first ? j0 : j1;
  const int64_t b = first ? blockIdx.x : blockIdx.x - j0.blocks;
  const int G = J.G, E = 256 / G;
  const int el = threadIdx.x % E, g = threadIdx.x / E;
  const int64_t e4 = b * E + el;
  const int s0 = g * splits / G, s1 = (g + 1) * splits / G;
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
  if (e4 < J.n4) {
    int s = s0;
    for (; s + 4 <= s1; s += 4) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldg(J.ws + (int64_t)(s + u) * J.n4 + e4);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a.x += v[u].x;
        a.y += v[u].y;
        a.z += v[u].z;
        a.w += v[u].w;
      }
    }
    for (; s < s1; ++s) {
      const float4 v = __ldg(J.ws + (int64_t)s * J.n4 + e4);
      a.x += v.x;
      a.y += v.y;
      a.z += v.z;
      a.w += v.w;
    }
  }
  __shared__ float4 red[256];
  red[threadIdx.x] = a;
  __syncthreads();
  if (g != 0 || e4 >= J.n4) return;
  float4 r = red[el];
  for (int k = 1; k < G; ++k) {
    const float4 v = red[k * E + el];
    r.x += v.x;
    r.y += v.y;
    r.z += v.z;
    r.w += v.w;
  }
  if (!J.transpose) {
    reinterpret_cast<float4*>(J.out)[e4] = r;
  } else {
    const int64_t t = 4 * e4, i = t / J.n, j = t - i * J.n;  // n % 4 == 0: same i
    J.out[j * J.m + i] = r.x;
    J.out[(j + 1) * J.m + i] = r.y;
    J.out[(j + 2) * J.m + i] = r.z;
    J.out[(j + 3) * J.m + i] = r.w;
  }
}

inline RedJob red_job(const float* ws, float* out, int64_t n, int splits, int64_t m,
                      int64_t nn, int transpose) {
  RedJob j{};
  j.ws = reinterpret_cast<const float4*>(ws);
  j.out = out;
  j.n4 = n / 4;
  j.m = m;
  j.n = nn;
  j.transpose = transpose;
  // split groups only while the outputs alone do not fill the machine, and
  // never more groups than splits
  int G = 1;
  while (G < 64 && G * 2 <= splits && j.n4 * G < 148 * 2048) G *= 2;
  j.G = G;
  j.blocks = (j.n4 + (256 / G) - 1) / (256 / G);
  return j;
}

inline bool red_ok(const float* ws, const float* out, int64_t n) {
  return n % 4 == 0 && reinterpret_cast<uintptr_t>(ws) % 16 == 0 &&
         reinterpret_cast<uintptr_t>(out) % 16 == 0;
}

__global__ void splitk_reduce_scalar(const float* __restrict__ ws, float* __restrict__ out,
                                     int splits, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[i] = ordered_sum(ws + i, splits, n);
  }
}

__global__ void zero_insert_kernel(const uint4* __restrict__ dy, uint4* __restrict__ out,
                                   int64_t frames, int64_t ho, int64_t wo, int64_t c8) {
  const int64_t H = 2 * ho, W = 2 * wo;
  const int64_t total = frames * H * W * c8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = i % c8;
    int64_t r = i / c8;
    const int64_t w = r % W;
    r /= W;
    const int64_t h = r % H;
    const int64_t f = r / H;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (!(h & 1) && !(w & 1)) v = dy[((f * ho + h / 2) * wo + w / 2) * c8 + c];
    out[i] = v;
  }
}

// Pass 1: each of <= kColsumBlocks blocks reduces a contiguous row range.
// Thread t owns 8 columns (one 16-byte vector) and a row lane; row lanes are
// combined through shared memory in a fixed order.
constexpr int kColsumBlocks = 592;  // 4 x 148 SMs
constexpr int kColsumThreads = 256;
__global__ void __launch_bounds__(kColsumThreads)
    colsum_partial(const uint4* __restrict__ g, float* __restrict__ part, int64_t rows,
                   int64_t rows_per_block, int c8) {
  __shared__ float red[kColsumThreads * 8];
  const int lanes = kColsumThreads / c8;  // row lanes per block
  const int col = threadIdx.x % c8, lane = threadIdx.x / c8;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t r1 = min(rows, r0 + rows_per_block);
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (lane < lanes) {
    // four rows in flight per thread, accumulated in row order
    int64_t r = r0 + lane;
    for (; r + 3 * lanes < r1; r += 4 * lanes) {
      uint4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(g + (r + u * lanes) * c8 + col);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&v[u]);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += __bfloat162float(b[i]);
      }
    }
    for (; r < r1; r += lanes) {
      const uint4 v = __ldcs(g + r * c8 + col);
      const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += __bfloat162float(b[i]);
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) red[threadIdx.x * 8 + i] = acc[i];
  __syncthreads();
  const int c = c8 * 8;
  for (int j = threadIdx.x; j < c; j += blockDim.x) {
    const int cc = j / 8, ii = j % 8;
    float a = 0.f;
    for (int l = 0; l < lanes; ++l) a += red[(l * c8 + cc) * 8 + ii];
    part[(int64_t)blockIdx.x * c + j] = a;
  }
}

// Pass 2: 8 columns per block, 32 row groups (each a strided chain over the
// partials) combined in a fixed order — a wide grid, short chains.
__global__ void __launch_bounds__(256)
    colsum_final(const float* __restrict__ part, float* __restrict__ db, int64_t blocks,
                 int64_t c) {
  __shared__ float red[32][9];
  const int cl = threadIdx.x & 7, grp = threadIdx.x >> 3;
  const int64_t j = blockIdx.x * 8 + cl;
  float a = 0.f;
  if (j < c)
    for (int64_t b = grp; b < blocks; b += 32) a += part[b * c + j];
  red[grp][cl] = a;
  __syncthreads();
  if (grp == 0 && j < c) {
    float s = red[0][cl];
    for (int g2 = 1; g2 < 32; ++g2) s += red[g2][cl];
    db[j] = s;
  }
}

__device__ __forceinline__ void weights_bf16_body(const WeightJob& j, int64_t i0, int64_t step) {
  const int64_t total = j.co * j.k_pad;
  const int64_t kr = (int64_t)j.kk * j.ci;
  auto* wf = static_cast<__nv_bfloat16*>(j.w_fwd);
  auto* wd = static_cast<__nv_bfloat16*>(j.w_dgrad);
  for (int64_t i = i0; i < total; i += step) {
    const int64_t o = i / j.k_pad, k = i - o * j.k_pad;
    const float v = k < kr ? j.w[o * kr + k] : 0.f;
    wf[i] = __float2bfloat16_rn(v);
    if (wd && k < kr) {
      const int64_t t = k / j.ci, c = k - t * j.ci;
      // dgrad operand: [ci][kk][co] with the tap index reversed
      wd[(c * j.kk + (j.kk - 1 - t)) * j.co + o] = __float2bfloat16_rn(v);
    }
  }
}

__global__ void weights_bf16_kernel(WeightJob j) {
  weights_bf16_body(j, blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
                    (int64_t)gridDim.x * blockDim.x);
}

// All tensors of a network in one launch: blockIdx.y selects the job.
// Unpadded jobs go through 32x32 tiles (per tap t, the [co][ci] slice of W):
// W and the forward copy are read / written along c_in, the tap-flipped
// dgrad copy [ci][kk][co] is written along c_out from the transposed smem
// tile — both sides coalesced (the element-wise form scattered the dgrad
// writes with a c_out stride).  Padded jobs keep the element-wise form.
__global__ void __launch_bounds__(256) weights_bf16_batch_kernel(const WeightJob* __restrict__ jobs) {
  const WeightJob j = jobs[blockIdx.y];
  const int64_t kr = (int64_t)j.kk * j.ci;
  if (j.k_pad != kr) {
    weights_bf16_body(j, blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
                      (int64_t)gridDim.x * blockDim.x);
    return;
  }
  __shared__ float tile[32][33];
  auto* wf = static_cast<__nv_bfloat16*>(j.w_fwd);
  auto* wd = static_cast<__nv_bfloat16*>(j.w_dgrad);
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  const int64_t to = (j.co + 31) / 32, tci = (j.ci + 31) / 32;
  const int64_t tiles = (int64_t)j.kk * to * tci;
  for (int64_t tile_i = blockIdx.x; tile_i < tiles; tile_i += gridDim.x) {
    const int64_t t = tile_i / (to * tci), rem = tile_i - t * to * tci;
    const int64_t o0 = (rem / tci) * 32, c0 = (rem % tci) * 32;
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int64_t o = o0 + ty + 8 * r, c = c0 + tx;
      float v = 0.f;
      if (o < j.co && c < j.ci) {
        const int64_t idx = o * kr + t * j.ci + c;
        v = j.w[idx];
        wf[idx] = __float2bfloat16_rn(v);
      }
      tile[ty + 8 * r][tx] = v;
    }
    if (wd) {
      __syncthreads();
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int64_t c = c0 + ty + 8 * r, o = o0 + tx;
        if (c < j.ci && o < j.co)
          wd[(c * j.kk + (j.kk - 1 - t)) * j.co + o] = __float2bfloat16_rn(tile[tx][ty + 8 * r]);
      }
    }
    __syncthreads();
  }
}

template <typename T>
__device__ __forceinline__ float to_f(T v) {
  return static_cast<float>(v);
}
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) {
  return __bfloat162float(v);
}
template <typename T>
__device__ __forceinline__ T from_f(float v) {
  return static_cast<T>(v);
}
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

// Per-frame transpose [c][hw] -> [hw][c_pad] through a 32x33 smem tile.
template <typename T>
__global__ void to_nthwc_kernel(const T* __restrict__ x, __nv_bfloat16* __restrict__ y,
                                int64_t c, int64_t hw, int64_t c_pad) {
  __shared__ float tile[32][33];
  const int64_t f = blockIdx.z;
  const int64_t c0 = (int64_t)blockIdx.y * 32, p0 = (int64_t)blockIdx.x * 32;
  const T* xf = x + f * c * hw;
  __nv_bfloat16* yf = y + f * hw * c_pad;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t cc = c0 + i, pp = p0 + threadIdx.x;
    tile[i][threadIdx.x] = (cc < c && pp < hw) ? to_f(xf[cc * hw + pp]) : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t pp = p0 + i, cc = c0 + threadIdx.x;
    if (pp < hw && cc < c_pad) yf[pp * c_pad + cc] = __float2bfloat16_rn(tile[threadIdx.x][i]);
  }
}

template <typename T>
__global__ void to_ntchw_kernel(const __nv_bfloat16* __restrict__ x, T* __restrict__ y,
                                int64_t c, int64_t hw) {
  __shared__ float tile[32][33];
  const int64_t f = blockIdx.z;
  const int64_t p0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
  const __nv_bfloat16* xf = x + f * hw * c;
  T* yf = y + f * c * hw;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t pp = p0 + i, cc = c0 + threadIdx.x;
    tile[i][threadIdx.x] = (pp < hw && cc < c) ? __bfloat162float(xf[pp * c + cc]) : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int64_t cc = c0 + i, pp = p0 + threadIdx.x;
    if (cc < c && pp < hw) yf[cc * hw + pp] = from_f<T>(tile[threadIdx.x][i]);
  }
}

__global__ void relu_mask_kernel(const uint4* __restrict__ gy, const uint4* __restrict__ y,
                                 const uint32_t* __restrict__ bits, uint4* __restrict__ g,
                                 int64_t n8) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n8;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint4 a = gy[i];
    if (bits) {  // bitmask (pair-interleaved order, tc::bits_keep): 8 channels
      const uint32_t w = __ldg(bits + i / 4);
      const int b = (int)(i % 4);
      uint32_t* aw = reinterpret_cast<uint32_t*>(&a);
#pragma unroll
      for (int k = 0; k < 4; ++k) aw[k] &= ((w >> (4 * b + k)) & 0x00010001u) * 0xFFFFu;
      g[i] = a;
      continue;
    }
    const uint4 m = y[i];
    const __nv_bfloat16* mb = reinterpret_cast<const __nv_bfloat16*>(&m);
    __nv_bfloat16* ab = reinterpret_cast<__nv_bfloat16*>(&a);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (!(__bfloat162float(mb[k]) > 0.f)) ab[k] = __float2bfloat16_rn(0.f);
    g[i] = a;
  }
}

// Boundary frames of the adjoint shift when the dgrad epilogue moved rows by
// +-H*W with TMA (rows leaving the clip clipped): channels [0,F) of frame
// T-1 and [F,F+B) of frame 0 received nothing and hold +0.0 + residual,
// masked (kernels.cpp:127-157 leaves those cotangent frames zero).
__global__ void shift_boundary_kernel(uint4* __restrict__ dx, const uint4* __restrict__ res,
                                      const uint4* __restrict__ mask,
                                      const uint32_t* __restrict__ bits, int64_t clips, int64_t T,
                                      int64_t hw, int64_t c8, int64_t f8, int64_t b8) {
  const int64_t per = hw * (f8 + b8);
  const int64_t total = clips * per;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = i / per, rem = i - n * per;
    const int64_t p = rem / (f8 + b8), g = rem - p * (f8 + b8);
    const int64_t t = g < f8 ? T - 1 : 0;
    const int64_t idx = ((n * T + t) * hw + p) * c8 + g;
    uint4 v = res ? res[idx] : make_uint4(0, 0, 0, 0);
    if (bits) {  // bitmask (pair-interleaved order, tc::bits_keep): 8 channels
      const uint32_t w = __ldg(bits + idx / 4);
      const int b = (int)(idx % 4);
      uint32_t* vw = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
      for (int k = 0; k < 4; ++k) vw[k] &= ((w >> (4 * b + k)) & 0x00010001u) * 0xFFFFu;
    } else if (mask) {
      const uint4 m = mask[idx];
      const __nv_bfloat16* mb = reinterpret_cast<const __nv_bfloat16*>(&m);
      __nv_bfloat16* vb = reinterpret_cast<__nv_bfloat16*>(&v);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (!(__bfloat162float(mb[k]) > 0.f)) vb[k] = __float2bfloat16_rn(0.f);
    }
    dx[idx] = v;
  }
}

}  // namespace

tsm_status shift_out_boundary(void* dx, const void* residual, const void* mask, int64_t clips,
                              int64_t T, int64_t hw, int64_t c, int64_t F, int64_t B,
                              cudaStream_t st, const uint32_t* mask_bits) {
  if (mask_bits && c % 32) return fail(TSM_ERR_UNSUPPORTED, "shift_out_boundary: bits need c % 32");
  if (c % 8 || F % 8 || B % 8) return fail(TSM_ERR_UNSUPPORTED, "shift_out_boundary: % 8");
  const int64_t total = clips * hw * (F + B) / 8;
  if (total == 0) return TSM_OK;
  shift_boundary_kernel<<<grid_for(total), kT, 0, st>>>(
      static_cast<uint4*>(dx), static_cast<const uint4*>(residual),
      static_cast<const uint4*>(mask), mask_bits, clips, T, hw, c / 8, F / 8, B / 8);
  count_launches();
  return cuda_status(cudaGetLastError(), "shift_out_boundary");
}

namespace {
// out[j][i] = sum_s ws[s][i][j]: reads coalesced along j, fixed split order.
__global__ void splitk_reduce_t_kernel(const float* __restrict__ ws, float* __restrict__ out,
                                       int splits, int64_t m, int64_t n) {
  const int64_t total = m * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const float a = ordered_sum(ws + t, splits, total);
    const int64_t i = t / n, j = t - i * n;
    out[j * m + i] = a;
  }
}
}  // namespace

tsm_status splitk_reduce_transpose(const float* ws, float* out, int splits, int64_t m, int64_t n,
                                   cudaStream_t st) {
  const RedJob j = red_job(ws, out, m * n, splits, m, n, 1);
  if (n % 4 == 0 && red_ok(ws, out, m * n) && j.G > 1) {
    RedJob none{};
    ordered_reduce_kernel<<<(unsigned)j.blocks, 256, 0, st>>>(j, none, splits);
    count_launches();
    return cuda_status(cudaGetLastError(), "splitk_reduce_transpose");
  }
  splitk_reduce_t_kernel<<<grid_for(m * n), kT, 0, st>>>(ws, out, splits, m, n);
  count_launches();
  return cuda_status(cudaGetLastError(), "splitk_reduce_transpose");
}

namespace {
// Virtual-channel layout of a shift split narrower than one 32-channel slab
// (tc_gemm.cuh OpLoad::vg): real channel c of the shifted conv's input lives
// at virtual channel c (c < F, frame t-1), vg + c (F <= c < F + B, frame t+1)
// or 2 vg + c (the rest, frame t).
__device__ __forceinline__ int64_t vchan(int64_t c, int64_t F, int64_t B, int64_t vg) {
  return c < F ? c : (c < F + B ? vg + c : 2 * vg + c);
}

__global__ void splitk_reduce_t_vmap_kernel(const float* __restrict__ ws, float* __restrict__ out,
                                            int splits, int64_t m_v, int64_t ci, int64_t co,
                                            int64_t F, int64_t B, int64_t vg) {
  const int64_t total = ci * co;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = t / co, o = t - c * co;  // reads run along o: coalesced
    out[o * ci + c] = ordered_sum(ws + vchan(c, F, B, vg) * co + o, splits, m_v * co);
  }
}

}  // namespace

tsm_status splitk_reduce_transpose_vmap(const float* ws, float* out, int splits, int64_t m_v,
                                        int64_t ci, int64_t co, int64_t F, int64_t B, int64_t vg,
                                        cudaStream_t st) {
  splitk_reduce_t_vmap_kernel<<<grid_for(ci * co), kT, 0, st>>>(ws, out, splits, m_v, ci, co, F,
                                                                B, vg);
  count_launches();
  return cuda_status(cudaGetLastError(), "splitk_reduce_transpose_vmap");
}

tsm_status splitk_reduce(const float* ws, float* out, int splits, int64_t n, cudaStream_t st) {
  // (G = 1, i.e. the outputs alone fill the machine: the scalar kernel with
  // eight loads in flight per thread measured faster than one float4 chain)
  const RedJob j = red_job(ws, out, n, splits, 0, 0, 0);
  if (red_ok(ws, out, n) && j.G > 1) {
    RedJob none{};
    ordered_reduce_kernel<<<(unsigned)j.blocks, 256, 0, st>>>(j, none, splits);
  } else
    splitk_reduce_scalar<<<grid_for(n), kT, 0, st>>>(ws, out, splits, n);
  count_launches();
  return cuda_status(cudaGetLastError(), "splitk_reduce");
}

tsm_status zero_insert(const void* dy, void* out, int64_t frames, int64_t ho, int64_t wo,
                       int64_t c, cudaStream_t st) {
  if (c % 8) return fail(TSM_ERR_UNSUPPORTED, "zero_insert: c % 8");
  const int64_t total = frames * 4 * ho * wo * (c / 8);
  zero_insert_kernel<<<grid_for(total), kT, 0, st>>>(static_cast<const uint4*>(dy),
                                                     static_cast<uint4*>(out), frames, ho, wo,
                                                     c / 8);
  count_launches();
  return cuda_status(cudaGetLastError(), "zero_insert");
}

int64_t colsum_workspace_floats(int64_t rows, int64_t c) {
  (void)rows;
  return (int64_t)kColsumBlocks * c;
}

tsm_status colsum_bf16(const void* g, float* db, float* ws, int64_t rows, int64_t c,
                       cudaStream_t st) {
  if (c % 8 || c / 8 > kColsumThreads) return fail(TSM_ERR_UNSUPPORTED, "colsum: c");
  const int c8 = (int)(c / 8);
  const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>(kColsumBlocks, (rows + 63) / 64));
  const int64_t rpb = (rows + blocks - 1) / blocks;
  colsum_partial<<<(unsigned)blocks, kColsumThreads, 0, st>>>(static_cast<const uint4*>(g), ws,
                                                             rows, rpb, c8);
  colsum_final<<<(unsigned)((c + 7) / 8), 256, 0, st>>>(ws, db, blocks, c);
  count_launches(2);
  return cuda_status(cudaGetLastError(), "colsum");
}

tsm_status weights_to_bf16(const float* w, void* w_fwd, void* w_dgrad, int64_t co, int64_t ci,
                           int k, int64_t k_pad, cudaStream_t st) {
  WeightJob j{w, w_fwd, w_dgrad, co, ci, k * k, k_pad};
  weights_bf16_kernel<<<grid_for(co * k_pad), kT, 0, st>>>(j);
  count_launches();
  return cuda_status(cudaGetLastError(), "weights_to_bf16");
}

tsm_status weights_to_bf16_batch(const WeightJob* jobs_dev, int njobs, cudaStream_t st) {
  if (njobs <= 0) return TSM_OK;
  weights_bf16_batch_kernel<<<dim3(148, (unsigned)njobs), kT, 0, st>>>(jobs_dev);
  count_launches();
  return cuda_status(cudaGetLastError(), "weights_to_bf16_batch");
}

namespace {
__global__ void splitk_reduce2_kernel(const float* __restrict__ ws1, float* __restrict__ out1,
                                      int64_t n1, const float* __restrict__ ws2,
                                      float* __restrict__ out2, int64_t n2, int splits) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n1 + n2;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool first = i < n1;
    const float* ws = first ? ws1 : ws2;
    const int64_t n = first ? n1 : n2, j = first ? i : i - n1;
    (first ? out1 : out2)[j] = ordered_sum(ws + j, splits, n);
  }
}
}  // namespace

tsm_status splitk_reduce2(const float* ws1, float* out1, int64_t n1, const float* ws2,
                          float* out2, int64_t n2, int splits, cudaStream_t st) {
  const RedJob j0 = red_job(ws1, out1, n1, splits, 0, 0, 0);
  if (red_ok(ws1, out1, n1) && (n2 == 0 || red_ok(ws2, out2, n2)) && j0.G > 1) {
    RedJob j1{};
    if (n2) j1 = red_job(ws2, out2, n2, splits, 0, 0, 0);
    ordered_reduce_kernel<<<(unsigned)(j0.blocks + j1.blocks), 256, 0, st>>>(j0, j1, splits);
    count_launches();
    return cuda_status(cudaGetLastError(), "splitk_reduce2");
  }
  splitk_reduce2_kernel<<<grid_for(n1 + n2), kT, 0, st>>>(ws1, out1, n1, ws2, out2, n2, splits);
  count_launches();
  return cuda_status(cudaGetLastError(), "splitk_reduce2");
}

tsm_status ntchw_to_nthwc(const void* x, tsm_dtype dt, void* y, int64_t frames, int64_t c,
                          int64_t hw, int64_t c_pad, cudaStream_t st) {
  dim3 block(32, 8);
  dim3 grid((unsigned)((hw + 31) / 32), (unsigned)((c_pad + 31) / 32), (unsigned)frames);
  auto* yo = static_cast<__nv_bfloat16*>(y);
  switch (dt) {
    case TSM_F32:
      to_nthwc_kernel<float><<<grid, block, 0, st>>>(static_cast<const float*>(x), yo, c, hw, c_pad);
      break;
    case TSM_F64:
      to_nthwc_kernel<double><<<grid, block, 0, st>>>(static_cast<const double*>(x), yo, c, hw,
                                                      c_pad);
      break;
    case TSM_BF16:
      to_nthwc_kernel<__nv_bfloat16><<<grid, block, 0, st>>>(
          static_cast<const __nv_bfloat16*>(x), yo, c, hw, c_pad);
      break;
    default:
      return fail(TSM_ERR_UNSUPPORTED, "ntchw_to_nthwc: dtype");
  }
  count_launches();
  return cuda_status(cudaGetLastError(), "ntchw_to_nthwc");
}

tsm_status nthwc_to_ntchw(const void* x, void* y, tsm_dtype dt, int64_t frames, int64_t c,
                          int64_t hw, cudaStream_t st) {
  dim3 block(32, 8);
  dim3 grid((unsigned)((c + 31) / 32), (unsigned)((hw + 31) / 32), (unsigned)frames);
  auto* xi = static_cast<const __nv_bfloat16*>(x);
  switch (dt) {
    case TSM_F32:
      to_ntchw_kernel<float><<<grid, block, 0, st>>>(xi, static_cast<float*>(y), c, hw);
      break;
    case TSM_F64:
      to_ntchw_kernel<double><<<grid, block, 0, st>>>(xi, static_cast<double*>(y), c, hw);
      break;
    case TSM_BF16:
      to_ntchw_kernel<__nv_bfloat16><<<grid, block, 0, st>>>(
          xi, static_cast<__nv_bfloat16*>(y), c, hw);
      break;
    default:
      return fail(TSM_ERR_UNSUPPORTED, "nthwc_to_ntchw: dtype");
  }
  count_launches();
  return cuda_status(cudaGetLastError(), "nthwc_to_ntchw");
}

tsm_status relu_mask(const void* gy, const void* y, void* g, int64_t n, cudaStream_t st,
                     const uint32_t* bits) {
  if (n % 8 || (bits && n % 32)) return fail(TSM_ERR_UNSUPPORTED, "relu_mask: n % 8");
  relu_mask_kernel<<<grid_for(n / 8), kT, 0, st>>>(static_cast<const uint4*>(gy),
                                                   static_cast<const uint4*>(y), bits,
                                                   static_cast<uint4*>(g), n / 8);
  count_launches();
  return cuda_status(cudaGetLastError(), "relu_mask");
}

}  // namespace tsm
