// Non-GEMM layers of TSM-ResNet-50 (build_tsm8f, arch.cpp:140-161) and the
// optimizer: 3x3/s2 max pool with the reference's first-max tie rule, global
// average pool, the 2048->classes fully-connected head, the Sigma-y^2 loss
// and momentum SGD.  All gather-form / fixed-order, no float atomics.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <set>
#include <utility>

#include "common.cuh"
#include "head_kernels.cuh"
#include "pool_bwd.cuh"
#include "tc_common.cuh"

namespace tsm {
namespace {

constexpr int kT = 256;

__device__ __forceinline__ uint32_t tc_pack(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

inline unsigned blocks_for(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + kT - 1) / kT, 148 * 32));
}

// max_pool_forward (kernels.cpp:353-390) for the spatial 1x3x3 / stride 2 /
// pad 1 window on NTHWC bf16: padded taps never win; ties keep the first
// element in (h, w) scan order (strict >).  Records the winning tap (0..8).
// One block per output row (frame, ho); one thread = 8 channels (16-byte
// loads) of one output pixel; 32-bit index math only.
__global__ void maxpool_fwd_kernel(const uint4* __restrict__ x, uint4* __restrict__ y,
                                   uint2* __restrict__ arg, int H, int W, int Ho, int Wo,
                                   int C8) {
  // Packed bf16x2 form (the kernel is issue-bound): the window's first valid
  // tap seeds (best, argmax) exactly like the reference's "first element
  // taken" rule, every later tap replaces where v > best (strict, so NaN
  // never replaces and ties keep the first) via compare masks + LOP3 selects.
  const int ho = blockIdx.x % Ho;
  const int64_t f = blockIdx.x / Ho;
  const uint4* xf = x + f * H * W * C8;
  const int64_t orow = (int64_t)blockIdx.x * Wo * C8;
  const int n = Wo * C8;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int wo = i / C8, c = i - wo * C8;
    uint32_t best[4], barg[4];
    bool first = true;
#pragma unroll
    for (int dh = 0; dh < 3; ++dh) {
      const int h = ho * 2 - 1 + dh;
      if (h < 0 || h >= H) continue;
#pragma unroll
      for (int dw = 0; dw < 3; ++dw) {
        const int w = wo * 2 - 1 + dw;
        if (w < 0 || w >= W) continue;
        const uint4 v = __ldg(xf + (h * W + w) * C8 + c);
        const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
        const uint32_t tt = (uint32_t)(dh * 3 + dw) * 0x00010001u;
        if (first) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            best[k] = vw[k];
            barg[k] = tt;
          }
          first = false;
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint32_t m = __hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&vw[k]),
                                           *reinterpret_cast<const __nv_bfloat162*>(&best[k]));
            best[k] = (vw[k] & m) | (best[k] & ~m);
            barg[k] = (tt & m) | (barg[k] & ~m);
          }
        }
      }
    }
    y[orow + i] = make_uint4(best[0], best[1], best[2], best[3]);
    // 16-bit argmax lanes -> one byte per channel
    arg[orow + i] = make_uint2(__byte_perm(barg[0], barg[1], 0x6420),
                               __byte_perm(barg[2], barg[3], 0x6420));
  }
}

// The same pool with the window rows staged by one 1-D TMA bulk copy per
// block: a block owns kPoolR output rows of one frame, i.e. 2 kPoolR + 1
// contiguous input rows (every byte of the input moves HBM -> SMEM in large
// asynchronous copies; the row shared with the next block is an L2 hit).  Taps are then read from shared memory (16-byte chunks, 8 lanes
// per 128-byte pixel: conflict-free) in the same scan order and with the
// same compare / select code as maxpool_fwd_kernel — bitwise the same output
// and argmax.
template <int kPoolR>
__global__ void __launch_bounds__(kT)
    maxpool_fwd_bulk_kernel(const uint4* __restrict__ x, uint4* __restrict__ y,
                            uint2* __restrict__ arg, int H, int W, int Ho, int Wo, int C8,
                            int strips) {
  extern __shared__ __align__(16) uint4 rows[];
  __shared__ __align__(8) uint64_t bar;
  const int strip = blockIdx.x % strips;
  const int64_t f = blockIdx.x / strips;
  const int ho0 = strip * kPoolR;
  const int hbase = 2 * ho0 - 1;  // input row of local row 0
  const int hlo = max(hbase, 0), hhi = min(hbase + 2 * kPoolR, H - 1);
  const int rowq = W * C8;        // uint4 per input row
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
    const uint32_t bytes = (uint32_t)(hhi - hlo + 1) * rowq * 16;
    tc::mbar_arrive_expect_tx(&bar, bytes);
    tc::bulk_load(rows + (hlo - hbase) * rowq, x + (f * H + hlo) * rowq, bytes, &bar);
  }
  __syncthreads();
  tc::mbar_wait(&bar, 0);
  const int per_row = Wo * C8;
  const int n = min(kPoolR, Ho - ho0) * per_row;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int k = i / per_row, r = i - k * per_row;
    const int wo = r / C8, c = r - wo * C8;
    uint32_t best[4], barg[4];
    bool first = true;
#pragma unroll
    for (int dh = 0; dh < 3; ++dh) {
      const int hl = 2 * k + dh, h = hbase + hl;
      if (h < 0 || h >= H) continue;
#pragma unroll
      for (int dw = 0; dw < 3; ++dw) {
        const int w = wo * 2 - 1 + dw;
        if (w < 0 || w >= W) continue;
        const uint4 v = rows[hl * rowq + w * C8 + c];
        const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
        const uint32_t tt = (uint32_t)(dh * 3 + dw) * 0x00010001u;
        if (first) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            best[q] = vw[q];
            barg[q] = tt;
          }
          first = false;
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t m = __hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&vw[q]),
                                           *reinterpret_cast<const __nv_bfloat162*>(&best[q]));
            best[q] = (vw[q] & m) | (best[q] & ~m);
            barg[q] = (tt & m) | (barg[q] & ~m);
          }
        }
      }
    }
    const int64_t o = (f * Ho + ho0 + k) * (int64_t)per_row + r;
    __stcs(y + o, make_uint4(best[0], best[1], best[2], best[3]));
    __stcs(arg + o, make_uint2(__byte_perm(barg[0], barg[1], 0x6420),
                               __byte_perm(barg[2], barg[3], 0x6420)));
  }
}

// max_pool_backward (kernels.cpp:392-455): each input element gathers the
// gradients of the (at most 2x2) windows whose recorded argmax it is, in
// ascending (ho, wo) order.  One block per input row (frame, h).
__global__ void maxpool_bwd_kernel(const uint4* __restrict__ gy, const uint2* __restrict__ arg,
                                   uint4* __restrict__ gx, int H, int W, int Ho, int Wo,
                                   int C8) {
  const int h = blockIdx.x % H;
  const int64_t f = blockIdx.x / H;
  const int64_t obase = f * Ho * Wo * C8;
  const int64_t irow = (int64_t)blockIdx.x * W * C8;
  const int ho0 = max(0, h / 2), ho1 = min(Ho - 1, (h + 1) / 2);
  const int n = W * C8;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int w = i / C8, c = i - w * C8;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int wo0 = max(0, w / 2), wo1 = min(Wo - 1, (w + 1) / 2);
    // the (<= 2 x 2) windows containing (h, w), summed in ascending (ho, wo)
    // order.  The window rows (one for even h, two for odd) are uniform over
    // the block, so that loop is a real loop; the two column candidates are
    // predicated (lanes differ in w parity).
    for (int ho = ho0; ho <= ho1; ++ho) {
      const int dh = h - (ho * 2 - 1);
      if (dh < 0 || dh > 2) continue;
      uint2 av[2];
      uint4 gv[2];
      uint32_t t4[2];
      bool ok[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int wo = wo0 + j, dw = w - (wo * 2 - 1);
        ok[j] = wo <= wo1 && dw >= 0 && dw <= 2;
        t4[j] = (uint32_t)(dh * 3 + dw) * 0x01010101u;
        if (ok[j]) {
          const int64_t o = obase + (ho * Wo + wo) * C8 + c;
          av[j] = __ldg(arg + o);
          gv[j] = __ldg(gy + o);
        }
      }
      // SIMD select: exact per-byte tap equality (bit 7 of each byte of e),
      // widened to bf16-lane masks; unselected lanes add +0
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (!ok[j]) continue;
        auto eqbytes = [&](uint32_t x) {
          x ^= t4[j];
          return ~(((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x) & 0x80808080u;
        };
        const uint32_t m0 = (eqbytes(av[j].x) >> 7) * 0xFFu, m1 = (eqbytes(av[j].y) >> 7) * 0xFFu;
        const uint32_t g[4] = {gv[j].x & __byte_perm(m0, 0, 0x1100),
                               gv[j].y & __byte_perm(m0, 0, 0x3322),
                               gv[j].z & __byte_perm(m1, 0, 0x1100),
                               gv[j].w & __byte_perm(m1, 0, 0x3322)};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          acc[2 * k] += __uint_as_float(g[k] << 16);
          acc[2 * k + 1] += __uint_as_float(g[k] & 0xFFFF0000u);
        }
      }
    }
    uint4 o;
    __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(&o);
#pragma unroll
    for (int k = 0; k < 8; ++k) ob[k] = __float2bfloat16_rn(acc[k]);
    __stcs(gx + irow + i, o);
  }
}

// Even extents (H = 2 Ho, W = 2 Wo): one thread per 2 x 2 input block
// (2a..2a+1, 2b..2b+1) x 8 channels.  Its pixels are covered by the windows
// (a + da, b + db), da, db in {0, 1}: each window's argmax and gradient are
// loaded once (4 loads for 4 pixels instead of 9) and routed by tap:
//   (0,0) <- w00:4                 (0,1) <- w00:5, w01:3
//   (1,0) <- w00:7, w10:1          (1,1) <- w00:8, w01:6, w10:2, w11:0
// summed per pixel in ascending (ho, wo) order, as the general kernel does.
using poolbwd::add_tap;
using poolbwd::pack8;

__global__ void maxpool_bwd2x2_kernel(const uint4* __restrict__ gy, const uint2* __restrict__ arg,
                                      uint4* __restrict__ gx, int Ho, int Wo, int C8) {
  const int a = blockIdx.x % Ho;
  const int64_t f = blockIdx.x / Ho;
  const int W = 2 * Wo;
  const int64_t ob = (f * Ho + a) * Wo * C8;       // window row a
  const int64_t ib = (f * 2 * Ho + 2 * a) * W * C8;  // input row 2a
  const bool down = a + 1 < Ho;
  const int n = Wo * C8;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int b = i / C8, c = i - b * C8;
    const bool right = b + 1 < Wo;
    const int64_t o00 = ob + (int64_t)b * C8 + c;
    const uint2 a00 = __ldg(arg + o00);
    const uint4 g00 = __ldg(gy + o00);
    uint2 a01 = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu), a10 = a01, a11 = a01;  // no tap matches
    uint4 g01 = make_uint4(0, 0, 0, 0), g10 = g01, g11 = g01;
    if (right) {
      a01 = __ldg(arg + o00 + C8);
      g01 = __ldg(gy + o00 + C8);
    }
    if (down) {
      const int64_t o10 = o00 + (int64_t)Wo * C8;
      a10 = __ldg(arg + o10);
      g10 = __ldg(gy + o10);
      if (right) {
        a11 = __ldg(arg + o10 + C8);
        g11 = __ldg(gy + o10 + C8);
      }
    }
    float p00[8] = {0, 0, 0, 0, 0, 0, 0, 0}, p01[8] = {0, 0, 0, 0, 0, 0, 0, 0},
          p10[8] = {0, 0, 0, 0, 0, 0, 0, 0}, p11[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    add_tap(p00, a00, g00, 4);
    add_tap(p01, a00, g00, 5);
    if (right) add_tap(p01, a01, g01, 3);
    add_tap(p10, a00, g00, 7);
    if (down) add_tap(p10, a10, g10, 1);
    add_tap(p11, a00, g00, 8);
    if (right) add_tap(p11, a01, g01, 6);
    if (down) add_tap(p11, a10, g10, 2);
    if (down && right) add_tap(p11, a11, g11, 0);
    const int64_t x0 = ib + (int64_t)(2 * b) * C8 + c;
    __stcs(gx + x0, pack8(p00));
    __stcs(gx + x0 + C8, pack8(p01));
    __stcs(gx + x0 + (int64_t)W * C8, pack8(p10));
    __stcs(gx + x0 + (int64_t)W * C8 + C8, pack8(p11));
  }
}

// maxpool_bwd2x2_kernel with the window rows of gradient and argmax staged
// by 1-D TMA bulk copies: a block owns kPoolBR window rows (2 kPoolBR input
// rows) and loads kPoolBR + 1 rows of each; same routing and summation
// order as maxpool_bwd2x2_kernel (bitwise the same gx).
template <int kPoolBR>
__global__ void __launch_bounds__(kT)
    maxpool_bwd2x2_bulk_kernel(const uint4* __restrict__ gy, const uint2* __restrict__ arg,
                               uint4* __restrict__ gx, int Ho, int Wo, int C8, int strips) {
  extern __shared__ __align__(16) uint4 smg[];
  __shared__ __align__(8) uint64_t bar;
  const int strip = blockIdx.x % strips;
  const int64_t f = blockIdx.x / strips;
  const int a0 = strip * kPoolBR;
  const int nrows = min(kPoolBR + 1, Ho - a0);  // window rows staged
  const int rowq = Wo * C8;                      // uint4 of gy per window row
  uint2* sa = reinterpret_cast<uint2*>(smg + (kPoolBR + 1) * rowq);
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
    const uint32_t gb = (uint32_t)nrows * rowq * 16, ab = (uint32_t)nrows * rowq * 8;
    tc::mbar_arrive_expect_tx(&bar, gb + ab);
    tc::bulk_load(smg, gy + (f * Ho + a0) * rowq, gb, &bar);
    tc::bulk_load(sa, arg + (f * Ho + a0) * rowq, ab, &bar);
  }
  __syncthreads();
  tc::mbar_wait(&bar, 0);
  const int W = 2 * Wo;
  const int n = min(kPoolBR, Ho - a0) * rowq;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int k = i / rowq, r = i - k * rowq;
    const int b = r / C8, c = r - b * C8;
    const int a = a0 + k;
    const bool right = b + 1 < Wo, down = a + 1 < Ho;
    const int s00 = k * rowq + r;
    const uint2 a00 = sa[s00];
    const uint4 g00 = smg[s00];
    uint2 a01 = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu), a10 = a01, a11 = a01;  // no tap matches
    uint4 g01 = make_uint4(0, 0, 0, 0), g10 = g01, g11 = g01;
    if (right) {
      a01 = sa[s00 + C8];
      g01 = smg[s00 + C8];
    }
    if (down) {
      a10 = sa[s00 + rowq];
      g10 = smg[s00 + rowq];
      if (right) {
        a11 = sa[s00 + rowq + C8];
        g11 = smg[s00 + rowq + C8];
      }
    }
    float p00[8] = {0, 0, 0, 0, 0, 0, 0, 0}, p01[8] = {0, 0, 0, 0, 0, 0, 0, 0},
          p10[8] = {0, 0, 0, 0, 0, 0, 0, 0}, p11[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    add_tap(p00, a00, g00, 4);
    add_tap(p01, a00, g00, 5);
    if (right) add_tap(p01, a01, g01, 3);
    add_tap(p10, a00, g00, 7);
    if (down) add_tap(p10, a10, g10, 1);
    add_tap(p11, a00, g00, 8);
    if (right) add_tap(p11, a01, g01, 6);
    if (down) add_tap(p11, a10, g10, 2);
    if (down && right) add_tap(p11, a11, g11, 0);
    const int64_t x0 = ((f * 2 * Ho + 2 * a) * W + 2 * b) * (int64_t)C8 + c;
    __stcs(gx + x0, pack8(p00));
    __stcs(gx + x0 + C8, pack8(p01));
    __stcs(gx + x0 + (int64_t)W * C8, pack8(p10));
    __stcs(gx + x0 + (int64_t)W * C8 + C8, pack8(p11));
  }
}

// global_avg_pool_forward (kernels.cpp:457-478): mean over (t, h, w) per
// (clip, channel).  x: [clips][rows][C] bf16 -> y: [clips][C] fp32.
// 8 channels (16-byte loads) x 32 row lanes per 256-thread block; each lane
// sums its rows in order, the 32 lane sums are added in lane order
// (deterministic).  (One 2-byte load per thread and row was latency-bound.)
__global__ void __launch_bounds__(256) gap_fwd_kernel(const uint4* __restrict__ x,
                                                      float* __restrict__ y, int64_t rows, int C) {
  __shared__ float part[32][64 + 1];
  const int64_t n = blockIdx.y;
  const int cg = threadIdx.x & 7, lane = threadIdx.x >> 3;  // 8 chunks of 8 channels, 32 lanes
  const int c8 = C / 8, chunk = blockIdx.x * 8 + cg;
  float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (chunk < c8) {
    const uint4* xn = x + n * rows * c8 + chunk;
    for (int64_t r = lane; r < rows; r += 32) {
      const uint4 v = __ldg(xn + r * c8);
      const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        acc[2 * k] += __uint_as_float(w[k] << 16);
        acc[2 * k + 1] += __uint_as_float(w[k] & 0xFFFF0000u);
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) part[lane][cg * 8 + i] = acc[i];
  __syncthreads();
  if (threadIdx.x < 64) {
    const int cc = blockIdx.x * 64 + threadIdx.x;
    float s = 0.f;
    for (int l = 0; l < 32; ++l) s += part[l][threadIdx.x];
    if (cc < C) y[n * C + cc] = s / (float)rows;
  }
}

// global_avg_pool_backward (kernels.cpp:480-501), writing bf16 NTHWC.
// One block per (row chunk, clip); one thread = 8 channels (16-byte store).
__global__ void gap_bwd_kernel(const float* __restrict__ gy, uint4* __restrict__ gx,
                               int64_t rows, int C) {
  const int64_t n = blockIdx.y;
  const float inv = 1.f / (float)rows;
  const int c8n = C / 8;
  const float* g = gy + n * C;
  for (int t = threadIdx.x; t < c8n; t += blockDim.x) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(g) + 2 * t);
    const float4 b = __ldg(reinterpret_cast<const float4*>(g) + 2 * t + 1);
    const uint4 o = make_uint4(tc_pack(a.x * inv, a.y * inv), tc_pack(a.z * inv, a.w * inv),
                               tc_pack(b.x * inv, b.y * inv), tc_pack(b.z * inv, b.w * inv));
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) gx[(n * rows + r) * c8n + t] = o;
  }
}

// fc_forward (kernels.cpp:525-540): y[n][j] = b[j] + sum_i w[j][i] x[n][i].
// One warp per output; lanes stride over i, fixed-order shuffle reduction.
__global__ void fc_fwd_kernel(const float* __restrict__ x, const float* __restrict__ w,
                              const float* __restrict__ b, float* __restrict__ y, int N, int Cin,
                              int Cout) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= N * Cout) return;
  const int n = warp / Cout, j = warp % Cout;
  float acc = 0.f;
  for (int i = lane; i < Cin; i += 32) acc += w[(int64_t)j * Cin + i] * x[(int64_t)n * Cin + i];
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) y[warp] = acc + b[j];
}

// fc_forward / fc_backward (kernels.cpp:525-576) as a small fp32 GEMM: C[m][n] = sum_k
// A(m, k) B(k, n) (+ bias[n]) with arbitrary element strides (transposes
// by stride), 64 x 64 tiles through shared memory, 4 x 4 outputs per
// thread, k summed in order (deterministic).  The one-thread-per-output
// kernels re-read the 8 MB weight / feature matrices from L2 per output and
// were latency-bound (23-55 us each at 64 clips).
struct SmallGemm {
  const float* a;
  const float* b;
  const float* bias;  // nullable, per n
  float* c;
  int M, N, K;
  int64_t a_m, a_k, b_k, b_n, c_m;  // element strides
};

template <int T>  // T x T tile, 16 x 16 threads of (T / 16)^2 outputs
__global__ void __launch_bounds__(256) small_gemm_kernel(SmallGemm g) {
  constexpr int R = T / 16;
  __shared__ float As[16][T + 4], Bs[16][T + 4];
  const int m0 = blockIdx.y * T, n0 = blockIdx.x * T;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  float acc[R][R] = {};
  for (int k0 = 0; k0 < g.K; k0 += 16) {
    for (int idx = threadIdx.x; idx < 16 * T; idx += 256) {
      // coalesce along whichever index is contiguous in memory
      int kk, mm;
      if (g.a_k == 1) {
        kk = idx & 15;
        mm = idx >> 4;
      } else {
        mm = idx % T;
        kk = idx / T;
      }
      const int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < g.M && k < g.K) ? __ldg(g.a + m * g.a_m + k * g.a_k) : 0.f;
      int kb, nn;
      if (g.b_n == 1) {
        nn = idx % T;
        kb = idx / T;
      } else {
        kb = idx & 15;
        nn = idx >> 4;
      }
      const int n = n0 + nn, kq = k0 + kb;
      Bs[kb][nn] = (n < g.N && kq < g.K) ? __ldg(g.b + kq * g.b_k + n * g.b_n) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float av[R], bv[R];
#pragma unroll
      for (int i = 0; i < R; ++i) {
        av[i] = As[kk][ty * R + i];
        bv[i] = Bs[kk][tx * R + i];
      }
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int j = 0; j < R; ++j) acc[i][j] += av[i] * bv[j];
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int m = m0 + ty * R + i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int n = n0 + tx * R + j;
      if (n < g.N) g.c[m * g.c_m + n] = acc[i][j] + (g.bias ? g.bias[n] : 0.f);
    }
  }
}

// db[j] = sum_n g[n][j] in n order.
__global__ void fc_bias_grad_kernel(const float* __restrict__ g, float* __restrict__ db, int N,
                                    int Cout) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= Cout) return;
  float a = 0.f;
  for (int n = 0; n < N; ++n) a += g[(int64_t)n * Cout + j];
  db[j] = a;
}

// loss = sum y^2 (net.cpp:141-146) and g = 2 y (net.cpp:180-181).
constexpr int kLossT = 1024;
__global__ void __launch_bounds__(kLossT) sq_loss_kernel(const float* __restrict__ y,
                                                         float* __restrict__ g,
                                                         float* __restrict__ loss, int n) {
  // one block, fixed-order tree (deterministic)
  __shared__ float part[kLossT];
  float acc = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const float v = __ldg(y + i);
    acc += v * v;
    g[i] = 2.f * v;
  }
  part[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kLossT / 2; s; s >>= 1) {
    if ((int)threadIdx.x < s) part[threadIdx.x] += part[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = part[0];
}

// Momentum SGD with decoupled-from-bias weight decay:
//   v = mu v + (g * grad_scale + wd_mask * wd * w);  w -= lr v
// hp (optional): {lr, mu, wd, grad_scale} read from device memory instead of
// the arguments (a captured CUDA graph replays with new hyperparameters).
__global__ void sgd_kernel(float* __restrict__ w, const float* __restrict__ g,
                           float* __restrict__ v, const uint8_t* __restrict__ decay, int64_t n,
                           float lr, float mu, float wd, float grad_scale,
                           const float* __restrict__ hp) {
  if (hp) {
    lr = hp[0];
    mu = hp[1];
    wd = hp[2];
    grad_scale = hp[3];
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float d = g[i] * grad_scale + (decay[i] ? wd * w[i] : 0.f);
    const float vn = mu * v[i] + d;
    v[i] = vn;
    w[i] -= lr * vn;
  }
}

// Rows per block of the bulk-staged pool kernels (0: the per-thread-load
// kernels).  Measured at the stem shape (tools/bench_pool.py): forward
// 289 us (per-thread loads) / 203 (R 1) / 222 (R 2) / 273 (R 3); backward
// 252 / 222 (2) / 218 (4) / 238 (8).  TSM_POOL_R / TSM_POOL_BR override the forward (1..3) and
// backward (2, 4, 8) values for A/B runs.
int pool_rows(int bwd) {
  static const int r[2] = {[] {
                             const char* e = getenv("TSM_POOL_R");
                             return e ? atoi(e) : 1;
                           }(),
                           [] {
                             const char* e = getenv("TSM_POOL_BR");
                             return e ? atoi(e) : 4;
                           }()};
  return r[bwd];
}

constexpr size_t kPoolSmemMax = 100 * 1024;

// the dynamic shared-memory opt-in, once per device
tsm_status pool_smem_attr(const void* fn) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  TSM_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (done.insert({fn, dev}).second)
    TSM_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)kPoolSmemMax));
  return TSM_OK;
}

}  // namespace

tsm_status maxpool_fwd(const void* x, void* y, uint8_t* arg, int64_t frames, int H, int W,
                       int C, cudaStream_t s) {
  if (C % 8) return fail(TSM_ERR_UNSUPPORTED, "maxpool: C % 8");
  const int Ho = (H + 2 - 3) / 2 + 1, Wo = (W + 2 - 3) / 2 + 1;
  const int R = pool_rows(0);
  const size_t smem = (size_t)(2 * R + 1) * W * C * 2;
  if (R > 0 && smem <= kPoolSmemMax) {
    auto kern = R == 1 ? maxpool_fwd_bulk_kernel<1>
                       : R == 3 ? maxpool_fwd_bulk_kernel<3> : maxpool_fwd_bulk_kernel<2>;
    TSM_TRY(pool_smem_attr(reinterpret_cast<const void*>(kern)));
    const int strips = (Ho + R - 1) / R;
    kern<<<(unsigned)(frames * strips), kT, smem, s>>>(
        static_cast<const uint4*>(x), static_cast<uint4*>(y), reinterpret_cast<uint2*>(arg), H,
        W, Ho, Wo, C / 8, strips);
  } else {
    maxpool_fwd_kernel<<<(unsigned)(frames * Ho), kT, 0, s>>>(
        static_cast<const uint4*>(x), static_cast<uint4*>(y), reinterpret_cast<uint2*>(arg), H,
        W, Ho, Wo, C / 8);
  }
  count_launches();
  return cuda_status(cudaGetLastError(), "maxpool_fwd");
}

tsm_status maxpool_bwd(const void* gy, const uint8_t* arg, void* gx, int64_t frames, int H,
                       int W, int C, cudaStream_t s) {
  if (C % 8) return fail(TSM_ERR_UNSUPPORTED, "maxpool: C % 8");
  const int Ho = (H + 2 - 3) / 2 + 1, Wo = (W + 2 - 3) / 2 + 1;
  const int R = pool_rows(1);
  const size_t bsmem = (size_t)(R + 1) * Wo * C * 3;  // gy bf16 + argmax bytes
  // (16-byte bulk sizes and offsets for the argmax rows: Wo * C / 8 even)
  if (H == 2 * Ho && W == 2 * Wo && R > 0 && bsmem <= kPoolSmemMax && (Wo * (C / 8)) % 2 == 0) {
    auto kern = R == 2 ? maxpool_bwd2x2_bulk_kernel<2>
                       : R == 8 ? maxpool_bwd2x2_bulk_kernel<8> : maxpool_bwd2x2_bulk_kernel<4>;
    TSM_TRY(pool_smem_attr(reinterpret_cast<const void*>(kern)));
    const int strips = (Ho + R - 1) / R;
    kern<<<(unsigned)(frames * strips), kT, bsmem, s>>>(
        static_cast<const uint4*>(gy), reinterpret_cast<const uint2*>(arg),
        static_cast<uint4*>(gx), Ho, Wo, C / 8, strips);
  } else if (H == 2 * Ho && W == 2 * Wo)
    maxpool_bwd2x2_kernel<<<(unsigned)(frames * Ho), kT, 0, s>>>(
        static_cast<const uint4*>(gy), reinterpret_cast<const uint2*>(arg),
        static_cast<uint4*>(gx), Ho, Wo, C / 8);
  else
    maxpool_bwd_kernel<<<(unsigned)(frames * H), kT, 0, s>>>(
        static_cast<const uint4*>(gy), reinterpret_cast<const uint2*>(arg),
        static_cast<uint4*>(gx), H, W, Ho, Wo, C / 8);
  count_launches();
  return cuda_status(cudaGetLastError(), "maxpool_bwd");
}

tsm_status gap_fwd(const void* x, float* y, int64_t clips, int64_t rows, int C, cudaStream_t s) {
  if (C % 8) return fail(TSM_ERR_UNSUPPORTED, "gap_fwd: C % 8");
  dim3 grid((unsigned)((C + 63) / 64), (unsigned)clips);
  gap_fwd_kernel<<<grid, 256, 0, s>>>(static_cast<const uint4*>(x), y, rows, C);
  count_launches();
  return cuda_status(cudaGetLastError(), "gap_fwd");
}

tsm_status gap_bwd(const float* gy, void* gx, int64_t clips, int64_t rows, int C,
                   cudaStream_t s) {
  if (C % 8) return fail(TSM_ERR_UNSUPPORTED, "gap_bwd: C % 8");
  const dim3 grid((unsigned)std::min<int64_t>(rows, 64), (unsigned)clips);
  gap_bwd_kernel<<<grid, kT, 0, s>>>(gy, static_cast<uint4*>(gx), rows, C);
  count_launches();
  return cuda_status(cudaGetLastError(), "gap_bwd");
}

// 64 x 64 tiles when they fill the machine, else 32 x 32 (fc dx: 64 x 2048)
static void small_gemm(const SmallGemm& g, cudaStream_t s) {
  const int64_t t64 = (int64_t)((g.N + 63) / 64) * ((g.M + 63) / 64);
  if (t64 >= 148)
    small_gemm_kernel<64><<<dim3((unsigned)((g.N + 63) / 64), (unsigned)((g.M + 63) / 64)), 256, 0,
                            s>>>(g);
  else
    small_gemm_kernel<32><<<dim3((unsigned)((g.N + 31) / 32), (unsigned)((g.M + 31) / 32)), 256, 0,
                            s>>>(g);
}

tsm_status fc_fwd(const float* x, const float* w, const float* b, float* y, int N, int Cin,
                  int Cout, cudaStream_t s) {
  // (K = 2048 is long for tiles of a 64 x 400 output: one warp per output)
  const int64_t threads = (int64_t)N * Cout * 32;
  fc_fwd_kernel<<<(unsigned)((threads + kT - 1) / kT), kT, 0, s>>>(x, w, b, y, N, Cin, Cout);
  count_launches();
  return cuda_status(cudaGetLastError(), "fc_fwd");
}

tsm_status sq_loss(const float* y, float* g, float* loss, int n, cudaStream_t s) {
  sq_loss_kernel<<<1, kLossT, 0, s>>>(y, g, loss, n);
  count_launches();
  return cuda_status(cudaGetLastError(), "sq_loss");
}

tsm_status fc_bwd(const float* g, const float* x, const float* w, float* dx, float* dw, float* db,
                  int N, int Cin, int Cout, cudaStream_t s) {
  // dx[n][c] = sum_j g[n][j] w[j][c];  dw[j][c] = sum_n g[n][j] x[n][c];  db[j] = sum_n g[n][j]
  small_gemm({g, w, nullptr, dx, N, Cin, Cout, Cout, 1, Cin, 1, Cin}, s);
  small_gemm({g, x, nullptr, dw, Cout, Cin, N, 1, Cout, Cin, 1, Cin}, s);
  fc_bias_grad_kernel<<<(unsigned)((Cout + 255) / 256), 256, 0, s>>>(g, db, N, Cout);
  count_launches(3);
  return cuda_status(cudaGetLastError(), "fc_bwd");
}

tsm_status sgd_update(float* w, const float* g, float* v, const uint8_t* decay, int64_t n,
                      float lr, float mu, float wd, float grad_scale, cudaStream_t s,
                      const float* hp) {
  sgd_kernel<<<blocks_for(n), kT, 0, s>>>(w, g, v, decay, n, lr, mu, wd, grad_scale, hp);
  count_launches();
  return cuda_status(cudaGetLastError(), "sgd_update");
}

}  // namespace tsm

// ---------------------------------------------------------------------------
// conv1 (the 7x7 / stride 2 / pad 3 stem, 3 -> 64 channels).  With only 3
// input channels an implicit-GEMM operand would be 6-byte rows, so the stem
// materialises its im2col matrix once per step straight from the reference
// NTCHW input: A[p][k], p = (frame, ho, wo), k = (r*7 + s)*3 + c for k < 147,
// zero for 147 <= k < 192.  The same matrix feeds the forward GEMM and the
// weight-gradient GEMM of the backward.
namespace tsm {
namespace {

// One block per (frame, output row ho): the 7 input rows x 3 channels the
// row's windows touch are staged in shared memory (coalesced reads, zero
// padding), then the Wo x 192 bf16 output rows — contiguous in memory — are
// written 16 bytes per thread, consecutive threads on consecutive chunks.
constexpr int kStemMaxW = 256;
constexpr int kStemThreads = 192;  // 24 K-chunks x 8 output columns

template <typename T>
__global__ void __launch_bounds__(kStemThreads)
    stem_im2col_kernel(const T* __restrict__ x, uint4* __restrict__ a, int H, int W, int Ho,
                       int Wo) {
  // One block per pair of output rows (frame, ho0..ho0+1): their windows
  // cover 9 input rows, staged channel-minor as [row][w + 3][c] (3 zero
  // columns each side).  For output row ho = ho0 + j the 21 K-values (s, c)
  // of filter row r are contiguous at ((2j + r) * PW + 2 wo) * 3, so K index
  // k = r * 21 + s * 3 + c reads flat[kbase(k) + 2j * 3 PW + 6 wo].  Each
  // thread owns one 16-byte K chunk (source offsets in registers) and walks
  // output columns; the kernel is issue-bound, so no per-element division.
  constexpr int K8 = kStemK / 8;         // 16-byte chunks per output row
  constexpr int PW = kStemMaxW + 6;      // padded input row
  constexpr int WS = kStemThreads / K8;  // output columns in flight per block
  constexpr int NR = 9;                  // staged input rows
  __shared__ float rows[NR * PW * 3];
  const int hp = (Ho + 1) / 2;
  const int ho0 = (blockIdx.x % hp) * 2;
  const int64_t f = blockIdx.x / hp;
  const T* xf = x + f * 3 * (int64_t)H * W;
  // staging: (row, channel) pairs outer, columns across threads (coalesced).
  // fp32 input goes through cp.async (every load in flight at once, zero
  // fill for the padding) — a load -> store loop would serialise ~27
  // global latencies per block.
  for (int rc = 0; rc < NR * 3; ++rc) {
    const int r = rc / 3, c = rc - 3 * (rc / 3);
    const int h = ho0 * 2 - 3 + r;
    const bool hin = h >= 0 && h < H;
    const T* src = xf + ((int64_t)c * H + (hin ? h : 0)) * W;
    float* dst = rows + r * PW * 3 + c;
    for (int wp = threadIdx.x; wp < PW; wp += kStemThreads) {
      const int w = wp - 3;
      const bool in = hin && w >= 0 && w < W;
      if constexpr (sizeof(T) == 4) {
        const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst + wp * 3));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(d),
                     "l"(src + (in ? w : 0)), "r"(in ? 4 : 0)
                     : "memory");
      } else {
        dst[wp * 3] = in ? (float)__ldg(src + w) : 0.f;
      }
    }
  }
  if constexpr (sizeof(T) == 4) asm volatile("cp.async.wait_all;" ::: "memory");
  const int chunk = threadIdx.x % K8, ws = threadIdx.x / K8;
  int src[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int k = chunk * 8 + e;
    src[e] = k < 147 ? (k / 21) * PW * 3 + (k % 21) : -1;
  }
  __syncthreads();
  if (ws >= WS) return;
#pragma unroll 1
  for (int j = 0; j < 2 && ho0 + j < Ho; ++j) {
    const float* fr = rows + j * 2 * PW * 3;
    uint4* out = a + ((int64_t)f * Ho + ho0 + j) * Wo * K8 + chunk;
    if (chunk < 18) {  // K chunks 0..17 hold k < 144: all 8 values real
#pragma unroll 2
      for (int wo = ws; wo < Wo; wo += WS) {
        const float* q = fr + 6 * wo;
        uint4 o;
        o.x = tc_pack(q[src[0]], q[src[1]]);
        o.y = tc_pack(q[src[2]], q[src[3]]);
        o.z = tc_pack(q[src[4]], q[src[5]]);
        o.w = tc_pack(q[src[6]], q[src[7]]);
        out[(int64_t)wo * K8] = o;
      }
    } else {
      for (int wo = ws; wo < Wo; wo += WS) {
        const float* q = fr + 6 * wo;
        float v[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = src[e] >= 0 ? q[src[e]] : 0.f;
        out[(int64_t)wo * K8] = make_uint4(tc_pack(v[0], v[1]), tc_pack(v[2], v[3]),
                                           tc_pack(v[4], v[5]), tc_pack(v[6], v[7]));
      }
    }
  }
}

// Space-to-depth stem input (even H, W): the 7x7 / stride-2 / pad-3 conv
// over x becomes a 4x4 / stride-1 conv (window offsets -2..+1) over
//   xs[f][h][w][(2p + q) * 4 + c] = x[f][c][2h + p][2w + q]   (c < 3, else 0)
// with W'[o][i][j][(2p + q) * 4 + c] = W[o][2i + p - 1][2j + q - 1][c]
// (zero outside the 7x7 window): input row 2(ho + i - 2) + p = 2ho + r - 3
// for r = 2i + p - 1.  16 channels = one 32-byte row per s2d pixel.
template <typename T>
__global__ void stem_s2d_kernel(const T* __restrict__ x, uint4* __restrict__ xs, int H, int W,
                                int npix) {
  const int H2 = H / 2, W2 = W / 2, hw2 = H2 * W2;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < npix; i += gridDim.x * blockDim.x) {
    const int f = i / hw2, rem = i - f * hw2;
    const int h = rem / W2, w = rem - h * W2;
    const T* xf = x + (int64_t)f * 3 * H * W;
    float v[16];
#pragma unroll
    for (int pq = 0; pq < 4; ++pq) {
      const int p = pq >> 1, q = pq & 1;
#pragma unroll
      for (int c = 0; c < 3; ++c) v[pq * 4 + c] = (float)__ldg(xf + ((int64_t)c * H + 2 * h + p) * W + 2 * w + q);
      // padding channels are 0, except channel 3 (group p = q = 0) = 1: its
      // conv weights are zero (forward unaffected) and its weight-gradient row
      // at the centre tap is the bias gradient sum(dY) (stem_s2d_wgrad)
      v[pq * 4 + 3] = pq == 0 ? 1.f : 0.f;
    }
    uint32_t o[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = tc_pack(v[2 * k], v[2 * k + 1]);
    xs[2 * (int64_t)i] = make_uint4(o[0], o[1], o[2], o[3]);
    xs[2 * (int64_t)i + 1] = make_uint4(o[4], o[5], o[6], o[7]);
  }
}

// The stem weight gradient folds the 4 horizontal taps into channels:
//   x4[f][h][w][j * 16 + c] = xs[f][h][w + j - 2][c]   (0 outside the row)
// so the remaining 4 vertical taps run on 64-channel (128-byte) pixels.
__global__ void stem_x4_kernel(const uint4* __restrict__ xs, uint4* __restrict__ x4, int W2) {
  // one block per (frame, row): the row's 16-channel pixels (+ 2 zero pixels
  // each side) staged in shared memory, then 64-channel output pixels
  // written as contiguous 16-byte chunks
  extern __shared__ uint4 row[];  // [(W2 + 4) * 2]
  const int64_t r = blockIdx.x;
  const uint4* src = xs + r * W2 * 2;
  for (int i = threadIdx.x; i < (W2 + 4) * 2; i += blockDim.x) {
    const int w = i / 2 - 2;
    row[i] = (w >= 0 && w < W2) ? __ldg(src + 2 * w + (i & 1)) : make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  uint4* dst = x4 + r * W2 * 8;
  for (int i = threadIdx.x; i < W2 * 8; i += blockDim.x) {
    const int w = i / 8, k = i % 8;           // chunk k = (j, half) of pixel w
    dst[i] = row[2 * (w + k / 2) + (k & 1)];  // xs pixel w + j - 2 (+2 border offset)
  }
}

// master [64][7][7][8] fp32 -> bf16 W' [64][4][4][16] (K = 256, see above)
__global__ void stem_weights_s2d_kernel(const float* __restrict__ w, __nv_bfloat16* __restrict__ wf) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 64 * 256) return;
  const int o = i / 256, k = i - o * 256;
  const int tap = k / 16, ch = k - tap * 16;
  const int ti = tap / 4, tj = tap - ti * 4, pq = ch / 4, c = ch - pq * 4;
  const int r = 2 * ti + (pq >> 1) - 1, sc = 2 * tj + (pq & 1) - 1;
  float v = 0.f;
  if (c < 3 && r >= 0 && r < 7 && sc >= 0 && sc < 7) v = w[(o * 49 + r * 7 + sc) * 8 + c];
  wf[i] = __float2bfloat16_rn(v);
}

// dW' [64][256] -> master-gradient layout [64][7][7][8]
__global__ void stem_wgrad_scatter_s2d_kernel(const float* __restrict__ g, float* __restrict__ gw) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 64 * 49 * 8) return;
  const int c = i % 8, rs = (i / 8) % 49, o = i / (49 * 8);
  const int r = rs / 7, sc = rs - r * 7;
  const int ti = (r + 1) >> 1, p = (r + 1) & 1, tj = (sc + 1) >> 1, q = (sc + 1) & 1;
  gw[i] = c < 3 ? g[o * 256 + (ti * 4 + tj) * 16 + (2 * p + q) * 4 + c] : 0.f;
}

// master [64][7][7][8] fp32 (GEMM layout, channels 3..7 zero) -> bf16 [64][192]
__global__ void stem_weights_kernel(const float* __restrict__ w, __nv_bfloat16* __restrict__ wf) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 64 * kStemK) return;
  const int o = i / kStemK, k = i - o * kStemK;
  float v = 0.f;
  if (k < 147) {
    const int tap = k / 3, c = k - tap * 3;
    v = w[(o * 49 + tap) * 8 + c];
  }
  wf[i] = __float2bfloat16_rn(v);
}

// dW [64][192] (GEMM order) -> master-gradient layout [64][7][7][8]
__global__ void stem_wgrad_scatter_kernel(const float* __restrict__ g, float* __restrict__ gw) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 64 * 49 * 8) return;
  const int c = i % 8, tap = (i / 8) % 49, o = i / (49 * 8);
  gw[i] = c < 3 ? g[o * kStemK + tap * 3 + c] : 0.f;
}

}  // namespace

tsm_status stem_im2col(const void* x, tsm_dtype dt, void* a, int64_t frames, int H, int W,
                       cudaStream_t s) {
  const int Ho = (H + 6 - 7) / 2 + 1, Wo = (W + 6 - 7) / 2 + 1;
  if (W > kStemMaxW) return fail(TSM_ERR_UNSUPPORTED, "stem: input width > 256");
  const unsigned grid = (unsigned)(frames * ((Ho + 1) / 2));  // two output rows per block
  auto* ao = static_cast<uint4*>(a);
  switch (dt) {
    case TSM_F32:
      stem_im2col_kernel<float><<<grid, kStemThreads, 0, s>>>(static_cast<const float*>(x), ao, H, W, Ho,
                                                     Wo);
      break;
    case TSM_F64:
      stem_im2col_kernel<double><<<grid, kStemThreads, 0, s>>>(static_cast<const double*>(x), ao, H, W,
                                                      Ho, Wo);
      break;
    default:
      return fail(TSM_ERR_UNSUPPORTED, "stem input dtype must be f32 or f64");
  }
  count_launches();
  return cuda_status(cudaGetLastError(), "stem_im2col");
}

tsm_status stem_weights(const float* w, void* wf, cudaStream_t s) {
  stem_weights_kernel<<<(64 * kStemK + kT - 1) / kT, kT, 0, s>>>(w,
                                                                 static_cast<__nv_bfloat16*>(wf));
  count_launches();
  return cuda_status(cudaGetLastError(), "stem_weights");
}

tsm_status stem_s2d(const void* x, tsm_dtype dt, void* xs, int64_t frames, int H, int W,
                    cudaStream_t s) {
  if (H % 2 || W % 2) return fail(TSM_ERR_UNSUPPORTED, "stem_s2d: even extents only");
  const int64_t npix = frames * (H / 2) * (W / 2);
  if (npix >= (1LL << 31)) return fail(TSM_ERR_UNSUPPORTED, "stem_s2d: too many pixels");
  const unsigned grid = (unsigned)std::min<int64_t>((npix + kT - 1) / kT, 148 * 16);
  auto* o = static_cast<uint4*>(xs);
  switch (dt) {
    case TSM_F32:
      stem_s2d_kernel<float><<<grid, kT, 0, s>>>(static_cast<const float*>(x), o, H, W, (int)npix);
      break;
    case TSM_F64:
      stem_s2d_kernel<double><<<grid, kT, 0, s>>>(static_cast<const double*>(x), o, H, W, (int)npix);
      break;
    default:
      return fail(TSM_ERR_UNSUPPORTED, "stem input dtype must be f32 or f64");
  }
  count_launches();
  return cuda_status(cudaGetLastError(), "stem_s2d");
}

tsm_status stem_x4(const void* xs, void* x4, int64_t frames, int64_t H2, int64_t W2,
                   cudaStream_t s) {
  stem_x4_kernel<<<(unsigned)(frames * H2), kT, (size_t)(W2 + 4) * 32, s>>>(
      static_cast<const uint4*>(xs), static_cast<uint4*>(x4), (int)W2);
  count_launches();
  return cuda_status(cudaGetLastError(), "stem_x4");
}

tsm_status stem_weights_s2d(const float* w, void* wf, cudaStream_t s) {
  stem_weights_s2d_kernel<<<(64 * 256 + kT - 1) / kT, kT, 0, s>>>(w, static_cast<__nv_bfloat16*>(wf));
  count_launches();
  return cuda_status(cudaGetLastError(), "stem_weights_s2d");
}

tsm_status stem_wgrad_scatter_s2d(const float* g, float* gw, cudaStream_t s) {
  stem_wgrad_scatter_s2d_kernel<<<(64 * 49 * 8 + kT - 1) / kT, kT, 0, s>>>(g, gw);
  count_launches();
  return cuda_status(cudaGetLastError(), "stem_wgrad_scatter_s2d");
}

tsm_status stem_wgrad_scatter(const float* g, float* gw, cudaStream_t s) {
  stem_wgrad_scatter_kernel<<<(64 * 49 * 8 + kT - 1) / kT, kT, 0, s>>>(g, gw);
  count_launches();
  return cuda_status(cudaGetLastError(), "stem_wgrad_scatter");
}

// Input gradient of the 7x7 / stride 2 / pad 3 stem conv (conv_backward's
// grad_x gather, kernels.cpp:246-280, for the network's first layer):
//   gx[f][c][h][w] = sum_{o, kh, kw} gy[f][ho][wo][o] * W[o][kh][kw][c],
//   h = 2 ho - 3 + kh,  w = 2 wo - 3 + kw,
// gy NTHWC bf16 [frames][Ho][Wo][64], W fp32 [64][7][7][8] (c < 3 used), gx
// NTCHW (the reference layout of Gradients::input, net.hpp:36-40) in f32 or
// f64.  Only the drop-in executor asks for it (the training step does not
// need dL/dx).  One thread per input pixel; the weights sit in shared memory
// as [tap][c][o] so a warp's lanes read the same words.
template <typename T>
__global__ void stem_dgrad_kernel(const __nv_bfloat16* __restrict__ gy, const float* __restrict__ w,
                                  T* __restrict__ gx, int H, int W, int Ho, int Wo,
                                  int64_t npix) {
  __shared__ float ws[49 * 3 * 64];
  for (int i = threadIdx.x; i < 49 * 3 * 64; i += blockDim.x) {
    const int o = i % 64, c = (i / 64) % 3, tap = i / 192;
    ws[i] = w[(o * 49 + tap) * 8 + c];
  }
  __syncthreads();
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npix;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t f = p / ((int64_t)H * W);
    const int rem = (int)(p - f * H * W), h = rem / W, x = rem - h * W;
    float acc[3] = {0.f, 0.f, 0.f};
    for (int kh = (h + 3) & 1; kh < 7; kh += 2) {
      const int ho = (h + 3 - kh) >> 1;
      if (ho < 0 || ho >= Ho) continue;
      for (int kw = (x + 3) & 1; kw < 7; kw += 2) {
        const int wo = (x + 3 - kw) >> 1;
        if (wo < 0 || wo >= Wo) continue;
        const uint4* g = reinterpret_cast<const uint4*>(gy + ((f * Ho + ho) * Wo + wo) * 64);
        const float* wt = ws + (kh * 7 + kw) * 192;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint4 v = __ldg(g + q);
          const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float gv = __bfloat162float(e[j]);
#pragma unroll
            for (int c = 0; c < 3; ++c) acc[c] += gv * wt[c * 64 + q * 8 + j];
          }
        }
      }
    }
    T* out = gx + f * 3 * H * W + rem;
#pragma unroll
    for (int c = 0; c < 3; ++c) out[(int64_t)c * H * W] = (T)acc[c];
  }
}

tsm_status stem_dgrad(const void* gy, const float* w, void* gx, tsm_dtype dt, int64_t frames,
                      int H, int W, int Ho, int Wo, cudaStream_t s) {
  const int64_t npix = frames * H * W;
  const unsigned grid = (unsigned)std::min<int64_t>((npix + kT - 1) / kT, 148 * 8);
  const auto* g = static_cast<const __nv_bfloat16*>(gy);
  switch (dt) {
    case TSM_F32:
      stem_dgrad_kernel<float><<<grid, kT, 0, s>>>(g, w, static_cast<float*>(gx), H, W, Ho, Wo, npix);
      break;
    case TSM_F64:
      stem_dgrad_kernel<double><<<grid, kT, 0, s>>>(g, w, static_cast<double*>(gx), H, W, Ho, Wo,
                                                    npix);
      break;
    default:
      return fail(TSM_ERR_UNSUPPORTED, "stem input gradient dtype must be f32 or f64");
  }
  count_launches();
  return cuda_status(cudaGetLastError(), "stem_dgrad");
}

}  // namespace tsm
