// Direct (CUDA-core) convolutions for bottleneck units whose channel counts
// do not fit the tcgen05 tiles (channels not multiples of 64), e.g. the
// reference's micro-tsm preset (arch.cpp:220-233: 8 -> 16 channels, width 4).
// A correctness path for small test networks, still entirely on the GPU.
//
// NTHWC bf16 activations, fp32 master weights [c_out][k][k][c_in], fp32
// accumulation in the reference's orders:
//   forward  bias first, then ci, dh, dw ascending   (kernels.cpp:171-200)
//   grad_x   gather over (co, dh, dw)                 (kernels.cpp:246-280)
//   grad_w   per (co, ci, dh, dw) over (n, t, h, w)   (kernels.cpp:282-310)
//   grad_b   over (n, t, h, w)                        (kernels.cpp:312-325)
// The temporal shift before conv1 (channels [0,F) read t-1, [F,F+B) read
// t+1, +0.0 outside the clip, kernels.cpp:97-125) is applied in the operand
// gathers; its adjoint (kernels.cpp:127-157) in the input-gradient gather.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "generic_conv.h"
#include "tc_common.cuh"

namespace tsm {
namespace {

constexpr int kT = 256;

inline unsigned blocks_for(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + kT - 1) / kT, 148 * 64));
}

struct G {
  int T, H, W, Ho, Wo, Ci, Co, k, s, p, F, B;
  int64_t frames;
};

// frame offset of channel ci in the shifted operand (forward direction)
__device__ __forceinline__ int shift_dt(const G& g, int ci) {
  return ci < g.F ? -1 : (ci < g.F + g.B ? 1 : 0);
}

__global__ void gconv_fwd_kernel(const __nv_bfloat16* __restrict__ x, const float* __restrict__ w,
                                 const float* __restrict__ bias,
                                 const __nv_bfloat16* __restrict__ res,
                                 __nv_bfloat16* __restrict__ y, int relu, G g) {
  const int64_t total = g.frames * g.Ho * g.Wo * g.Co;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int co = (int)(i % g.Co);
    int64_t r = i / g.Co;
    const int wo = (int)(r % g.Wo);
    r /= g.Wo;
    const int ho = (int)(r % g.Ho);
    const int64_t f = r / g.Ho;
    const int t = (int)(f % g.T);
    const int64_t n0 = f - t;  // first frame of the clip
    float acc = bias ? bias[co] : 0.f;
    for (int ci = 0; ci < g.Ci; ++ci) {
      const int tt = t + shift_dt(g, ci);
      if (tt < 0 || tt >= g.T) continue;
      for (int dh = 0; dh < g.k; ++dh) {
        const int h = ho * g.s + dh - g.p;
        if (h < 0 || h >= g.H) continue;
        for (int dw = 0; dw < g.k; ++dw) {
          const int ww = wo * g.s + dw - g.p;
          if (ww < 0 || ww >= g.W) continue;
          acc += __bfloat162float(x[(((n0 + tt) * g.H + h) * g.W + ww) * g.Ci + ci]) *
                 w[((int64_t)(co * g.k + dh) * g.k + dw) * g.Ci + ci];
        }
      }
    }
    if (res) acc += __bfloat162float(res[i]);
    if (relu) acc = fmaxf(acc, 0.f);
    y[i] = __float2bfloat16_rn(acc);
  }
}

__global__ void gconv_dgrad_kernel(const __nv_bfloat16* __restrict__ dy,
                                   const float* __restrict__ w,
                                   const __nv_bfloat16* __restrict__ res,
                                   const __nv_bfloat16* __restrict__ mask,
                                   const uint32_t* __restrict__ mbits,
                                   __nv_bfloat16* __restrict__ dx, G g) {
  const int64_t total = g.frames * g.H * g.W * g.Ci;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int ci = (int)(i % g.Ci);
    int64_t r = i / g.Ci;
    const int wi = (int)(r % g.W);
    r /= g.W;
    const int hi = (int)(r % g.H);
    const int64_t f = r / g.H;
    const int t = (int)(f % g.T);
    const int64_t n0 = f - t;
    // adjoint shift: x[t] fed the shifted operand at frame t - dt
    const int ts = t - shift_dt(g, ci);
    float acc = 0.f;
    if (ts >= 0 && ts < g.T) {
      for (int co = 0; co < g.Co; ++co)
        for (int dh = 0; dh < g.k; ++dh) {
          const int hn = hi + g.p - dh;
          if (hn < 0 || hn % g.s) continue;
          const int ho = hn / g.s;
          if (ho >= g.Ho) continue;
          for (int dw = 0; dw < g.k; ++dw) {
            const int wn = wi + g.p - dw;
            if (wn < 0 || wn % g.s) continue;
            const int wo = wn / g.s;
            if (wo >= g.Wo) continue;
            acc += __bfloat162float(dy[(((n0 + ts) * g.Ho + ho) * g.Wo + wo) * g.Co + co]) *
                   w[((int64_t)(co * g.k + dh) * g.k + dw) * g.Ci + ci];
          }
        }
    }
    if (res) acc += __bfloat162float(res[i]);
    if (mask && !(__bfloat162float(mask[i]) > 0.f)) acc = 0.f;
    if (mbits && !tc::bit_of(mbits[i / 32], (int)(i % 32))) acc = 0.f;
    dx[i] = __float2bfloat16_rn(acc);
  }
}

// one thread per weight element; db by the threads with (dh, dw, ci) = 0
__global__ void gconv_wgrad_kernel(const __nv_bfloat16* __restrict__ x,
                                   const __nv_bfloat16* __restrict__ dy, float* __restrict__ dw,
                                   float* __restrict__ db, G g) {
  const int64_t total = (int64_t)g.Co * g.k * g.k * g.Ci;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int ci = (int)(i % g.Ci);
    int64_t r = i / g.Ci;
    const int kw = (int)(r % g.k);
    r /= g.k;
    const int kh = (int)(r % g.k);
    const int co = (int)(r / g.k);
    const int dt = shift_dt(g, ci);
    float acc = 0.f, accb = 0.f;
    const bool do_b = db && kh == 0 && kw == 0 && ci == 0;
    for (int64_t f = 0; f < g.frames; ++f) {
      const int t = (int)(f % g.T);
      const int tt = t + dt;
      const bool tin = tt >= 0 && tt < g.T;
      for (int ho = 0; ho < g.Ho; ++ho) {
        const int h = ho * g.s + kh - g.p;
        for (int wo = 0; wo < g.Wo; ++wo) {
          const float d = __bfloat162float(dy[((f * g.Ho + ho) * g.Wo + wo) * g.Co + co]);
          if (do_b) accb += d;
          const int ww = wo * g.s + kw - g.p;
          if (!tin || h < 0 || h >= g.H || ww < 0 || ww >= g.W) continue;
          acc += d * __bfloat162float(x[(((f - t + tt) * g.H + h) * g.W + ww) * g.Ci + ci]);
        }
      }
    }
    dw[i] = acc;
    if (do_b) db[co] = accb;
  }
}

G make_g(const ConvShape& s) {
  G g{};
  g.T = (int)s.T;
  g.H = (int)s.H;
  g.W = (int)s.W;
  g.Ho = (int)s.h_out();
  g.Wo = (int)s.w_out();
  g.Ci = (int)s.c_in;
  g.Co = (int)s.c_out;
  g.k = s.k;
  g.s = s.stride;
  g.p = s.k / 2;
  g.F = (int)s.F;
  g.B = (int)s.B;
  g.frames = s.clips * s.T;
  return g;
}

}  // namespace

tsm_status gconv_fwd(const ConvShape& s, const void* x, const float* w, const float* bias,
                     const void* residual, void* y, int relu, cudaStream_t st) {
  const G g = make_g(s);
  gconv_fwd_kernel<<<blocks_for(g.frames * g.Ho * g.Wo * g.Co), kT, 0, st>>>(
      static_cast<const __nv_bfloat16*>(x), w, bias, static_cast<const __nv_bfloat16*>(residual),
      static_cast<__nv_bfloat16*>(y), relu, g);
  count_launches();
  return cuda_status(cudaGetLastError(), "gconv_fwd");
}

tsm_status gconv_dgrad(const ConvShape& s, const void* dy, const float* w, const void* residual,
                       const void* mask, const uint32_t* mask_bits, void* dx, cudaStream_t st) {
  const G g = make_g(s);
  if (mask_bits && s.c_in % 32)
    return fail(TSM_ERR_UNSUPPORTED, "gconv_dgrad: bitmask needs c_in % 32");
  gconv_dgrad_kernel<<<blocks_for(g.frames * g.H * g.W * g.Ci), kT, 0, st>>>(
      static_cast<const __nv_bfloat16*>(dy), w, static_cast<const __nv_bfloat16*>(residual),
      static_cast<const __nv_bfloat16*>(mask), mask_bits, static_cast<__nv_bfloat16*>(dx), g);
  count_launches();
  return cuda_status(cudaGetLastError(), "gconv_dgrad");
}

tsm_status gconv_wgrad(const ConvShape& s, const void* x, const void* dy, float* dw, float* db,
                       cudaStream_t st) {
  const G g = make_g(s);
  gconv_wgrad_kernel<<<blocks_for((int64_t)g.Co * g.k * g.k * g.Ci), kT, 0, st>>>(
      static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(dy), dw, db, g);
  count_launches();
  return cuda_status(cudaGetLastError(), "gconv_wgrad");
}

}  // namespace tsm
