// Non-GEMM layers of TSM-ResNet-50 (build_tsm8f, arch.cpp:140-161) and the
// optimizer: 3x3/s2 max pool with the reference's first-max tie rule, global
// average pool, the 2048->classes fully-connected head, the Sigma-y^2 loss
// and momentum SGD.  All gather-form / fixed-order, no float atomics.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "common.cuh"
#include "head_kernels.cuh"

namespace tsm {
namespace {

constexpr int kT = 256;

inline unsigned blocks_for(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + kT - 1) / kT, 148 * 32));
}

// max_pool_forward (kernels.cpp:353-390) for the spatial 1x3x3 / stride 2 /
// pad 1 window on NTHWC bf16: padded taps never win; ties keep the first
// element in (h, w) scan order (strict >).  Records the winning tap (0..8).
// One thread = 8 channels (16-byte loads) of one output pixel.
__global__ void maxpool_fwd_kernel(const uint4* __restrict__ x, uint4* __restrict__ y,
                                   uint2* __restrict__ arg, int64_t frames, int H, int W, int Ho,
                                   int Wo, int C8) {
  const int64_t total = frames * Ho * Wo * C8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C8);
    int64_t r = i / C8;
    const int wo = (int)(r % Wo);
    r /= Wo;
    const int ho = (int)(r % Ho);
    const int64_t f = r / Ho;
    float best[8];
    uint8_t barg[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      best[k] = 0.f;
      barg[k] = 0xff;
    }
    for (int dh = 0; dh < 3; ++dh) {
      const int h = ho * 2 - 1 + dh;
      if (h < 0 || h >= H) continue;
      for (int dw = 0; dw < 3; ++dw) {
        const int w = wo * 2 - 1 + dw;
        if (w < 0 || w >= W) continue;
        const uint4 v = x[((f * H + h) * W + w) * C8 + c];
        const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float e = __bfloat162float(vb[k]);
          if (barg[k] == 0xff || e > best[k]) {
            best[k] = e;
            barg[k] = (uint8_t)(dh * 3 + dw);
          }
        }
      }
    }
    uint4 o;
    __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(&o);
#pragma unroll
    for (int k = 0; k < 8; ++k) ob[k] = __float2bfloat16_rn(best[k]);
    y[i] = o;
    arg[i] = *reinterpret_cast<const uint2*>(barg);
  }
}

// max_pool_backward (kernels.cpp:392-455): each input element gathers the
// gradients of the (at most 2x2) windows whose recorded argmax it is.
__global__ void maxpool_bwd_kernel(const uint4* __restrict__ gy, const uint2* __restrict__ arg,
                                   uint4* __restrict__ gx, int64_t frames, int H, int W, int Ho,
                                   int Wo, int C8) {
  const int64_t total = frames * H * W * C8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C8);
    int64_t r = i / C8;
    const int w = (int)(r % W);
    r /= W;
    const int h = (int)(r % H);
    const int64_t f = r / H;
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    // windows ho with 2ho-1 <= h <= 2ho+1, in ascending (ho, wo) order
    const int ho0 = max(0, h / 2), ho1 = min(Ho - 1, (h + 1) / 2);
    const int wo0 = max(0, w / 2), wo1 = min(Wo - 1, (w + 1) / 2);
    for (int ho = ho0; ho <= ho1; ++ho) {
      const int dh = h - (ho * 2 - 1);
      if (dh < 0 || dh > 2) continue;
      for (int wo = wo0; wo <= wo1; ++wo) {
        const int dw = w - (wo * 2 - 1);
        if (dw < 0 || dw > 2) continue;
        const int64_t o = ((f * Ho + ho) * Wo + wo) * C8 + c;
        const uint2 a = arg[o];
        const uint8_t* ab = reinterpret_cast<const uint8_t*>(&a);
        const uint4 g = gy[o];
        const __nv_bfloat16* gb = reinterpret_cast<const __nv_bfloat16*>(&g);
        const uint8_t tap = (uint8_t)(dh * 3 + dw);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (ab[k] == tap) acc[k] += __bfloat162float(gb[k]);
      }
    }
    uint4 o;
    __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(&o);
#pragma unroll
    for (int k = 0; k < 8; ++k) ob[k] = __float2bfloat16_rn(acc[k]);
    gx[i] = o;
  }
}

// global_avg_pool_forward (kernels.cpp:457-478): mean over (t, h, w) per
// (clip, channel).  x: [clips][rows][C] bf16 -> y: [clips][C] fp32.
__global__ void gap_fwd_kernel(const __nv_bfloat16* __restrict__ x, float* __restrict__ y,
                               int64_t rows, int C) {
  const int64_t n = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= C) return;
  const __nv_bfloat16* xn = x + n * rows * C;
  float acc = 0.f;
  for (int64_t r = 0; r < rows; ++r) acc += __bfloat162float(xn[r * C + c]);
  y[n * C + c] = acc / (float)rows;
}

// global_avg_pool_backward (kernels.cpp:480-501), writing bf16 NTHWC.
__global__ void gap_bwd_kernel(const float* __restrict__ gy, __nv_bfloat16* __restrict__ gx,
                               int64_t clips, int64_t rows, int C) {
  const int64_t total = clips * rows * C;
  const float inv = 1.f / (float)rows;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i % C);
    const int64_t n = i / (rows * C);
    gx[i] = __float2bfloat16_rn(gy[n * C + c] * inv);
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

// loss = sum y^2 (net.cpp:141-146) and g = 2 y (net.cpp:180-181).
__global__ void sq_loss_kernel(const float* __restrict__ y, float* __restrict__ g,
                               float* __restrict__ loss, int n) {
  __shared__ float part[kT];
  float acc = 0.f;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    acc += y[i] * y[i];
    g[i] = 2.f * y[i];
  }
  part[threadIdx.x] = acc;
  __syncthreads();
  for (int s = kT / 2; s; s >>= 1) {
    if ((int)threadIdx.x < s) part[threadIdx.x] += part[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) *loss = part[0];
}

// fc_backward (kernels.cpp:542-576).
__global__ void fc_bwd_dx_kernel(const float* __restrict__ g, const float* __restrict__ w,
                                 float* __restrict__ dx, int N, int Cin, int Cout) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)N * Cin) return;
  const int n = (int)(i / Cin), c = (int)(i % Cin);
  float acc = 0.f;
  for (int j = 0; j < Cout; ++j) acc += g[(int64_t)n * Cout + j] * w[(int64_t)j * Cin + c];
  dx[i] = acc;
}

__global__ void fc_bwd_dw_kernel(const float* __restrict__ g, const float* __restrict__ x,
                                 float* __restrict__ dw, float* __restrict__ db, int N, int Cin,
                                 int Cout) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= (int64_t)Cout * Cin) return;
  const int j = (int)(i / Cin), c = (int)(i % Cin);
  float acc = 0.f;
  for (int n = 0; n < N; ++n) acc += g[(int64_t)n * Cout + j] * x[(int64_t)n * Cin + c];
  dw[i] = acc;
  if (c == 0) {
    float a = 0.f;
    for (int n = 0; n < N; ++n) a += g[(int64_t)n * Cout + j];
    db[j] = a;
  }
}

// Momentum SGD with decoupled-from-bias weight decay:
//   v = mu v + (g * grad_scale + wd_mask * wd * w);  w -= lr v
__global__ void sgd_kernel(float* __restrict__ w, const float* __restrict__ g,
                           float* __restrict__ v, const uint8_t* __restrict__ decay, int64_t n,
                           float lr, float mu, float wd, float grad_scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float d = g[i] * grad_scale + (decay[i] ? wd * w[i] : 0.f);
    const float vn = mu * v[i] + d;
    v[i] = vn;
    w[i] -= lr * vn;
  }
}

}  // namespace

tsm_status maxpool_fwd(const void* x, void* y, uint8_t* arg, int64_t frames, int H, int W,
                       int C, cudaStream_t s) {
  if (C % 8) return fail(TSM_ERR_UNSUPPORTED, "maxpool: C % 8");
  const int Ho = (H + 2 - 3) / 2 + 1, Wo = (W + 2 - 3) / 2 + 1;
  maxpool_fwd_kernel<<<blocks_for(frames * Ho * Wo * (C / 8)), kT, 0, s>>>(
      static_cast<const uint4*>(x), static_cast<uint4*>(y), reinterpret_cast<uint2*>(arg), frames,
      H, W, Ho, Wo, C / 8);
  count_launches();
  return cuda_status(cudaGetLastError(), "maxpool_fwd");
}

tsm_status maxpool_bwd(const void* gy, const uint8_t* arg, void* gx, int64_t frames, int H,
                       int W, int C, cudaStream_t s) {
  if (C % 8) return fail(TSM_ERR_UNSUPPORTED, "maxpool: C % 8");
  const int Ho = (H + 2 - 3) / 2 + 1, Wo = (W + 2 - 3) / 2 + 1;
  maxpool_bwd_kernel<<<blocks_for(frames * H * W * (C / 8)), kT, 0, s>>>(
      static_cast<const uint4*>(gy), reinterpret_cast<const uint2*>(arg),
      static_cast<uint4*>(gx), frames, H, W, Ho, Wo, C / 8);
  count_launches();
  return cuda_status(cudaGetLastError(), "maxpool_bwd");
}

tsm_status gap_fwd(const void* x, float* y, int64_t clips, int64_t rows, int C, cudaStream_t s) {
  dim3 grid((unsigned)((C + 127) / 128), (unsigned)clips);
  gap_fwd_kernel<<<grid, 128, 0, s>>>(static_cast<const __nv_bfloat16*>(x), y, rows, C);
  count_launches();
  return cuda_status(cudaGetLastError(), "gap_fwd");
}

tsm_status gap_bwd(const float* gy, void* gx, int64_t clips, int64_t rows, int C,
                   cudaStream_t s) {
  gap_bwd_kernel<<<blocks_for(clips * rows * C), kT, 0, s>>>(
      gy, static_cast<__nv_bfloat16*>(gx), clips, rows, C);
  count_launches();
  return cuda_status(cudaGetLastError(), "gap_bwd");
}

tsm_status fc_fwd(const float* x, const float* w, const float* b, float* y, int N, int Cin,
                  int Cout, cudaStream_t s) {
  const int64_t threads = (int64_t)N * Cout * 32;
  fc_fwd_kernel<<<(unsigned)((threads + kT - 1) / kT), kT, 0, s>>>(x, w, b, y, N, Cin, Cout);
  count_launches();
  return cuda_status(cudaGetLastError(), "fc_fwd");
}

tsm_status sq_loss(const float* y, float* g, float* loss, int n, cudaStream_t s) {
  sq_loss_kernel<<<1, kT, 0, s>>>(y, g, loss, n);
  count_launches();
  return cuda_status(cudaGetLastError(), "sq_loss");
}

tsm_status fc_bwd(const float* g, const float* x, const float* w, float* dx, float* dw, float* db,
                  int N, int Cin, int Cout, cudaStream_t s) {
  fc_bwd_dx_kernel<<<(unsigned)(((int64_t)N * Cin + kT - 1) / kT), kT, 0, s>>>(g, w, dx, N, Cin,
                                                                             Cout);
  fc_bwd_dw_kernel<<<(unsigned)(((int64_t)Cout * Cin + kT - 1) / kT), kT, 0, s>>>(g, x, dw, db, N,
                                                                                Cin, Cout);
  count_launches(2);
  return cuda_status(cudaGetLastError(), "fc_bwd");
}

tsm_status sgd_update(float* w, const float* g, float* v, const uint8_t* decay, int64_t n,
                      float lr, float mu, float wd, float grad_scale, cudaStream_t s) {
  sgd_kernel<<<blocks_for(n), kT, 0, s>>>(w, g, v, decay, n, lr, mu, wd, grad_scale);
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
template <typename T>
__global__ void __launch_bounds__(256)
    stem_im2col_kernel(const T* __restrict__ x, uint4* __restrict__ a, int H, int W, int Ho,
                       int Wo) {
  constexpr int K8 = kStemK / 8;    // 16-byte chunks per output row
  constexpr int PW = kStemMaxW + 6;  // padded input row (3 zero columns each side)
  __shared__ float rows[7][3][PW];
  __shared__ int kofs[kStemK];  // k -> offset of (r, c, s) in `rows`, -1 = padding
  const int ho = blockIdx.x % Ho;
  const int64_t f = blockIdx.x / Ho;
  const T* xf = x + f * 3 * (int64_t)H * W;
  for (int k = threadIdx.x; k < kStemK; k += blockDim.x) {
    int o = -1;
    if (k < 147) {
      const int tap = k / 3, c = k - tap * 3;
      const int rr = tap / 7, ss = tap - rr * 7;
      o = (rr * 3 + c) * PW + ss;
    }
    kofs[k] = o;
  }
  for (int i = threadIdx.x; i < 7 * 3 * PW; i += blockDim.x) {
    const int wp = i % PW, c = (i / PW) % 3, r = i / (3 * PW);
    const int h = ho * 2 - 3 + r, w = wp - 3;
    float v = 0.f;
    if (h >= 0 && h < H && w >= 0 && w < W) v = (float)xf[((int64_t)c * H + h) * W + w];
    rows[r][c][wp] = v;
  }
  __syncthreads();
  const float* flat = &rows[0][0][0];
  uint4* out = a + ((int64_t)f * Ho + ho) * Wo * K8;
  for (int i = threadIdx.x; i < Wo * K8; i += blockDim.x) {
    const int wo = i / K8, chunk = i - wo * K8;
    uint4 o;
    uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      const int k0 = kofs[chunk * 8 + e], k1 = kofs[chunk * 8 + e + 1];
      // input column 2wo - 3 + s sits at padded index 2wo + s
      const float v0 = k0 >= 0 ? flat[k0 + wo * 2] : 0.f;
      const float v1 = k1 >= 0 ? flat[k1 + wo * 2] : 0.f;
      __nv_bfloat162 b = __floats2bfloat162_rn(v0, v1);
      ow[e / 2] = *reinterpret_cast<uint32_t*>(&b);
    }
    out[i] = o;
  }
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
  const unsigned grid = (unsigned)(frames * Ho);
  auto* ao = static_cast<uint4*>(a);
  switch (dt) {
    case TSM_F32:
      stem_im2col_kernel<float><<<grid, 256, 0, s>>>(static_cast<const float*>(x), ao, H, W, Ho,
                                                     Wo);
      break;
    case TSM_F64:
      stem_im2col_kernel<double><<<grid, 256, 0, s>>>(static_cast<const double*>(x), ao, H, W,
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

tsm_status stem_wgrad_scatter(const float* g, float* gw, cudaStream_t s) {
  stem_wgrad_scatter_kernel<<<(64 * 49 * 8 + kT - 1) / kT, kT, 0, s>>>(g, gw);
  count_launches();
  return cuda_status(cudaGetLastError(), "stem_wgrad_scatter");
}

}  // namespace tsm
