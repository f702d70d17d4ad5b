// Stem pool, head and optimizer kernels (see head_kernels.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "tsm_b200.h"

namespace tsm {

// 1x3x3 / stride 2 / pad 1 spatial max pool on NTHWC bf16 (+ argmax taps).
tsm_status maxpool_fwd(const void* x, void* y, uint8_t* arg, int64_t frames, int H, int W, int C,
                       cudaStream_t s);
tsm_status maxpool_bwd(const void* gy, const uint8_t* arg, void* gx, int64_t frames, int H, int W,
                       int C, cudaStream_t s);
// global average pool over all `rows` (T*H*W) of each clip: bf16 -> fp32 [clips][C]
tsm_status gap_fwd(const void* x, float* y, int64_t clips, int64_t rows, int C, cudaStream_t s);
tsm_status gap_bwd(const float* gy, void* gx, int64_t clips, int64_t rows, int C, cudaStream_t s);
tsm_status fc_fwd(const float* x, const float* w, const float* b, float* y, int N, int Cin,
                  int Cout, cudaStream_t s);
tsm_status fc_bwd(const float* g, const float* x, const float* w, float* dx, float* dw, float* db,
                  int N, int Cin, int Cout, cudaStream_t s);
tsm_status sq_loss(const float* y, float* g, float* loss, int n, cudaStream_t s);
// conv1 stem: im2col matrix [frames*Ho*Wo][kStemK] bf16 from NTCHW f32/f64
// input (K = 7*7*3 = 147 zero-padded to 192), bf16 weights [64][192], and
// the scatter of the GEMM-order weight gradient back to [64][7][7][8].
constexpr int kStemK = 192;
tsm_status stem_im2col(const void* x, tsm_dtype dt, void* a, int64_t frames, int H, int W,
                       cudaStream_t s);
tsm_status stem_weights(const float* w, void* wf, cudaStream_t s);
// Space-to-depth stem (even H, W): x NTCHW f32/f64 -> xs [frames][H/2][W/2][16]
// bf16, making the 7x7/s2 stem a 4x4/s1 conv (K = 256) with weights W'
// [64][4][4][16]; stem_wgrad_scatter_s2d maps dW' back to the master layout.
tsm_status stem_s2d(const void* x, tsm_dtype dt, void* xs, int64_t frames, int H, int W,
                    cudaStream_t s);
tsm_status stem_weights_s2d(const float* w, void* wf, cudaStream_t s);
// x4[f][h][w][j*16 + c] = xs[f][h][w + j - 2][c] (horizontal taps folded into channels)
tsm_status stem_x4(const void* xs, void* x4, int64_t frames, int64_t H2, int64_t W2,
                   cudaStream_t s);
tsm_status stem_wgrad_scatter_s2d(const float* g, float* gw, cudaStream_t s);
tsm_status stem_wgrad_scatter(const float* g, float* gw, cudaStream_t s);
// dL/dx of the 7x7/s2/pad-3 stem: gy NTHWC bf16 [frames][Ho][Wo][64], w fp32
// [64][7][7][8] -> gx NTCHW [frames][3][H][W] (f32 / f64).
tsm_status stem_dgrad(const void* gy, const float* w, void* gx, tsm_dtype dt, int64_t frames,
                      int H, int W, int Ho, int Wo, cudaStream_t s);
tsm_status sgd_update(float* w, const float* g, float* v, const uint8_t* decay, int64_t n,
                      float lr, float mu, float wd, float grad_scale, cudaStream_t s,
                      const float* hp = nullptr);

}  // namespace tsm
