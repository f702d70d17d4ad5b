// Bandwidth-bound helper kernels around the tcgen05 convs: layout
// conversion, weight re-layouts, split-K reduction, bias gradients, ReLU
// masks, zero insertion, pooling, the classifier head and the SGD update.
// All are deterministic (gather form, fixed-order sums, no float atomics).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "tsm_b200.h"

namespace tsm {

// out[i] = sum_{s < splits} ws[s * n + i], summed in split order.
tsm_status splitk_reduce(const float* ws, float* out, int splits, int64_t n, cudaStream_t st);
// out[j][i] = sum_{s < splits} ws[s][i][j] for ws [splits][m][n] (transposing reduce).
tsm_status splitk_reduce_transpose(const float* ws, float* out, int splits, int64_t m, int64_t n,
                                   cudaStream_t st);

// dy [frames][ho][wo][c] -> out [frames][2ho][2wo][c], zeros off the even grid.
tsm_status zero_insert(const void* dy, void* out, int64_t frames, int64_t ho, int64_t wo,
                       int64_t c, cudaStream_t st);

// Column sums of a bf16 [rows][c] matrix into fp32 db[c] (bias gradient,
// kernels.cpp:312-325).  `ws` needs colsum_workspace_floats(rows, c) floats.
int64_t colsum_workspace_floats(int64_t rows, int64_t c);
tsm_status colsum_bf16(const void* g, float* db, float* ws, int64_t rows, int64_t c,
                       cudaStream_t st);

// fp32 master weights -> bf16 operands:
//   w_fwd [co][k*k][ci]        (K-major forward operand, K padded to k_pad)
//   w_dgrad [ci][k*k][co]      (tap-flipped transpose for dgrad; nullable)
tsm_status weights_to_bf16(const float* w, void* w_fwd, void* w_dgrad, int64_t co, int64_t ci,
                           int k, int64_t k_pad, cudaStream_t st);
// The same for many tensors in one launch (job table in device memory).
struct WeightJob {
  const float* w;
  void* w_fwd;
  void* w_dgrad;
  int64_t co, ci;
  int kk;
  int64_t k_pad;
};
tsm_status weights_to_bf16_batch(const WeightJob* jobs_dev, int njobs, cudaStream_t st);
// Narrow shift splits (F + B <= vg = 32, not multiples of 32) in virtual
// channels (tc_gemm.cuh OpLoad::vg): the weight gradient's split-K reduction
// reading the virtual rows [m_v][co] back into [co][ci].
tsm_status splitk_reduce_transpose_vmap(const float* ws, float* out, int splits, int64_t m_v,
                                        int64_t ci, int64_t co, int64_t F, int64_t B, int64_t vg,
                                        cudaStream_t st);
// Two independent split-K reductions in one launch (weight + bias partials).
tsm_status splitk_reduce2(const float* ws1, float* out1, int64_t n1, const float* ws2,
                          float* out2, int64_t n2, int splits, cudaStream_t st);

// NTCHW (fp32/fp64/bf16) <-> NTHWC bf16, with optional channel padding c -> c_pad (zeros).
tsm_status ntchw_to_nthwc(const void* x, tsm_dtype dt, void* y, int64_t frames, int64_t c,
                          int64_t hw, int64_t c_pad, cudaStream_t st);
tsm_status nthwc_to_ntchw(const void* x, void* y, tsm_dtype dt, int64_t frames, int64_t c,
                          int64_t hw, cudaStream_t st);

// Fill the boundary frames the TMA adjoint-shift epilogue leaves unwritten:
// dx[:, T-1, :, 0:F] and dx[:, 0, :, F:F+B] = mask?(residual or 0).
tsm_status shift_out_boundary(void* dx, const void* residual, const void* mask, int64_t clips,
                              int64_t T, int64_t hw, int64_t c, int64_t F, int64_t B,
                              cudaStream_t st, const uint32_t* mask_bits = nullptr);

// g = gy * (y > 0)  (relu_backward, kernels.cpp:587-596), bf16, elementwise;
// with `bits` (ReLU bitmask of y, n % 32 == 0) y is not read.
tsm_status relu_mask(const void* gy, const void* y, void* g, int64_t n, cudaStream_t st,
                     const uint32_t* bits = nullptr);

}  // namespace tsm
