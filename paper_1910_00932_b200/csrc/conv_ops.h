// Internal (C++) entry points of the tcgen05 conv engine and its helpers.
// The C ABI in capi.cu wraps these; layouts are documented in
// include/tsm_b200.h.  Activations NTHWC bf16; weights bf16 [c_out][k][k][c_in]
// (K-major GEMM operand); weight gradients fp32 in the same layout.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "tsm_b200.h"

namespace tsm {

struct ConvShape {
  int64_t clips = 1, T = 1, H = 1, W = 1;  // input extents; frames = clips * T
  int64_t c_in = 0, c_out = 0;
  int k = 1, stride = 1;                   // square kernel, padding k/2
  int64_t F = 0, B = 0;                    // temporal shift split before the conv (k=1, s=1)
  int64_t h_out() const { return (H + 2 * (k / 2) - k) / stride + 1; }
  int64_t w_out() const { return (W + 2 * (k / 2) - k) / stride + 1; }
};

// ReLU bitmasks: [rows][c / 32] uint32 words, bit j of word w = channel
// 32 w + j.  conv_fwd's `bits_out` records bf16(y) > 0; conv_dgrad's
// `mask_bits` applies such a mask in place of the bf16 `mask` tensor.
tsm_status conv_fwd(const ConvShape& s, const void* x, const void* w, const float* bias,
                    const void* residual, void* y, int relu, cudaStream_t stream,
                    uint32_t* bits_out = nullptr);
// accumulate (strided 1x1 only): dx rows of the stride grid become
// bf16(dx + value) instead of dx being zeroed and overwritten — the strided
// projection's input gradient added onto conv1's (no zero fill, no full-size
// skip tensor).
tsm_status conv_dgrad(const ConvShape& s, const void* dy, const void* wt, const void* residual,
                      const void* mask, void* dx, void* scratch, cudaStream_t stream,
                      const uint32_t* mask_bits = nullptr, int accumulate = 0);
int wgrad_splits(const ConvShape& s);
size_t wgrad_workspace_bytes(const ConvShape& s);
tsm_status conv_wgrad(const ConvShape& s, const void* x, const void* dy, float* dw, float* db, float* ws,
                      cudaStream_t stream);

// Narrow shift splits (F + B <= kVShift, not multiples of 32 — res2.0's 8 +
// 8 of 64 channels): conv_wgrad takes them in virtual channels when c_out =
// 64 (conv_ops.cu conv_wgrad_vshift).
constexpr int kVShift = 32;
bool vshift_ok(const ConvShape& s);

// The res2 identity bottleneck unit (c_in = c_out = 256, width 64, F = B =
// 32, stride 1) in one kernel (fused_block.cuh): x, y NTHWC bf16; bf16
// weights in the forward GEMM layout; writes y, the saved r1 / r2 and the
// three ReLU bitmasks exactly as the three-kernel sequence does.
tsm_status bottleneck_fused_fwd(const void* x, const void* w1f, const void* w2f, const void* w3f,
                                const float* b1, const float* b2, const float* b3, void* y,
                                void* r1, void* r2, uint32_t* r1_bits, uint32_t* r2_bits,
                                uint32_t* y_bits, int64_t clips, int64_t T, int64_t H, int64_t W,
                                cudaStream_t stream);

// Space-to-depth stem conv (see head_kernels.cuh stem_s2d).
bool stem_pool_enabled();
bool stem_pool_bwd_enabled();
tsm_status stem_s2d_wgrad_pool(const void* xs, const void* gy, const uint8_t* arg, float* dw,
                               float* db, float* ws, int64_t clips, int64_t T, int64_t H2,
                               int64_t W2, cudaStream_t stream);
tsm_status stem_pool_fwd(const void* xs, const void* wf, const float* bias, void* y,
                         uint8_t* arg, int64_t frames, int64_t H2, int64_t W2,
                         cudaStream_t stream);
tsm_status stem_s2d_fwd(const void* xs, const void* wf, const float* bias, void* y,
                        int64_t frames, int64_t H2, int64_t W2, cudaStream_t stream);
size_t stem_s2d_wgrad_workspace_bytes(int64_t clips, int64_t T, int64_t H2, int64_t W2);
tsm_status stem_s2d_wgrad(const void* xs, const void* dy, float* dw, float* db, float* ws,
                          int64_t clips, int64_t T, int64_t H2, int64_t W2, cudaStream_t stream);

}  // namespace tsm
