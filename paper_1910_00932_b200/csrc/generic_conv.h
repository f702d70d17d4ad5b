// Direct (CUDA-core) convolutions for units whose channel counts do not fit
// the tcgen05 tiles (e.g. the reference's micro-tsm preset).  Same
// semantics as conv_ops.h (NTHWC bf16 activations, padding k/2, temporal
// shift F/B before a 1x1 stride-1 conv), but fp32 master weights
// [c_out][k][k][c_in] are read directly.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "conv_ops.h"

namespace tsm {

// y = act(conv(shift(x)) + bias (+ residual))
tsm_status gconv_fwd(const ConvShape& s, const void* x, const float* w, const float* bias,
                     const void* residual, void* y, int relu, cudaStream_t st);
// dx = mask? (shift_adjoint(dgrad(dy)) + residual); mask as bf16 tensor or bitmask
tsm_status gconv_dgrad(const ConvShape& s, const void* dy, const float* w, const void* residual,
                       const void* mask, const uint32_t* mask_bits, void* dx, cudaStream_t st);
// dw (and db, nullable) = sum over positions of dy (x) shift(x) windows
tsm_status gconv_wgrad(const ConvShape& s, const void* x, const void* dy, float* dw, float* db,
                       cudaStream_t st);

}  // namespace tsm
