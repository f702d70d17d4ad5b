// Internal (C++) entry points of the tcgen05 conv engine.  The C ABI in
// capi.cu wraps these; layouts are documented in include/tsm_b200.h.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "tsm_b200.h"

namespace tsm {

tsm_status conv1x1_fwd(const void* x, const void* w, const float* bias, const void* residual,
                       void* y, int64_t clips, int64_t T, int64_t HW, int64_t c_in,
                       int64_t c_out, int64_t F, int64_t B, int relu, cudaStream_t stream);

}  // namespace tsm
