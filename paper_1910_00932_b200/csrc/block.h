// Planner + executor of one residual-shift bottleneck unit (see block.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "conv_ops.h"
#include "tsm_b200.h"

namespace tsm {

struct BlockPlan {
  tsm_block_desc d;
  int64_t width, frames, ho, wo;
  bool has_proj;
  // channel counts that do not fit the tcgen05 tiles (c_in, c_out/4 not
  // multiples of 64, e.g. micro-tsm): direct CUDA-core convs (generic_conv.h)
  bool generic;
  // the res2 identity unit (256 -> 64 -> 256, shift 1/8, stride 1) runs its
  // forward as one fused kernel (fused_block.cuh) when TSM_FUSED_BLOCK=1
  bool fused;
  ConvShape c1, c2, c3, cp;
  // workspace offsets (bytes)
  size_t o_w1f, o_w1d, o_w2f, o_w2d, o_w3f, o_w3d, o_wpf, o_wpd;
  size_t o_r1, o_r2, o_skip, o_g, o_g2, o_g1, o_gs, o_zi, o_wg, o_cs;
  size_t o_r1b, o_r2b;  // ReLU bitmasks of r1 / r2 (backward masks)
  size_t o_yb;          // fused forward: the output's bitmask when the caller keeps none
  size_t bytes;
  explicit BlockPlan(const tsm_block_desc& d);
  tsm_status validate() const;
};

tsm_status block_prepare_weights(const BlockPlan& P, const tsm_block_params& p, uint8_t* ws,
                                 bool dgrad, cudaStream_t s);
// y_bits (nullable): also record the output's ReLU bitmask ([rows][c_out/32]).
tsm_status block_forward(const BlockPlan& P, const tsm_block_params& p, const void* x, void* y,
                         uint8_t* ws, uint32_t* y_bits, cudaStream_t s);
// g_in: gradient w.r.t. the unit output y; if !g_is_masked it is multiplied
// by (y > 0) first (from y_bits when given).  gx_mask / gx_mask_bits
// (nullable, at most one): multiply gx by the producer's ReLU mask.
tsm_status block_backward(const BlockPlan& P, const tsm_block_params& p, const void* x,
                          const void* g_in, bool g_is_masked, const void* y, void* gx,
                          const void* gx_mask, const tsm_block_grads& g, uint8_t* ws,
                          cudaStream_t s, const uint32_t* y_bits = nullptr,
                          const uint32_t* gx_mask_bits = nullptr);

// Weight gradients on a second stream: `sw` runs the unit's wgrads (and the
// bias-gradient copies) concurrently with the input-gradient chain on `s`,
// forked by `fork[0..2]` (gm ready / g2 ready / g1 ready).  The unit's
// parameter gradients are final when `sw` reaches its end of this call.
struct WgradStream {
  cudaStream_t sw = nullptr;
  cudaEvent_t fork[3] = {nullptr, nullptr, nullptr};
};
tsm_status block_backward(const BlockPlan& P, const tsm_block_params& p, const void* x,
                          const void* g_in, bool g_is_masked, const void* y, void* gx,
                          const void* gx_mask, const tsm_block_grads& g, uint8_t* ws,
                          cudaStream_t s, const uint32_t* y_bits, const uint32_t* gx_mask_bits,
                          const WgradStream& side);

}  // namespace tsm
