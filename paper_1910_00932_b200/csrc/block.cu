// The residual-shift TSM bottleneck unit on the tcgen05 conv engine.
//
// Reference: expand_layer (arch.cpp:278-323) builds
//   [TemporalShift(frac), 1x1 c_in->w +ReLU, 1x3x3 stride s +ReLU, 1x1 w->c_out]
//   + projection 1x1 stride s iff s != 1 or c_in != c_out, residual = true;
// run_unit (net.cpp:85-126) executes it with the skip on the UNSHIFTED input,
// loss_gradients (net.cpp:184-248) reverses it.
//
// Here the shift never exists as a tensor: forward it rides in conv1's TMA
// loads, backward its adjoint rides in conv1's dgrad epilogue (row
// permutation) and in conv1's wgrad B-operand loads.  ReLU backward masks and
// the skip-gradient add are fused into the dgrad epilogues.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "aux_kernels.cuh"
#include "block.h"
#include "common.cuh"
#include "generic_conv.h"

namespace tsm {

namespace {
inline size_t align256(size_t b) { return (b + 255) & ~size_t(255); }
}  // namespace

BlockPlan::BlockPlan(const tsm_block_desc& d) : d(d) {
  width = d.c_out / 4;
  frames = d.n * d.t;
  ho = (d.h + 2 - 3) / d.stride + 1;
  wo = (d.w + 2 - 3) / d.stride + 1;
  has_proj = d.stride != 1 || d.c_in != d.c_out;
  // the tcgen05 convs stage the shifted channel groups in slabs of 8+
  // channels; any other integral split (e.g. 1/16 of 64) runs on the direct
  // convs rather than failing at step time
  generic = d.c_in % 64 != 0 || width % 64 != 0 || d.fold_fwd % 8 != 0 || d.fold_bwd % 8 != 0;
  const char* fe = getenv("TSM_FUSED_BLOCK");
  fused = !generic && fe && atoi(fe) != 0 && d.c_in == 256 && d.c_out == 256 && d.stride == 1 &&
          d.fold_fwd == 32 && d.fold_bwd == 32;

  c1 = ConvShape{d.n, d.t, d.h, d.w, d.c_in, width, 1, 1, d.fold_fwd, d.fold_bwd};
  c2 = ConvShape{d.n, d.t, d.h, d.w, width, width, 3, (int)d.stride, 0, 0};
  c3 = ConvShape{d.n, d.t, ho, wo, width, d.c_out, 1, 1, 0, 0};
  cp = ConvShape{d.n, d.t, d.h, d.w, d.c_in, d.c_out, 1, (int)d.stride, 0, 0};

  const int64_t pin = frames * d.h * d.w, pout = frames * ho * wo;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += align256(bytes);
    return o;
  };
  // bf16 weights (forward + dgrad operands)
  o_w1f = take(width * d.c_in * 2);
  o_w1d = take(width * d.c_in * 2);
  o_w2f = take(width * 9 * width * 2);
  o_w2d = take(width * 9 * width * 2);
  o_w3f = take(d.c_out * width * 2);
  o_w3d = take(d.c_out * width * 2);
  o_wpf = has_proj ? take(d.c_out * d.c_in * 2) : 0;
  o_wpd = has_proj ? take(d.c_out * d.c_in * 2) : 0;
  // saved activations
  o_r1 = take(pin * width * 2);
  o_r2 = take(pout * width * 2);
  o_r1b = take(pin * width / 8);   // 1 bit per element
  o_r2b = take(pout * width / 8);
  o_yb = fused ? take(pout * d.c_out / 8) : 0;
  o_skip = has_proj ? take(pout * d.c_out * 2) : 0;
  // backward scratch
  o_g = take(pout * d.c_out * 2);
  o_g2 = take(pout * width * 2);
  o_g1 = take(pin * width * 2);
  o_gs = has_proj ? take(pin * d.c_in * 2) : 0;
  // zero-insert buffer: only odd extents miss the sub-pixel strided dgrad
  const bool zi = d.stride != 1 && (d.h != 2 * ho || d.w != 2 * wo);
  o_zi = zi ? take(pin * width * 2) : 0;
  size_t wg = std::max({wgrad_workspace_bytes(c1), wgrad_workspace_bytes(c2),
                        wgrad_workspace_bytes(c3)});
  if (has_proj) wg = std::max(wg, wgrad_workspace_bytes(cp));
  o_wg = take(wg);
  o_cs = take(colsum_workspace_floats(std::max(pin, pout), std::max(d.c_out, d.c_in)) * 4);
  bytes = off;
}

tsm_status BlockPlan::validate() const {
  if (d.n <= 0 || d.t <= 0 || d.h <= 0 || d.w <= 0 || d.c_in <= 0 || d.c_out <= 0)
    return fail(TSM_ERR_INVALID, "block: non-positive shape");
  if (d.c_out % 4 != 0)
    return fail(TSM_ERR_INVALID, "bottleneck channels_out is not a positive multiple of 4");
  if (d.stride != 1 && d.stride != 2) return fail(TSM_ERR_UNSUPPORTED, "block: stride 1 or 2");
  if (d.fold_fwd < 0 || d.fold_bwd < 0 || d.fold_fwd + d.fold_bwd > d.c_in)
    return fail(TSM_ERR_INVALID, "block: bad shift split");
  return TSM_OK;  // other channel counts run on the direct (generic) convs
}

tsm_status block_prepare_weights(const BlockPlan& P, const tsm_block_params& p, uint8_t* ws,
                                 bool dgrad, cudaStream_t s) {
  if (P.generic) return TSM_OK;  // the direct convs read the fp32 masters
  auto dg = [&](size_t o) -> void* { return dgrad ? ws + o : nullptr; };
  TSM_TRY(weights_to_bf16(p.w1, ws + P.o_w1f, dg(P.o_w1d), P.width, P.d.c_in, 1, P.d.c_in, s));
  TSM_TRY(weights_to_bf16(p.w2, ws + P.o_w2f, dg(P.o_w2d), P.width, P.width, 3, 9 * P.width, s));
  TSM_TRY(weights_to_bf16(p.w3, ws + P.o_w3f, dg(P.o_w3d), P.d.c_out, P.width, 1, P.width, s));
  if (P.has_proj)
    TSM_TRY(weights_to_bf16(p.wp, ws + P.o_wpf, dg(P.o_wpd), P.d.c_out, P.d.c_in, 1, P.d.c_in, s));
  return TSM_OK;
}

tsm_status block_forward(const BlockPlan& P, const tsm_block_params& p, const void* x, void* y,
                         uint8_t* ws, uint32_t* y_bits, cudaStream_t s) {
  if (P.generic) {
    if (y_bits) return fail(TSM_ERR_UNSUPPORTED, "block: no bitmask output on the generic path");
    TSM_TRY(gconv_fwd(P.c1, x, p.w1, p.b1, nullptr, ws + P.o_r1, 1, s));
    TSM_TRY(gconv_fwd(P.c2, ws + P.o_r1, p.w2, p.b2, nullptr, ws + P.o_r2, 1, s));
    const void* gskip_x = x;
    if (P.has_proj) {
      TSM_TRY(gconv_fwd(P.cp, x, p.wp, p.bp, nullptr, ws + P.o_skip, 0, s));
      gskip_x = ws + P.o_skip;
    }
    return gconv_fwd(P.c3, ws + P.o_r2, p.w3, p.b3, gskip_x, y, 1, s);
  }
  if (P.fused) {
    // conv1 -> conv2 -> conv3 + skip in one kernel, r1 / r2 on chip (the
    // saved activations and bitmasks are still written for the backward)
    TraceScope t("fused unit");
    return bottleneck_fused_fwd(x, ws + P.o_w1f, ws + P.o_w2f, ws + P.o_w3f, p.b1, p.b2, p.b3, y,
                                ws + P.o_r1, ws + P.o_r2, reinterpret_cast<uint32_t*>(ws + P.o_r1b),
                                reinterpret_cast<uint32_t*>(ws + P.o_r2b),
                                y_bits ? y_bits : reinterpret_cast<uint32_t*>(ws + P.o_yb),
                                P.d.n, P.d.t, P.d.h, P.d.w, s);
  }
  // Each ReLU output also leaves a 1-bit mask for its relu_backward (the
  // backward epilogues read bits instead of the bf16 activation).
  // r1 = relu(conv1x1(shift(x)) + b1): the fused shift + 1x1 conv
  const bool shifted = P.c1.F + P.c1.B > 0;
  if (shifted) probe_conv1_begin(s, P.c1.c_in, P.c1.c_out, P.c1.clips * P.c1.T * P.c1.H * P.c1.W);
  {
    TraceScope t1(shifted ? "shift+c1" : "c1");
    TSM_TRY(conv_fwd(P.c1, x, ws + P.o_w1f, p.b1, nullptr, ws + P.o_r1, 1, s,
                     reinterpret_cast<uint32_t*>(ws + P.o_r1b)));
  }
  if (shifted) probe_conv1_end(s);
  // r2 = relu(conv3x3_s(r1) + b2)
  {
    TraceScope t2("c2");
    TSM_TRY(conv_fwd(P.c2, ws + P.o_r1, ws + P.o_w2f, p.b2, nullptr, ws + P.o_r2, 1, s,
                     reinterpret_cast<uint32_t*>(ws + P.o_r2b)));
  }
  // skip = proj(x) (unshifted x) or x
  const void* skip = x;
  if (P.has_proj) {
    TraceScope tp("proj");
    TSM_TRY(conv_fwd(P.cp, x, ws + P.o_wpf, p.bp, nullptr, ws + P.o_skip, 0, s));
    skip = ws + P.o_skip;
  }
  // y = relu(conv1x1(r2) + b3 + skip)
  TraceScope t3("c3+res");
  return conv_fwd(P.c3, ws + P.o_r2, ws + P.o_w3f, p.b3, skip, y, 1, s, y_bits);
}

tsm_status block_backward(const BlockPlan& P, const tsm_block_params& p, const void* x,
                          const void* g_in, bool g_is_masked, const void* y, void* gx,
                          const void* gx_mask, const tsm_block_grads& g, uint8_t* ws,
                          cudaStream_t s, const uint32_t* y_bits,
                          const uint32_t* gx_mask_bits) {
  return block_backward(P, p, x, g_in, g_is_masked, y, gx, gx_mask, g, ws, s, y_bits,
                        gx_mask_bits, WgradStream{});
}

tsm_status block_backward(const BlockPlan& P, const tsm_block_params& p, const void* x,
                          const void* g_in, bool g_is_masked, const void* y, void* gx,
                          const void* gx_mask, const tsm_block_grads& g, uint8_t* ws,
                          cudaStream_t s, const uint32_t* y_bits,
                          const uint32_t* gx_mask_bits, const WgradStream& side){
  const auto* r1b = reinterpret_cast<const uint32_t*>(ws + P.o_r1b);
  const auto* r2b = reinterpret_cast<const uint32_t*>(ws + P.o_r2b);
  if (P.generic) {
    const int64_t pout_g = P.frames * P.ho * P.wo;
    const void* gm = g_in;
    if (!g_is_masked) {
      TSM_TRY(relu_mask(g_in, y, ws + P.o_g, pout_g * P.d.c_out, s, y_bits));
      gm = ws + P.o_g;
    }
    TSM_TRY(gconv_wgrad(P.c3, ws + P.o_r2, gm, g.w3, g.b3, s));
    TSM_TRY(gconv_dgrad(P.c3, gm, p.w3, nullptr, ws + P.o_r2, nullptr, ws + P.o_g2, s));
    TSM_TRY(gconv_wgrad(P.c2, ws + P.o_r1, ws + P.o_g2, g.w2, g.b2, s));
    TSM_TRY(gconv_dgrad(P.c2, ws + P.o_g2, p.w2, nullptr, ws + P.o_r1, nullptr, ws + P.o_g1, s));
    TSM_TRY(gconv_wgrad(P.c1, x, ws + P.o_g1, g.w1, g.b1, s));
    const void* gskip = gm;
    if (P.has_proj) {
      TSM_CUDA_TRY(cudaMemcpyAsync(g.bp, g.b3, P.d.c_out * sizeof(float),
                                   cudaMemcpyDeviceToDevice, s));
      TSM_TRY(gconv_wgrad(P.cp, x, gm, g.wp, nullptr, s));
      TSM_TRY(gconv_dgrad(P.cp, gm, p.wp, nullptr, nullptr, nullptr, ws + P.o_gs, s));
      gskip = ws + P.o_gs;
    }
    return gconv_dgrad(P.c1, ws + P.o_g1, p.w1, gskip, gx_mask, gx_mask_bits, gx, s);
  }
  const int64_t pout = P.frames * P.ho * P.wo;
  float* wgw = reinterpret_cast<float*>(ws + P.o_wg);
  // g = gy * (y > 0): relu backward of the residual output (net.cpp:192-198)
  const void* gm = g_in;
  if (!g_is_masked) {
    TraceScope t("relu mask");
    TSM_TRY(relu_mask(g_in, y, ws + P.o_g, pout * P.d.c_out, s, y_bits));
    gm = ws + P.o_g;
  }
  // Bias gradients (kernels.cpp:312-325) are fused into the weight-gradient
  // GEMM, which already streams dY through shared memory.  The weight
  // gradients only read (saved activations, this unit's own gradient
  // buffers), so they run on the side stream `sw` when one is given, each
  // forked once its dY exists: the dgrad chain on `s` (the critical path)
  // and the wgrads overlap, and each fills the other's kernel tails.
  cudaStream_t sw = side.sw ? side.sw : s;
  auto fork = [&](int k) -> tsm_status {
    if (sw == s) return TSM_OK;
    TSM_CUDA_TRY(cudaEventRecord(side.fork[k], s));
    TSM_CUDA_TRY(cudaStreamWaitEvent(sw, side.fork[k], 0));
    return TSM_OK;
  };
  // conv3: dW3 + db3, g2 = dgrad(g) masked by r2 > 0
  TSM_TRY(fork(0));
  {
    TraceScope t("wgrad c3");
    TSM_TRY(conv_wgrad(P.c3, ws + P.o_r2, gm, g.w3, g.b3, wgw, sw));
  }
  if (P.has_proj) {
    TraceScope t("wgrad proj");
    // the projection's bias gradient is the same column sum of g as db3
    TSM_CUDA_TRY(cudaMemcpyAsync(g.bp, g.b3, P.d.c_out * sizeof(float),
                                 cudaMemcpyDeviceToDevice, sw));
    TSM_TRY(conv_wgrad(P.cp, x, gm, g.wp, nullptr, wgw, sw));
  }
  {
    TraceScope t("dgrad c3");
    TSM_TRY(conv_dgrad(P.c3, gm, ws + P.o_w3d, nullptr, nullptr, ws + P.o_g2, nullptr, s, r2b));
  }
  // conv2: dW2 + db2, g1 = dgrad(g2) masked by r1 > 0
  TSM_TRY(fork(1));
  {
    TraceScope t("wgrad c2");
    TSM_TRY(conv_wgrad(P.c2, ws + P.o_r1, ws + P.o_g2, g.w2, g.b2, wgw, sw));
  }
  {
    TraceScope t(P.d.stride == 1 ? "dgrad c2" : "dgrad c2 (strided, sub-pixel classes)");
    TSM_TRY(conv_dgrad(P.c2, ws + P.o_g2, ws + P.o_w2d, nullptr, nullptr, ws + P.o_g1,
                       P.o_zi ? ws + P.o_zi : nullptr, s, r1b));
  }
  // conv1 (after the shift): dW1 with the shifted x read in the loads, + db1
  TSM_TRY(fork(2));
  {
    TraceScope t(P.c1.F + P.c1.B ? "wgrad c1 (shifted x)" : "wgrad c1");
    TSM_TRY(conv_wgrad(P.c1, x, ws + P.o_g1, g.w1, g.b1, wgw, sw));
  }
  // skip gradient
  const void* gskip = gm;
  // strided projection with bitmask (or no) masking: its gradient lands on
  // a quarter of the rows, so it is added onto conv1's gradient in place
  // (mask(a + b) = mask(a) + mask(b)) instead of through a zero-filled
  // full-size skip tensor read back as conv1's residual
  const bool proj_acc = P.has_proj && P.cp.stride != 1 && !gx_mask && P.d.c_in % 32 == 0;
  if (P.has_proj) {
    if (!proj_acc) {
      TraceScope t("dgrad proj");
      TSM_TRY(conv_dgrad(P.cp, gm, ws + P.o_wpd, nullptr, nullptr, ws + P.o_gs, nullptr, s));
      gskip = ws + P.o_gs;
    }
  }
  // gx = shift_adjoint(dgrad1(g1)) + skip_grad  (net.cpp:217-219, 238-247),
  // optionally masked by the producer's ReLU (the previous unit's output).
  if (!proj_acc) {
    TraceScope t1("dgrad c1 (adjoint shift + skip)");
    return conv_dgrad(P.c1, ws + P.o_g1, ws + P.o_w1d, gskip, gx_mask, gx, nullptr, s,
                      gx_mask_bits);
  }
  {
    TraceScope t1("dgrad c1 (adjoint shift)");
    TSM_TRY(conv_dgrad(P.c1, ws + P.o_g1, ws + P.o_w1d, nullptr, nullptr, gx, nullptr, s,
                       gx_mask_bits));
  }
  TraceScope tp("dgrad proj (+= into dx)");
  return conv_dgrad(P.cp, gm, ws + P.o_wpd, nullptr, nullptr, gx, nullptr, s, gx_mask_bits,
                    /*accumulate=*/1);
}

}  // namespace tsm
