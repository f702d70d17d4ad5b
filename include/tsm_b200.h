/* tsm_b200 — C ABI of the B200-native Temporal Shift Module hot path.
 *
 * This is the drop-in boundary for the reference library `vidperf`
 * (/root/reference/proj, C++20, CPU fp64).  Every entry point names the
 * reference interface it replaces.  Rules shared by all entry points:
 *
 *  - plain pointers and sizes only; device pointers unless stated; `stream`
 *    is a cudaStream_t passed as void* (NULL = legacy default stream);
 *  - tensors are dense row-major [N][T][C][H][W] (tensor.hpp:14-47) unless
 *    stated otherwise;
 *  - no exceptions cross the ABI: a tsm_status is returned and
 *    tsm_last_error() holds the message.  TSM_ERR_INVALID maps to
 *    vidperf::ValidationError (errors.hpp:11-13, CLI exit 1); TSM_ERR_CUDA /
 *    TSM_ERR_NCCL map to std::runtime_error (CLI exit 2,
 *    tools/vidperf.cpp:475-485);
 *  - the library never allocates on behalf of the caller on the shift path;
 *    everything is stream-ordered and reentrant on distinct streams;
 *  - results are bitwise deterministic run to run (no float atomics).
 *
 * There is no CPU fallback: if no sm_100 device is present every compute
 * entry point returns TSM_ERR_CUDA.
 */
#ifndef TSM_B200_H
#define TSM_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define TSM_API __attribute__((visibility("default")))
#else
#define TSM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum tsm_status {
  TSM_OK = 0,
  TSM_ERR_INVALID = 1,     /* bad split / shape / weights -> vidperf::ValidationError */
  TSM_ERR_ALIAS = 2,       /* x and y overlap; the shift is out-of-place (kernels.cpp:102) */
  TSM_ERR_UNSUPPORTED = 3, /* dtype / geometry this build does not implement */
  TSM_ERR_CUDA = 4,        /* CUDA runtime/driver failure or no sm_100 device */
  TSM_ERR_NCCL = 5         /* NCCL failure in the data-parallel step */
} tsm_status;

typedef enum tsm_dtype {
  TSM_F32 = 0,
  TSM_BF16 = 1,
  TSM_F64 = 2,
  TSM_F16 = 3
} tsm_dtype;

/* Message for the last non-OK status returned on this thread. */
TSM_API const char* tsm_last_error(void);
/* ABI version; bumped on any signature change. */
TSM_API int tsm_abi_version(void);
/* sha256 (hex) of the concatenated library sources this binary was built
 * from (sorted csrc/*.cu, *.cuh, *.h and include/*.h). */
TSM_API const char* tsm_source_hash(void);

/* ---------------------------------------------------------------------------
 * Channel split.  Replaces vidperf::validate_shift (kernels.hpp:22,
 * kernels.cpp:82-95) and the exact_multiple calls that follow it
 * (kernels.cpp:100-101; rational.cpp:50-61).  Fractions are exact rationals
 * (num/den); the split must be integral, non-negative and fwd+bwd <= C.
 * On success *fold_fwd / *fold_bwd receive the channel counts F and B. */
TSM_API tsm_status tsm_validate_shift(int64_t fwd_num, int64_t fwd_den, int64_t bwd_num,
                              int64_t bwd_den, int64_t channels, int64_t* fold_fwd,
                              int64_t* fold_bwd);

/* ---------------------------------------------------------------------------
 * Temporal shift.  Replaces vidperf::temporal_shift (kernels.hpp:24,
 * kernels.cpp:97-125):
 *     y[n,t,c]     = x[n,t-1,c]   for c <  F         (+0.0 at t = 0)
 *     y[n,t,c]     = x[n,t+1,c]   for F <= c < F+B   (+0.0 at t = T-1)
 *     y[n,t,c]     = x[n,t,c]     otherwise
 * fold_fwd = F, fold_bwd = B as returned by tsm_validate_shift (fold_div = 8
 * gives F = B = C/8).  Bitwise copy: any dtype, NaN payloads and -0.0 are
 * preserved; the boundary fill is all-zero bytes (+0.0).  x and y are device
 * buffers of n*t*c*h*w elements that must not overlap.  All dims >= 1. */
TSM_API tsm_status tsm_shift_fwd(const void* x, void* y, int64_t n, int64_t t, int64_t c, int64_t h,
                         int64_t w, int64_t fold_fwd, int64_t fold_bwd, tsm_dtype dtype,
                         void* stream);

/* The adjoint.  Replaces vidperf::temporal_shift_adjoint (kernels.hpp:26,
 * kernels.cpp:127-157): channels c < F read t+1, F <= c < F+B read t-1. */
TSM_API tsm_status tsm_shift_bwd(const void* dy, void* dx, int64_t n, int64_t t, int64_t c, int64_t h,
                         int64_t w, int64_t fold_fwd, int64_t fold_bwd, tsm_dtype dtype,
                         void* stream);

/* Host-buffer convenience with the reference's value semantics
 * (const Tensor5D& in, new Tensor5D out; kernels.cpp:97-157): copies host x
 * to the device, shifts, copies back into host y, synchronously.  x and y are
 * HOST pointers (pageable or pinned).  adjoint = 0 forward, 1 adjoint. */
TSM_API tsm_status tsm_shift_host(const void* x, void* y, int64_t n, int64_t t, int64_t c, int64_t h,
                          int64_t w, int64_t fold_fwd, int64_t fold_bwd, tsm_dtype dtype,
                          int adjoint);

/* ---------------------------------------------------------------------------
 * Bottleneck convolutions on the tensor cores (tcgen05 + TMEM + TMA).
 *
 * Block-internal layout is channels-last per frame, "NTHWC": x[n][t][h][w][c]
 * bf16 (rows = pixels, channels contiguous), fp32 accumulation.  Weights are
 * bf16 [c_out][kh][kw][c_in] (K zero-padded to a multiple of 64 when
 * kh*kw*c_in is not); biases fp32 [c_out].  Convolutions are square, padding
 * k/2, spatial stride `stride`, temporal kernel 1 (the frame-local path of
 * conv_forward, kernels.cpp:171-200).
 *
 * Forward (conv_forward, kernels.cpp:162-231):
 *     y = act( conv_k( temporal_shift(x, F, B) ) + bias (+ residual) )
 * With F, B > 0 (k = 1, stride 1 only) the shift is applied inside the TMA
 * loads of the GEMM (channel groups [0,F) / [F,F+B) fetched at frame t-1 /
 * t+1, out-of-clip frames zero-filled by TMA), so the shifted activation is
 * never materialised: the fused shift + 1x1 conv of north-star (b), i.e. the
 * first two ops of the unit expand_layer builds (arch.cpp:291-302).
 * act = ReLU when relu != 0, applied after the residual add when residual is
 * given, as in run_unit's relu(add(main, skip)) (net.cpp:119-124).
 * Requirements: c_out % 16 == 0; 1x1 stride-1: c_in % 64 == 0, F and F+B
 * multiples of 8; im2col path: c_in in {8, 32} or a multiple of 64. */
TSM_API tsm_status tsm_conv_fwd(const void* x, const void* w, const float* bias,
                                const void* residual, void* y, int64_t n, int64_t t, int64_t h,
                                int64_t w_, int64_t c_in, int64_t c_out, int k, int stride,
                                int64_t fold_fwd, int64_t fold_bwd, int relu, void* stream);

/* Input gradient (conv_backward grad_x, kernels.cpp:246-280), with the shift
 * adjoint (kernels.cpp:127-157) fused into the epilogue when F, B > 0:
 *     dx = mask? ( shift_adjoint( dgrad(dy) ) + residual )
 * wt is the dgrad operand: [c_in][k][k][c_out] with the taps reversed
 * (tsm_weights_to_bf16 produces it).  mask (optional, layout of dx):
 * dx *= (mask > 0), i.e. the relu_backward of the producing layer.
 * Stride 2 with k = 3 needs `scratch` of n*t*h*w*c_out bf16. */
TSM_API tsm_status tsm_conv_dgrad(const void* dy, const void* wt, const void* residual,
                                  const void* mask, void* dx, void* scratch, int64_t n,
                                  int64_t t, int64_t h, int64_t w_, int64_t c_in, int64_t c_out,
                                  int k, int stride, int64_t fold_fwd, int64_t fold_bwd,
                                  void* stream);

/* Weight gradient (conv_backward grad_w, kernels.cpp:282-310):
 *     dw[co][tap][ci] = sum_pixels dy[p][co] * im2col(shift(x))[p][tap][ci]
 * fp32, split over pixels deterministically; `ws` needs
 * tsm_conv_wgrad_workspace_bytes(...) bytes (an upper bound over every shift
 * split of the shape). */
TSM_API size_t tsm_conv_wgrad_workspace_bytes(int64_t n, int64_t t, int64_t h, int64_t w_,
                                              int64_t c_in, int64_t c_out, int k, int stride);
TSM_API tsm_status tsm_conv_wgrad(const void* x, const void* dy, float* dw, float* db, void* ws,
                                  int64_t n, int64_t t, int64_t h, int64_t w_, int64_t c_in,
                                  int64_t c_out, int k, int stride, int64_t fold_fwd,
                                  int64_t fold_bwd, void* stream);
/* (db, nullable: the bias gradient sum_pixels dy[p][co], kernels.cpp:312-325,
 * computed in the same pass over dy by the GEMM's epilogue warps.) */

/* fp32 master weights [c_out][k][k][c_in] -> bf16 forward operand (K padded
 * to k_pad) and, when w_dgrad != NULL, the dgrad operand [c_in][k][k][c_out]
 * with reversed taps. */
TSM_API tsm_status tsm_weights_to_bf16(const float* w, void* w_fwd, void* w_dgrad, int64_t c_out,
                                       int64_t c_in, int k, int64_t k_pad, void* stream);

/* Bias gradient: db[c] = sum over rows of g[rows][c] (kernels.cpp:312-325). */
TSM_API size_t tsm_bias_grad_workspace_bytes(int64_t rows, int64_t c);
/* Stem max pool 1x3x3 / stride 2 / pad 1 on NTHWC bf16 (max_pool_forward /
 * max_pool_backward, kernels.cpp:353-455): padded taps never win, ties keep
 * the first element in (h, w) scan order.  argmax: one byte per output
 * element (tap 0..8), written by fwd and read by bwd.  c % 8 == 0. */
TSM_API tsm_status tsm_maxpool_fwd(const void* x, void* y, uint8_t* argmax, int64_t frames,
                                   int64_t h, int64_t w, int64_t c, void* stream);
TSM_API tsm_status tsm_maxpool_bwd(const void* gy, const uint8_t* argmax, void* gx,
                                   int64_t frames, int64_t h, int64_t w, int64_t c, void* stream);

TSM_API tsm_status tsm_bias_grad(const void* g, float* db, void* ws, int64_t rows, int64_t c,
                                 void* stream);

/* Layout conversion between the reference's NTCHW (f32 / f64 / bf16) and the
 * block-internal NTHWC bf16; c_pad >= c pads channels with zeros. */
TSM_API tsm_status tsm_layout_to_nthwc(const void* x, tsm_dtype dtype, void* y, int64_t frames,
                                       int64_t c, int64_t h, int64_t w_, int64_t c_pad,
                                       void* stream);
TSM_API tsm_status tsm_layout_to_ntchw(const void* x, void* y, tsm_dtype dtype, int64_t frames,
                                       int64_t c, int64_t h, int64_t w_, void* stream);

/* ---------------------------------------------------------------------------
 * The residual-shift bottleneck unit (expand_layer, arch.cpp:278-323;
 * forward run_unit net.cpp:85-126; backward loss_gradients net.cpp:184-248
 * for one unit):
 *     r1 = relu(conv1x1(shift(x)) + b1)            c_in  -> width = c_out/4
 *     r2 = relu(conv3x3_stride(r1) + b2)           width -> width
 *     y  = relu(conv1x1(r2) + b3 + skip)           width -> c_out
 *     skip = x, or conv1x1_stride(x) + bp when stride != 1 or c_in != c_out
 * The skip reads the UNSHIFTED x (net.cpp:120).  x, y NTHWC bf16.  Weights
 * fp32 [c_out][kh][kw][c_in] (GEMM layout; the reference's (c_out, c_in, kt,
 * kh, kw) order is permuted on import), biases fp32.  The workspace holds the
 * bf16 weights and the saved activations between tsm_block_fwd and
 * tsm_block_bwd.  Gradients are fp32 sums over the batch (Sigma-loss
 * convention, net.cpp:141-146). */
typedef struct tsm_block_desc {
  int64_t n, t, h, w;          /* clips, frames per clip, input spatial extent */
  int64_t c_in, c_out;         /* block input / output channels; width = c_out / 4 */
  int32_t stride;              /* spatial stride of the 3x3 conv and the projection */
  int64_t fold_fwd, fold_bwd;  /* shift split of c_in (0, 0: no shift) */
} tsm_block_desc;

typedef struct tsm_block_params {
  const float *w1, *b1, *w2, *b2, *w3, *b3, *wp, *bp; /* wp, bp NULL without projection */
} tsm_block_params;

typedef struct tsm_block_grads {
  float *w1, *b1, *w2, *b2, *w3, *b3, *wp, *bp;
} tsm_block_grads;

TSM_API size_t tsm_block_workspace_bytes(const tsm_block_desc* d);
TSM_API tsm_status tsm_block_fwd(const tsm_block_desc* d, const tsm_block_params* p,
                                 const void* x, void* y, void* workspace, void* stream);
/* gy: gradient w.r.t. y; y: the forward output (for its ReLU mask). */
TSM_API tsm_status tsm_block_bwd(const tsm_block_desc* d, const tsm_block_params* p,
                                 const void* x, const void* y, const void* gy, void* gx,
                                 const tsm_block_grads* g, void* workspace, void* stream);

/* ---------------------------------------------------------------------------
 * TSM-ResNet-50 8-frame network and its data-parallel training step.
 *
 * Replaces vidperf::Network over build_tsm8f() (net.hpp:15-54; arch.cpp:
 * 140-161): conv1 7x7/s2 (+bias, linear) -> pool1 3x3/s2 -> res2..res5
 * bottleneck units {3,4,6,3} x {256,512,1024,2048} with the residual shift
 * -> global average pool -> fc.  loss = sum of squared logits (net.cpp:
 * 141-146); gradients are sums over the batch, so the data-parallel
 * allreduce is a SUM (equal to the full-batch reference gradient).
 *
 * Parameters: one flat fp32 device buffer in the reference declaration
 * order (net.cpp:63-75); each weight in the GEMM layout [c_out][kh][kw][c_in]
 * (conv1's 3 input channels zero-padded to 8).  tsm_net_param describes
 * each tensor so hosts can convert from/to the reference's (c_out, c_in, kt,
 * kh, kw).  The input x is the reference layout [N][T][3][H][W] on the device
 * (f32, f64 or bf16). */
/* Network presets (arch.cpp:140-161 build_tsm8f, 220-233 build_micro_tsm). */
enum {
  TSM_ARCH_TSM8F = 0,      /* TSM-ResNet-50, input (N, T, 3, H, W) */
  TSM_ARCH_MICRO_TSM = 1,  /* 2 bottlenecks of 16 channels, input (N, T, 8, H, W), no stem/pool */
};

typedef struct tsm_net_desc {
  int64_t batch;       /* clips per GPU */
  int64_t frames;      /* T (8; micro-tsm 4) */
  int64_t height, width;
  int64_t classes;     /* 400 (micro-tsm 4) */
  int64_t shift_num, shift_den; /* residual-shift fraction per direction (1/8); 0/1 disables */
  int64_t arch;        /* TSM_ARCH_* (ABI >= 3) */
} tsm_net_desc;

typedef struct tsm_net_param {
  int64_t offset;      /* first element in the flat buffer */
  int64_t numel;
  int64_t dims[4];     /* c_out, kh, kw, c_in (GEMM layout; biases c_out,1,1,1) */
  int64_t ci_ref;      /* input channels in the reference tensor (3 for conv1) */
  int32_t is_bias;
  char name[48];
} tsm_net_param;

typedef struct tsm_sgd {
  int32_t enabled;     /* 0: gradients only */
  float lr, momentum, weight_decay; /* decay on weights only, not biases */
  float grad_scale;    /* multiplies the (summed) gradient, e.g. 1/global_batch */
} tsm_sgd;

typedef struct tsm_net tsm_net;

TSM_API tsm_status tsm_net_create(const tsm_net_desc* d, tsm_net** out);
TSM_API void tsm_net_destroy(tsm_net* net);
TSM_API int64_t tsm_net_param_count(const tsm_net* net);
TSM_API int64_t tsm_net_param_tensors(const tsm_net* net);
TSM_API tsm_status tsm_net_param_info(const tsm_net* net, int64_t i, tsm_net_param* out);
/* Device pointers to the flat fp32 parameter / gradient buffers, the fp32
 * loss scalar and the fp32 logits [batch][classes] of the last forward.
 * Under data parallelism the loss is this rank's own Sigma y^2 over its
 * clips (the gradients, not the loss, are allreduced); NULL for a NULL
 * handle. */
TSM_API float* tsm_net_params(tsm_net* net);
TSM_API float* tsm_net_grads(tsm_net* net);
TSM_API float* tsm_net_loss(tsm_net* net);
TSM_API float* tsm_net_logits(tsm_net* net);
/* Network::forward (net.cpp:128-139); logits may be NULL. */
TSM_API tsm_status tsm_net_forward(tsm_net* net, const void* x, tsm_dtype dtype, float* logits,
                                   void* stream);
/* One training step: forward, loss, Network::loss_gradients' backward
 * (net.cpp:160-272), the bucketed NCCL gradient allreduce when dp is
 * initialised (overlapped with backward on a separate stream), and the SGD
 * update when opt->enabled. */
TSM_API tsm_status tsm_net_train_step(tsm_net* net, const void* x, tsm_dtype dtype,
                                      const tsm_sgd* opt, void* stream);
/* CUDA-graph mode (default off): tsm_net_train_step captures the whole step
 * (forward, loss, backward with its side-stream weight gradients, SGD) once
 * per (input pointer, dtype, opt->enabled) and replays it, with the SGD
 * hyperparameters of each call.  For launch-bound small batches (the step
 * is ~2,550 kernels).  Single-GPU only: with data parallelism, or while
 * tsm_probe_shift_conv1 records, the step runs eagerly. */
TSM_API tsm_status tsm_net_set_graph(tsm_net* net, int enable);

/* Reference-layout parameter exchange: `flat` is Network::param_vector()
 * (net.hpp:24; declaration order net.cpp:63-75), fp64 on the HOST, each conv
 * weight in ConvWeights layout (c_out, c_in, kt, kh, kw) (kernels.hpp:34-45),
 * fc weights (c_out, c_in).  The permutation to/from the flat GEMM layout
 * happens inside the library.  count must equal
 * tsm_net_reference_param_count(net) (24,301,072 for build_tsm8f, 772 for
 * build_micro_tsm).  Synchronous. */
TSM_API int64_t tsm_net_reference_param_count(const tsm_net* net);
TSM_API tsm_status tsm_net_set_params_reference(tsm_net* net, const double* flat, int64_t count);
TSM_API tsm_status tsm_net_get_params_reference(tsm_net* net, double* flat, int64_t count);
/* The gradients of the last tsm_net_train_step, same order and layout
 * (Gradients::params, net.hpp:38). */
TSM_API tsm_status tsm_net_get_grads_reference(tsm_net* net, double* flat, int64_t count);
/* dL/dx of the last tsm_net_train_step (Gradients::input, net.hpp:39): the
 * network input's shape [N][T][C][H][W], f32 or f64, device buffer, on
 * `stream`.  For build_tsm8f this is the stem conv's input gradient
 * (kernels.cpp:246-280); the training step itself never needs it. */
TSM_API tsm_status tsm_net_input_grad(tsm_net* net, void* gx, tsm_dtype dtype, void* stream);
/* Host-buffer calls with the reference's value semantics (x: fp64 NTCHW host
 * array of the network's input shape; results written to host arrays),
 * synchronous:
 *   tsm_net_forward_host         Network::forward (net.cpp:128-139): logits
 *                                [N][classes] (the reference's (N,1,classes,1,1))
 *   tsm_net_loss_gradients_host  Network::loss_gradients (net.cpp:160-272):
 *                                Sigma y^2, parameter gradients in reference
 *                                order/layout, and (if grad_input != NULL)
 *                                dL/dx; no parameter update. */
TSM_API tsm_status tsm_net_forward_host(tsm_net* net, const double* x, double* logits);
TSM_API tsm_status tsm_net_loss_gradients_host(tsm_net* net, const double* x, double* loss,
                                               double* grad_params, double* grad_input);

/* Data parallel: rank 0 calls tsm_nccl_unique_id and shares the 128 bytes
 * with every rank (e.g. via torch.distributed); each rank then calls
 * tsm_net_dp_init on its own device.  bucket_bytes 0 = 25 MiB.
 * Asynchronous NCCL errors (ncclCommGetAsyncError) are polled at dp_init
 * and at each train_step; on error the communicator is aborted and
 * TSM_ERR_NCCL is returned (then and for every later step). */
TSM_API tsm_status tsm_nccl_unique_id(void* out128);
TSM_API tsm_status tsm_net_dp_init(tsm_net* net, const void* id128, int rank, int world,
                                   size_t bucket_bytes);

/* Number of this library's kernels launched on this thread since process
 * start (a counter for bench.py's `gpu_launches`). */
TSM_API uint64_t tsm_launch_count(void);
/* Launch trace (measurement only, no reference counterpart): while enabled,
 * every kernel launch issued by this thread is recorded with the label of
 * the layer / op that issued it ("res4.2 bwd dgrad c3"), in issue order;
 * tsm_trace_dump writes one label per line.  Enabling clears the list.
 * Join it with a profiler launch list of a TSM_SIDE_STREAM=0 run
 * (tools/launch_labels.py). */
TSM_API tsm_status tsm_trace_enable(int on);
TSM_API tsm_status tsm_trace_dump(const char* path);

/* Measurement probe (no reference counterpart; bench.py's roofline leg):
 * while enabled, every fused shift + 1x1 conv forward launch inside a
 * bottleneck unit (conv1 with a temporal shift) whose channels are
 * c_in -> c_out is bracketed by CUDA events on its own stream (at most 256
 * launches).  c_in > 0 resets and starts recording, c_in == 0 stops.
 * tsm_probe_shift_conv1_read synchronises the events and returns the
 * launch count, the mean launch duration in µs and the pixels (rows) of
 * the recorded launches. */
TSM_API tsm_status tsm_probe_shift_conv1(int64_t c_in, int64_t c_out);
TSM_API tsm_status tsm_probe_shift_conv1_read(int* launches, double* mean_us, int64_t* pixels);

#ifdef __cplusplus
}
#endif
#endif /* TSM_B200_H */
