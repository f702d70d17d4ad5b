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
 * bf16 [c_out][kh][kw][c_in]; biases fp32 [c_out].  tsm_layout_* convert
 * from/to the reference's NTCHW.
 *
 * Fused shift + 1x1 conv (north-star (b); the first two ops of the unit that
 * expand_layer builds, arch.cpp:291-302, executed by run_unit net.cpp:97-99
 * then conv_forward kernels.cpp:171-200):
 *     y = act( conv1x1( temporal_shift(x, F, B) ) + bias (+ residual) )
 * The shift is applied inside the TMA loads (channel groups [0,F) / [F,F+B)
 * fetched at frame t-1 / t+1; out-of-clip frames zero-filled by TMA), so the
 * shifted tensor is never written.  F = B = 0 gives a plain 1x1 conv.
 * act = ReLU when relu != 0 (applied after the residual add when residual is
 * given, as in run_unit's relu(add(main, skip)), net.cpp:119-124).
 * Requirements: c_in % 64 == 0, c_out % 16 == 0, F and F+B multiples of 8. */
TSM_API tsm_status tsm_conv1x1_fwd(const void* x, const void* w, const float* bias,
                                   const void* residual, void* y, int64_t n, int64_t t,
                                   int64_t h, int64_t w_, int64_t c_in, int64_t c_out,
                                   int64_t fold_fwd, int64_t fold_bwd, int relu, void* stream);

/* Number of this library's kernels launched on this thread since process
 * start (a counter for bench.py's `gpu_launches`). */
TSM_API uint64_t tsm_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* TSM_B200_H */
