/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the TSM hot path.
 *
 * A plain-C restatement of the reference algorithm (vidperf, C++20/OpenMP,
 * fp64).  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it; the product path (libtsm_b200.so) never links it.
 *
 * Parity status: PINNED.  tests/test_oracle.py checks every function here
 * against (1) the unmodified reference compiled in place (oracle/_ref) and
 * (2) the golden vectors in tests/golden/ (the reference KATs of
 * kernels_test.cpp:41-100 and acceptance_test.cpp:115-166, plus FNV-1a
 * digests of the reference's own outputs at config C1).
 *
 * Layout everywhere: dense row-major [N][T][C][H][W] (tensor.hpp:42).
 * Conv weights: (c_out, c_in, kt, kh, kw) row-major, bias per c_out
 * (kernels.hpp:34-45).
 */
#ifndef TSM_ORACLE_H
#define TSM_ORACLE_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* tensor.cpp:41-55 — mt19937_64 + libstdc++ normal/uniform, flat order. */
void tso_random_normal(int64_t count, uint64_t seed, double stddev, double* out);
void tso_random_uniform(int64_t count, uint64_t seed, double lo, double hi, double* out);

/* 64-bit FNV-1a over raw bytes (golden digests). */
uint64_t tso_fnv1a64(const void* data, size_t len);

/* rational.cpp:10-61 + kernels.cpp:82-95.  Returns 0 and sets *fwd/*bwd to the
 * integral channel counts, or 1 (ValidationError) when a fraction is negative,
 * does not split `channels` evenly, or the two splits exceed `channels`. */
int tso_validate_shift(int64_t fwd_num, int64_t fwd_den, int64_t bwd_num, int64_t bwd_den,
                       int64_t channels, int64_t* fwd, int64_t* bwd);

/* kernels.cpp:97-125 (adjoint=0) and kernels.cpp:127-157 (adjoint=1), as a
 * bitwise copy of `elt`-byte elements: valid for f64, f32, bf16 alike because
 * the shift performs no arithmetic.  Out-of-range frames are +0.0 (all-zero
 * bytes).  x and out must not alias. */
void tso_shift_bytes(const void* x, void* out, int64_t n, int64_t t, int64_t c, int64_t hw,
                     int64_t fwd, int64_t bwd, int64_t elt, int adjoint);

/* kernels.cpp:162-231 — conv forward, fp64, bias first then ci, dt, dh, dw
 * ascending (the reference accumulation order).  k/s/p are (t,h,w). */
void tso_conv_forward(const double* x, const int64_t* shape, int64_t c_out, const int* k,
                      const int* s, const int* p, const double* w, const double* b, double* y,
                      int64_t* y_shape);

/* kernels.cpp:233-327 — dgrad (gather), wgrad (per co,ci), bias grad. */
void tso_conv_backward(const double* x, const int64_t* shape, int64_t c_out, const int* k,
                       const int* s, const int* p, const double* w, const double* gy, double* gx,
                       double* gw, double* gb);

/* One residual-shift bottleneck unit (arch.cpp:278-323 expansion; net.cpp:85-126
 * forward; net.cpp:184-248 backward for that unit).  w = {w1,b1,w2,b2,w3,b3,wp,bp}
 * (wp == NULL: identity skip).  gy == NULL: forward only.  Returns 1 on a bad
 * configuration (ValidationError), else 0. */
int tso_block(const double* x, const int64_t* shape, int64_t c_out, int stride, int64_t shift_num,
              int64_t shift_den, const double* const* w, double* y, int64_t* y_shape,
              const double* gy, double* gx, double* const* gw);

/* Same unit with bf16 storage emulation when bf16 != 0: activations (r1, r2,
 * skip, y) and gradients (g2, g1, projection dgrad, gx) are rounded to
 * bfloat16 where the GPU path stores them.  Test-only: sharpens GPU parity by
 * removing storage-rounding differences; bf16 == 0 is tso_block exactly. */
int tso_block_ex(const double* x, const int64_t* shape, int64_t c_out, int stride,
                 int64_t shift_num, int64_t shift_den, const double* const* w, double* y,
                 int64_t* y_shape, const double* gy, double* gx, double* const* gw, int bf16);

#ifdef __cplusplus
}
#endif
#endif
