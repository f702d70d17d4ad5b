/* TEST INFRASTRUCTURE ONLY — see tsm_oracle.h.  Every function cites the
 * reference file:line (under /root/reference/proj) whose behaviour it states. */
#include "tsm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* RNG: std::mt19937_64 (the standard's 64-bit Mersenne twister) and the
 * libstdc++ algorithms behind std::normal_distribution<double> (Marsaglia
 * polar method with one cached deviate) and std::uniform_real_distribution,
 * both fed through std::generate_canonical<double, 53> which, for a 2^64-range
 * engine, is one draw divided by 2^64 (clamped below 1).  tensor.cpp:41-55
 * constructs a fresh engine+distribution per tensor and draws in flat order. */

typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
    for (int i = 0; i < 312; ++i) {
      uint64_t y = (g->mt[i] & upper) | (g->mt[(i + 1) % 312] & lower);
      uint64_t v = g->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = v;
    }
    g->idx = 0;
  }
  uint64_t z = g->mt[g->idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= z >> 43;
  return z;
}

static double canonical(mt64* g) {
  double r = (double)mt64_next(g) / 18446744073709551616.0; /* 2^64 */
  if (r >= 1.0) r = nextafter(1.0, 0.0);
  return r;
}

void tso_random_normal(int64_t count, uint64_t seed, double stddev, double* out) {
  mt64 g;
  mt64_seed(&g, seed);
  int have_saved = 0;
  double saved = 0.0;
  for (int64_t i = 0; i < count; ++i) {
    double v;
    if (have_saved) {
      have_saved = 0;
      v = saved;
    } else {
      double x, y, r2;
      do {
        x = 2.0 * canonical(&g) - 1.0;
        y = 2.0 * canonical(&g) - 1.0;
        r2 = x * x + y * y;
      } while (r2 > 1.0 || r2 == 0.0);
      double mult = sqrt(-2.0 * log(r2) / r2);
      saved = x * mult;
      have_saved = 1;
      v = y * mult;
    }
    out[i] = v * stddev + 0.0;
  }
}

void tso_random_uniform(int64_t count, uint64_t seed, double lo, double hi, double* out) {
  mt64 g;
  mt64_seed(&g, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = canonical(&g) * (hi - lo) + lo;
}

uint64_t tso_fnv1a64(const void* data, size_t len) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 0xcbf29ce484222325ULL;
  for (size_t i = 0; i < len; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* ------------------------------------------------------------------------ */
/* Channel split.  Rational normalisation (rational.cpp:10-23) divides by the
 * gcd and moves the sign to the numerator; exact_multiple (rational.cpp:50-57)
 * throws unless num*count is divisible by den; validate_shift
 * (kernels.cpp:82-95) rejects negative fractions and fwd+bwd > channels. */

static int64_t gcd64(int64_t a, int64_t b) {
  if (a < 0) a = -a;
  while (b) {
    int64_t t = a % b;
    a = b;
    b = t;
  }
  return a;
}

static int normalise(int64_t* num, int64_t* den) {
  if (*den == 0) return 1;
  if (*den < 0) {
    *num = -*num;
    *den = -*den;
  }
  if (*num == 0) {
    *den = 1;
    return 0;
  }
  int64_t g = gcd64(*num, *den);
  *num /= g;
  *den /= g;
  return 0;
}

int tso_validate_shift(int64_t fn, int64_t fd, int64_t bn, int64_t bd, int64_t channels,
                       int64_t* fwd, int64_t* bwd) {
  if (normalise(&fn, &fd) || normalise(&bn, &bd)) return 1;
  if (fn < 0 || bn < 0) return 1;
  if ((fn * channels) % fd != 0 || (bn * channels) % bd != 0) return 1;
  int64_t f = fn * channels / fd, b = bn * channels / bd;
  if (f + b > channels) return 1;
  if (fwd) *fwd = f;
  if (bwd) *bwd = b;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Shift (kernels.cpp:97-125) and its adjoint (kernels.cpp:127-157).  The
 * output starts all-zero (Tensor5D ctor, tensor.cpp:16-22) and each (n,t,c)
 * plane is either copied from its source frame or left zero. */

void tso_shift_bytes(const void* x, void* out, int64_t n, int64_t t, int64_t c, int64_t hw,
                     int64_t fwd, int64_t bwd, int64_t elt, int adjoint) {
  const unsigned char* src = (const unsigned char*)x;
  unsigned char* dst = (unsigned char*)out;
  const int64_t plane = hw * elt;
  for (int64_t in = 0; in < n; ++in)
    for (int64_t it = 0; it < t; ++it)
      for (int64_t ic = 0; ic < c; ++ic) {
        int64_t st;
        if (ic < fwd) st = adjoint ? it + 1 : it - 1;
        else if (ic < fwd + bwd) st = adjoint ? it - 1 : it + 1;
        else st = it;
        unsigned char* d = dst + ((in * t + it) * c + ic) * plane;
        if (st < 0 || st >= t) {
          memset(d, 0, (size_t)plane);
          continue;
        }
        memcpy(d, src + ((in * t + st) * c + ic) * plane, (size_t)plane);
      }
}

/* ------------------------------------------------------------------------ */
/* Convolution, fp64.  Output extent (n + 2p - k)/s + 1 (arch.cpp:348-360).
 * Forward accumulates bias, then ci, dt, dh, dw ascending, skipping padded
 * taps (kernels.cpp:181-193, 208-224).  Backward: dgrad gathers over
 * (co, dt, dh, dw) with stride divisibility (kernels.cpp:246-280); wgrad sums
 * over (n, to, ho, wo) per (co, ci, dt, dh, dw) (kernels.cpp:282-310); bias
 * grad sums grad_out (kernels.cpp:312-325). */

static int64_t extent(int64_t n, int k, int s, int p) { return (n + 2 * p - k) / s + 1; }

#define IDX5(a, b, c_, d, e, B, C, D, E) ((((((a) * (B) + (b)) * (C) + (c_)) * (D) + (d)) * (E)) + (e))

void tso_conv_forward(const double* x, const int64_t* sh, int64_t c_out, const int* k,
                      const int* s, const int* p, const double* w, const double* b, double* y,
                      int64_t* ys) {
  const int64_t N = sh[0], T = sh[1], C = sh[2], H = sh[3], W = sh[4];
  const int64_t To = extent(T, k[0], s[0], p[0]), Ho = extent(H, k[1], s[1], p[1]),
                Wo = extent(W, k[2], s[2], p[2]);
  ys[0] = N; ys[1] = To; ys[2] = c_out; ys[3] = Ho; ys[4] = Wo;
  if (!y) return;
#pragma omp parallel for collapse(3)
  for (int64_t n = 0; n < N; ++n)
    for (int64_t to = 0; to < To; ++to)
      for (int64_t co = 0; co < c_out; ++co)
        for (int64_t ho = 0; ho < Ho; ++ho)
          for (int64_t wo = 0; wo < Wo; ++wo) {
            double acc = b[co];
            for (int64_t ci = 0; ci < C; ++ci)
              for (int dt = 0; dt < k[0]; ++dt) {
                int64_t ti = to * s[0] - p[0] + dt;
                if (ti < 0 || ti >= T) continue;
                for (int dh = 0; dh < k[1]; ++dh) {
                  int64_t hi = ho * s[1] - p[1] + dh;
                  if (hi < 0 || hi >= H) continue;
                  for (int dw = 0; dw < k[2]; ++dw) {
                    int64_t wi = wo * s[2] - p[2] + dw;
                    if (wi < 0 || wi >= W) continue;
                    acc += x[IDX5(n, ti, ci, hi, wi, T, C, H, W)] *
                           w[IDX5(co, ci, dt, dh, dw, C, k[0], k[1], k[2])];
                  }
                }
              }
            y[IDX5(n, to, co, ho, wo, To, c_out, Ho, Wo)] = acc;
          }
}

void tso_conv_backward(const double* x, const int64_t* sh, int64_t c_out, const int* k,
                       const int* s, const int* p, const double* w, const double* gy, double* gx,
                       double* gw, double* gb) {
  const int64_t N = sh[0], T = sh[1], C = sh[2], H = sh[3], W = sh[4];
  const int64_t To = extent(T, k[0], s[0], p[0]), Ho = extent(H, k[1], s[1], p[1]),
                Wo = extent(W, k[2], s[2], p[2]);
#pragma omp parallel for collapse(3)
  for (int64_t n = 0; n < N; ++n)
    for (int64_t ti = 0; ti < T; ++ti)
      for (int64_t ci = 0; ci < C; ++ci)
        for (int64_t hi = 0; hi < H; ++hi)
          for (int64_t wi = 0; wi < W; ++wi) {
            double acc = 0.0;
            for (int64_t co = 0; co < c_out; ++co)
              for (int dt = 0; dt < k[0]; ++dt) {
                int64_t tn = ti + p[0] - dt;
                if (tn < 0 || tn % s[0]) continue;
                int64_t to = tn / s[0];
                if (to >= To) continue;
                for (int dh = 0; dh < k[1]; ++dh) {
                  int64_t hn = hi + p[1] - dh;
                  if (hn < 0 || hn % s[1]) continue;
                  int64_t ho = hn / s[1];
                  if (ho >= Ho) continue;
                  for (int dw = 0; dw < k[2]; ++dw) {
                    int64_t wn = wi + p[2] - dw;
                    if (wn < 0 || wn % s[2]) continue;
                    int64_t wo = wn / s[2];
                    if (wo >= Wo) continue;
                    acc += gy[IDX5(n, to, co, ho, wo, To, c_out, Ho, Wo)] *
                           w[IDX5(co, ci, dt, dh, dw, C, k[0], k[1], k[2])];
                  }
                }
              }
            gx[IDX5(n, ti, ci, hi, wi, T, C, H, W)] = acc;
          }
#pragma omp parallel for collapse(2)
  for (int64_t co = 0; co < c_out; ++co)
    for (int64_t ci = 0; ci < C; ++ci)
      for (int dt = 0; dt < k[0]; ++dt)
        for (int dh = 0; dh < k[1]; ++dh)
          for (int dw = 0; dw < k[2]; ++dw) {
            double acc = 0.0;
            for (int64_t n = 0; n < N; ++n)
              for (int64_t to = 0; to < To; ++to) {
                int64_t ti = to * s[0] - p[0] + dt;
                if (ti < 0 || ti >= T) continue;
                for (int64_t ho = 0; ho < Ho; ++ho) {
                  int64_t hi = ho * s[1] - p[1] + dh;
                  if (hi < 0 || hi >= H) continue;
                  for (int64_t wo = 0; wo < Wo; ++wo) {
                    int64_t wi = wo * s[2] - p[2] + dw;
                    if (wi < 0 || wi >= W) continue;
                    acc += gy[IDX5(n, to, co, ho, wo, To, c_out, Ho, Wo)] *
                           x[IDX5(n, ti, ci, hi, wi, T, C, H, W)];
                  }
                }
              }
            gw[IDX5(co, ci, dt, dh, dw, C, k[0], k[1], k[2])] = acc;
          }
#pragma omp parallel for
  for (int64_t co = 0; co < c_out; ++co) {
    double acc = 0.0;
    for (int64_t n = 0; n < N; ++n)
      for (int64_t to = 0; to < To; ++to)
        for (int64_t ho = 0; ho < Ho; ++ho)
          for (int64_t wo = 0; wo < Wo; ++wo) acc += gy[IDX5(n, to, co, ho, wo, To, c_out, Ho, Wo)];
    gb[co] = acc;
  }
}

/* ------------------------------------------------------------------------ */
/* Bottleneck unit.  expand_layer (arch.cpp:278-323): [shift(frac) if frac != 0,
 * 1x1 c_in->C/4 +ReLU, 1x3x3 stride s pad 1 +ReLU, 1x1 C/4->C]; projection
 * 1x1 stride s iff strided or c_in != C; residual.  Forward order and the
 * unshifted skip follow run_unit (net.cpp:85-126); backward follows
 * loss_gradients for one unit (net.cpp:190-247).  ReLU: max(x,0) and
 * g*[x>0] (kernels.cpp:578-596). */

/* bf16 storage emulation (test-only knob, not part of the reference): round
 * through fp32 to bfloat16 (round-to-nearest-even), as the GPU path stores
 * activations and gradients between GEMMs. */
static double bf16r(double v) {
  float f = (float)v;
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7f800000u) != 0x7f800000u) u += 0x7fffu + ((u >> 16) & 1u);
  u &= 0xffff0000u;
  memcpy(&f, &u, 4);
  return (double)f;
}
static void round_all(double* a, int64_t n, int on) {
  if (!on) return;
  for (int64_t i = 0; i < n; ++i) a[i] = bf16r(a[i]);
}

static void relu_f(const double* a, double* o, int64_t n) {
  for (int64_t i = 0; i < n; ++i) o[i] = a[i] > 0.0 ? a[i] : 0.0;
}
static void relu_b(const double* pre, const double* g, double* o, int64_t n) {
  for (int64_t i = 0; i < n; ++i) o[i] = pre[i] > 0.0 ? g[i] : 0.0;
}
static int64_t numel(const int64_t* s) { return s[0] * s[1] * s[2] * s[3] * s[4]; }

int tso_block(const double* x, const int64_t* sh, int64_t c_out, int stride, int64_t shift_num,
              int64_t shift_den, const double* const* wts, double* y, int64_t* y_shape,
              const double* gy, double* gx, double* const* gw) {
  return tso_block_ex(x, sh, c_out, stride, shift_num, shift_den, wts, y, y_shape, gy, gx, gw, 0);
}

int tso_block_ex(const double* x, const int64_t* sh, int64_t c_out, int stride,
                 int64_t shift_num, int64_t shift_den, const double* const* wts, double* y,
                 int64_t* y_shape, const double* gy, double* gx, double* const* gw, int bf16) {
  if (c_out <= 0 || c_out % 4 != 0) return 1;
  const int64_t width = c_out / 4, cin = sh[2];
  int64_t F = 0, B = 0;
  int has_shift = shift_num != 0;
  if (has_shift && tso_validate_shift(shift_num, shift_den, shift_num, shift_den, cin, &F, &B))
    return 1;
  int has_proj = stride != 1 || cin != c_out;
  if (has_proj != (wts[6] != NULL)) return 1;

  const int k1[3] = {1, 1, 1}, s1[3] = {1, 1, 1}, p0[3] = {0, 0, 0};
  const int k3[3] = {1, 3, 3}, ss[3] = {1, stride, stride}, p1[3] = {0, 1, 1};
  const int64_t nx = numel(sh);

  double* xs = (double*)malloc(sizeof(double) * nx);
  if (has_shift) tso_shift_bytes(x, xs, sh[0], sh[1], cin, sh[3] * sh[4], F, B, 8, 0);
  else memcpy(xs, x, sizeof(double) * nx);

  int64_t s1s[5], s2s[5], s3s[5];
  tso_conv_forward(xs, sh, width, k1, s1, p0, wts[0], wts[1], NULL, s1s);
  double* a1 = (double*)malloc(sizeof(double) * numel(s1s));
  double* r1 = (double*)malloc(sizeof(double) * numel(s1s));
  tso_conv_forward(xs, sh, width, k1, s1, p0, wts[0], wts[1], a1, s1s);
  relu_f(a1, r1, numel(s1s));
  round_all(r1, numel(s1s), bf16);
  tso_conv_forward(r1, s1s, width, k3, ss, p1, wts[2], wts[3], NULL, s2s);
  double* a2 = (double*)malloc(sizeof(double) * numel(s2s));
  double* r2 = (double*)malloc(sizeof(double) * numel(s2s));
  tso_conv_forward(r1, s1s, width, k3, ss, p1, wts[2], wts[3], a2, s2s);
  relu_f(a2, r2, numel(s2s));
  round_all(r2, numel(s2s), bf16);
  tso_conv_forward(r2, s2s, c_out, k1, s1, p0, wts[4], wts[5], NULL, s3s);
  const int64_t ny = numel(s3s);
  double* pre = (double*)malloc(sizeof(double) * ny);
  tso_conv_forward(r2, s2s, c_out, k1, s1, p0, wts[4], wts[5], pre, s3s);
  if (has_proj) {
    double* sk = (double*)malloc(sizeof(double) * ny);
    int64_t tmp[5];
    tso_conv_forward(x, sh, c_out, k1, ss, p0, wts[6], wts[7], sk, tmp);
    round_all(sk, ny, bf16);
    for (int64_t i = 0; i < ny; ++i) pre[i] += sk[i];
    free(sk);
  } else {
    for (int64_t i = 0; i < ny; ++i) pre[i] += x[i];
  }
  memcpy(y_shape, s3s, sizeof s3s);
  if (y) {
    relu_f(pre, y, ny);
    round_all(y, ny, bf16);
  }

  if (gy) {
    double* g = (double*)malloc(sizeof(double) * ny);
    relu_b(pre, gy, g, ny); /* g is also the skip gradient */
    double* g2 = (double*)malloc(sizeof(double) * numel(s2s));
    tso_conv_backward(r2, s2s, c_out, k1, s1, p0, wts[4], g, g2, gw[4], gw[5]);
    relu_b(a2, g2, g2, numel(s2s));
    round_all(g2, numel(s2s), bf16);
    double* g1 = (double*)malloc(sizeof(double) * numel(s1s));
    tso_conv_backward(r1, s1s, width, k3, ss, p1, wts[2], g2, g1, gw[2], gw[3]);
    relu_b(a1, g1, g1, numel(s1s));
    round_all(g1, numel(s1s), bf16);
    double* g0 = (double*)malloc(sizeof(double) * nx);
    tso_conv_backward(xs, sh, width, k1, s1, p0, wts[0], g1, g0, gw[0], gw[1]);
    if (has_shift) tso_shift_bytes(g0, gx, sh[0], sh[1], cin, sh[3] * sh[4], F, B, 8, 1);
    else memcpy(gx, g0, sizeof(double) * nx);
    if (has_proj) {
      double* gp = (double*)malloc(sizeof(double) * nx);
      tso_conv_backward(x, sh, c_out, k1, ss, p0, wts[6], g, gp, gw[6], gw[7]);
      round_all(gp, nx, bf16);
      for (int64_t i = 0; i < nx; ++i) gx[i] += gp[i];
      free(gp);
    } else {
      for (int64_t i = 0; i < nx; ++i) gx[i] += g[i];
    }
    round_all(gx, nx, bf16);
    free(g); free(g2); free(g1); free(g0);
  }
  free(xs); free(a1); free(r1); free(a2); free(r2); free(pre);
  return 0;
}
