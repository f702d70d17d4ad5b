// Max-pool backward helpers shared by the pool kernels and the fused stem
// weight gradient: the 2x2-block gather of maxpool_bwd2x2 (each input pixel
// sums the gradients of the windows whose recorded argmax tap it is, in
// ascending window order).
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

namespace tsm {
namespace poolbwd {

// acc[0..7] += the gradient g (8 bf16) of a window whose argmax bytes a are
// `tap` (channels that picked another tap add +0.0)
__device__ __forceinline__ void add_tap(float (&acc)[8], uint2 a, uint4 g, uint32_t tap) {
  const uint32_t t4 = tap * 0x01010101u;
  const uint32_t m0 = __vcmpeq4(a.x, t4), m1 = __vcmpeq4(a.y, t4);  // 0xFF per equal byte
  const uint32_t w[4] = {g.x & __byte_perm(m0, 0, 0x1100), g.y & __byte_perm(m0, 0, 0x3322),
                         g.z & __byte_perm(m1, 0, 0x1100), g.w & __byte_perm(m1, 0, 0x3322)};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    acc[2 * k] += __uint_as_float(w[k] << 16);
    acc[2 * k + 1] += __uint_as_float(w[k] & 0xFFFF0000u);
  }
}

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ uint4 pack8(const float (&a)[8]) {
  return make_uint4(pack2(a[0], a[1]), pack2(a[2], a[3]), pack2(a[4], a[5]), pack2(a[6], a[7]));
}

// The windows of one 2 x 2 block, loaded (so a caller can keep the next
// block's loads in flight while it writes this one's result).
struct Block2x2 {
  uint2 a00, a01, a10, a11;
  uint4 g00, g01, g10, g11;
  bool right, down;
};

__device__ __forceinline__ Block2x2 load2x2(const uint4* __restrict__ gy,
                                            const uint2* __restrict__ arg, int64_t row, int b,
                                            int c, int C8, int Wo, bool down) {
  Block2x2 k;
  k.right = b + 1 < Wo;
  k.down = down;
  const int64_t o00 = row + (int64_t)b * C8 + c;
  k.a00 = __ldg(arg + o00);
  k.g00 = __ldg(gy + o00);
  k.a01 = k.a10 = k.a11 = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);  // no tap matches
  k.g01 = k.g10 = k.g11 = make_uint4(0, 0, 0, 0);
  if (k.right) {
    k.a01 = __ldg(arg + o00 + C8);
    k.g01 = __ldg(gy + o00 + C8);
  }
  if (down) {
    const int64_t o10 = o00 + (int64_t)Wo * C8;
    k.a10 = __ldg(arg + o10);
    k.g10 = __ldg(gy + o10);
    if (k.right) {
      k.a11 = __ldg(arg + o10 + C8);
      k.g11 = __ldg(gy + o10 + C8);
    }
  }
  return k;
}

__device__ __forceinline__ void route2x2(const Block2x2& k, uint4 (&out)[4]) {
  float p00[8] = {0, 0, 0, 0, 0, 0, 0, 0}, p01[8] = {0, 0, 0, 0, 0, 0, 0, 0},
        p10[8] = {0, 0, 0, 0, 0, 0, 0, 0}, p11[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  add_tap(p00, k.a00, k.g00, 4);
  add_tap(p01, k.a00, k.g00, 5);
  if (k.right) add_tap(p01, k.a01, k.g01, 3);
  add_tap(p10, k.a00, k.g00, 7);
  if (k.down) add_tap(p10, k.a10, k.g10, 1);
  add_tap(p11, k.a00, k.g00, 8);
  if (k.right) add_tap(p11, k.a01, k.g01, 6);
  if (k.down) add_tap(p11, k.a10, k.g10, 2);
  if (k.down && k.right) add_tap(p11, k.a11, k.g11, 0);
  out[0] = pack8(p00);
  out[1] = pack8(p01);
  out[2] = pack8(p10);
  out[3] = pack8(p11);
}

// The four pixels of input block (2a..2a+1, 2b..2b+1) x 8 channels (chunk c
// of C8): windows (a + da, b + db) that exist, taps routed as
//   (0,0) <- w00:4                 (0,1) <- w00:5, w01:3
//   (1,0) <- w00:7, w10:1          (1,1) <- w00:8, w01:6, w10:2, w11:0
// gy / arg rows of window row a start at `row` (= (f Ho + a) Wo C8).
__device__ __forceinline__ void block2x2(const uint4* __restrict__ gy,
                                         const uint2* __restrict__ arg, int64_t row, int b,
                                         int c, int C8, int Wo, bool down, uint4 (&out)[4]) {
  const bool right = b + 1 < Wo;
  const int64_t o00 = row + (int64_t)b * C8 + c;
  const uint2 a00 = __ldg(arg + o00);
  const uint4 g00 = __ldg(gy + o00);
  uint2 a01 = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu), a10 = a01, a11 = a01;  // no tap matches
  uint4 g01 = make_uint4(0, 0, 0, 0), g10 = g01, g11 = g01;
  if (right) {
    a01 = __ldg(arg + o00 + C8);
    g01 = __ldg(gy + o00 + C8);
  }
  if (down) {
    const int64_t o10 = o00 + (int64_t)Wo * C8;
    a10 = __ldg(arg + o10);
    g10 = __ldg(gy + o10);
    if (right) {
      a11 = __ldg(arg + o10 + C8);
      g11 = __ldg(gy + o10 + C8);
    }
  }
  float p00[8] = {0, 0, 0, 0, 0, 0, 0, 0}, p01[8] = {0, 0, 0, 0, 0, 0, 0, 0},
        p10[8] = {0, 0, 0, 0, 0, 0, 0, 0}, p11[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  add_tap(p00, a00, g00, 4);
  add_tap(p01, a00, g00, 5);
  if (right) add_tap(p01, a01, g01, 3);
  add_tap(p10, a00, g00, 7);
  if (down) add_tap(p10, a10, g10, 1);
  add_tap(p11, a00, g00, 8);
  if (right) add_tap(p11, a01, g01, 6);
  if (down) add_tap(p11, a10, g10, 2);
  if (down && right) add_tap(p11, a11, g11, 0);
  out[0] = pack8(p00);
  out[1] = pack8(p01);
  out[2] = pack8(p10);
  out[3] = pack8(p11);
}

}  // namespace poolbwd
}  // namespace tsm
