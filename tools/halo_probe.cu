// Probe: can a tcgen05 operand start at an arbitrary 128-byte row of a
// 128B-swizzled smem tile, with an 8-row-group stride (SBO) that is not a
// multiple of 1024?  (Needed for halo-tile 3x3 convolutions: every tap is a
// descriptor offset into one loaded pixel tile.)  Single CTA, exact integer
// data; prints the mismatch count per (case, base-offset mode, tap).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O2 \
//        -I paper_1910_00932_b200/csrc tools/halo_probe.cu -o /tmp/halo_probe -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc_common.cuh"

using namespace tsm;

constexpr int P = 10;        // halo pitch (pixels per halo row)
constexpr int HROWS = 18;    // halo rows
constexpr int NPIX = P * HROWS;

// case 0: K-major A (forward): rows m = i*8 + j (i < 16, j < 8) read pixel
//         (i + r) * P + (j + s); K = 64 channels.  B K-major [64 n][64 k].
// case 2: K-major A, SW32, 16 channels (32 B pixel rows), halo pitch 11:
//         rows m = i*8 + j read pixel (i + r) * 11 + (j + s); K = 16 (one
//         MMA k-step per tap).  B K-major [64 n][16 k] SW32.
// case 1: MN-major A (weight gradient): K-row k = i*8 + j (i, j < 8) reads
//         pixel (i + r) * P + (j + s); M = 2 slabs of 64 channels (tap pair
//         (r, s), (r, s+1): LBO = 128 B).  B MN-major [64 k][64 n] dense.
__global__ void probe(const __nv_bfloat16* ga, const __nv_bfloat16* gb, float* gd, int kase,
                      int mode, int r, int s) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = sm;                      // NPIX rows x 128 B
  uint8_t* sb = sm + 24 * 1024;          // 64 rows x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  if (kase == 2) {
    // SW32: 32 B rows, 16 B chunk c of row p at c ^ ((p >> 2) & 1)
    for (int i = tid; i < 19 * 11 * 2; i += blockDim.x) {
      const int p = i / 2, c = i % 2;
      *reinterpret_cast<uint4*>(sa + p * 32 + ((c ^ ((p >> 2) & 1)) << 4)) =
          reinterpret_cast<const uint4*>(ga)[i];
    }
    for (int i = tid; i < 64 * 2; i += blockDim.x) {
      const int p = i / 2, c = i % 2;
      *reinterpret_cast<uint4*>(sb + p * 32 + ((c ^ ((p >> 2) & 1)) << 4)) =
          reinterpret_cast<const uint4*>(gb)[i];
    }
  } else {
  // swizzled fill (absolute-address pattern: base is 1024-aligned)
  for (int i = tid; i < NPIX * 8; i += blockDim.x) {
    const int p = i / 8, c = i % 8;
    *reinterpret_cast<uint4*>(sa + p * 128 + ((c ^ (p & 7)) << 4)) =
        reinterpret_cast<const uint4*>(ga)[i];
  }
  for (int i = tid; i < 64 * 8; i += blockDim.x) {
    const int p = i / 8, c = i % 8;
    *reinterpret_cast<uint4*>(sb + p * 128 + ((c ^ (p & 7)) << 4)) =
        reinterpret_cast<const uint4*>(gb)[i];
  }
  }
  tc::fence_proxy_async();
  if (tid == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  if (tc::warp_id() == 0) tc::tmem_alloc<128>(&tslot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  const uint32_t a0 = tc::smem_u32(sa), b0 = tc::smem_u32(sb);
  if (tc::warp_id() == 0 && tc::elect_one()) {
    const uint32_t idesc = tc::idesc_bf16(128, 64, kase == 1, kase == 1);
    if (kase == 2) {
      const uint64_t ad = tc::smem_desc(a0 + (r * 11 + s) * 32, 16, 11 * 32, tc::kSw32);
      const uint64_t bd = tc::smem_desc(b0, 16, 256, tc::kSw32);
      tc::mma_bf16(tmem, ad, bd, idesc, 0u);
    } else
    for (int j = 0; j < 4; ++j) {
      uint32_t aaddr, lbo, sbo;
      if (kase == 0) {
        aaddr = a0 + (r * P + s) * 128 + j * 32;
        lbo = 16;
        sbo = P * 128;
      } else {
        aaddr = a0 + ((2 * j + r) * P + s) * 128;
        lbo = 128;  // next slab = tap (r, s+1): one pixel row further
        sbo = P * 128;
      }
      uint64_t ad = tc::smem_desc(aaddr, lbo, sbo, tc::kSw128);
      if (mode == 1) ad |= (uint64_t)((aaddr >> 7) & 7) << 49;
      uint64_t bd = kase == 0 ? tc::smem_desc(b0 + j * 32, 16, 1024, tc::kSw128)
                              : tc::smem_desc(b0 + j * 16 * 128, 8192, 1024, tc::kSw128);
      tc::mma_bf16(tmem, ad, bd, idesc, j > 0);
    }
    tc::mma_commit(&bar);
  }
  __syncwarp();
  tc::mbar_wait(&bar, 0);
  tc::tc_fence_after();
  const int q = tc::warp_id();
  for (int c0 = 0; c0 < 64; c0 += 16) {
    uint32_t v[16];
    tc::tmem_ld_32x32b_x16(tmem + ((uint32_t)(q * 32) << 16) + c0, v);
    tc::tmem_ld_wait();
    for (int i = 0; i < 16; ++i) gd[(q * 32 + tc::lane_id()) * 64 + c0 + i] = __uint_as_float(v[i]);
  }
  tc::tc_fence_before();
  __syncthreads();
  if (tc::warp_id() == 0) tc::tmem_dealloc<128>(tmem);
}

int main() {
  std::vector<__nv_bfloat16> ha(NPIX * 64), hb(64 * 64);
  std::vector<float> fa(NPIX * 64), fb(64 * 64);
  srand(1);
  for (int i = 0; i < NPIX * 64; ++i) { fa[i] = (float)(rand() % 9 - 4); ha[i] = __float2bfloat16(fa[i]); }
  for (int i = 0; i < 64 * 64; ++i) { fb[i] = (float)(rand() % 9 - 4); hb[i] = __float2bfloat16(fb[i]); }
  __nv_bfloat16 *da, *db;
  float* dd;
  cudaMalloc(&da, ha.size() * 2);
  cudaMalloc(&db, hb.size() * 2);
  cudaMalloc(&dd, 128 * 64 * 4);
  cudaMemcpy(da, ha.data(), ha.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb.data(), hb.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  std::vector<float> hd(128 * 64);
  for (int kase = 0; kase < 3; ++kase)
    for (int mode = 0; mode < (kase == 2 ? 1 : 2); ++mode)
      for (int r = 0; r < (kase == 2 ? 4 : 3); ++r)
        for (int s = 0; s < (kase == 0 ? 3 : kase == 2 ? 4 : 2); ++s) {
          cudaMemset(dd, 0xff, 128 * 64 * 4);
          probe<<<1, 128, 64 * 1024>>>(da, db, dd, kase, mode, r, s);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) { printf("kase %d mode %d r %d s %d: %s\n", kase, mode, r, s, cudaGetErrorString(e)); return 1; }
          cudaMemcpy(hd.data(), dd, hd.size() * 4, cudaMemcpyDeviceToHost);
          int bad = 0;
          for (int m = 0; m < 128; ++m)
            for (int n = 0; n < 64; ++n) {
              double ref = 0;
              if (kase == 2) {
                const int i = m / 8, j = m % 8, pix = (i + r) * 11 + j + s;
                for (int k = 0; k < 16; ++k) ref += fa[pix * 16 + k] * fb[n * 16 + k];
              } else if (kase == 0) {
                const int i = m / 8, j = m % 8, pix = (i + r) * P + j + s;
                for (int k = 0; k < 64; ++k) ref += fa[pix * 64 + k] * fb[n * 64 + k];
              } else {
                // M row m: slab m/64 = tap (r, s + m/64), channel m%64
                const int sl = m / 64, ch = m % 64;
                for (int k = 0; k < 64; ++k) {
                  const int i = k / 8, j = k % 8, pix = (i + r) * P + j + s + sl;
                  ref += fa[pix * 64 + ch] * fb[k * 64 + n];
                }
              }
              if (hd[m * 64 + n] != (float)ref) ++bad;
            }
          printf("case %s mode %d (base_offset %s) tap (%d,%d): %d / 8192 mismatches\n",
                 kase == 0 ? "K-major " : kase == 2 ? "K-SW32  " : "MN-major", mode, mode ? "addr" : "0   ", r, s, bad);
        }
  return 0;
}
