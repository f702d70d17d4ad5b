// Probe: tcgen05.mma issue rate from shared memory for the operand layouts
// the conv engine uses — K-major A/B (forward, dgrad) against MN-major A/B
// (weight gradients) — with no loads in the loop (the data are whatever the
// smem holds; only the rate matters).  One CTA per SM, 4 (or 8) MMAs per
// commit as in tc_gemm.cuh, M = 128, N = 256, bf16 -> fp32.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O2 \
//        -I paper_1910_00932_b200/csrc tools/mma_rate_probe.cu -o /tmp/mma_rate_probe
//   /tmp/mma_rate_probe        # prints cycles per MMA (N = 256: 128 is the tensor floor)
#include <cstdio>

#include "tc_common.cuh"

using namespace tsm;

template <bool MN>
__global__ void __launch_bounds__(128, 1) rate(int iters, int per_commit, long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (tc::smem_u32(raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tslot;
  const uint32_t a = tc::smem_u32(sm), b = a + 16 * 1024;  // A [128 x 64] 16 KB, B [256 x 64] 32 KB
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  if (tc::warp_id() == 0) tc::tmem_alloc<256>(&tslot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  constexpr uint32_t idesc = tc::idesc_bf16(128, 256, MN, MN);
  long long t0 = 0, t1 = 0;
  if (tc::warp_id() == 0) {
    uint32_t phase = 0;
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (tc::elect_one()) {
        for (int j = 0; j < per_commit; ++j) {
          const int q = j & 3;
          uint64_t ad, bd;
          if (MN) {
            // MN-major SW128: slabs of 64 MN x 64 K rows (8 KB), k-step q = 16 K rows
            ad = tc::smem_desc(a + q * 16 * 128, 8192, 1024, tc::kSw128);
            bd = tc::smem_desc(b + q * 16 * 128, 8192, 1024, tc::kSw128);
          } else {
            // K-major SW128: rows of 64 K, k-step q = 32 bytes
            ad = tc::smem_desc(a + q * 32, 16, 1024, tc::kSw128);
            bd = tc::smem_desc(b + q * 32, 16, 1024, tc::kSw128);
          }
          tc::mma_bf16(tmem, ad, bd, idesc, 1u);
        }
        tc::mma_commit(&bar);
      }
      __syncwarp();
      tc::mbar_wait(&bar, phase);
      phase ^= 1;
    }
    t1 = clock64();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (tc::warp_id() == 0) tc::tmem_dealloc<256>(tmem);
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  const int smem = 49 * 1024;
  cudaFuncSetAttribute(rate<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(rate<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 2000;
  for (int pc : {4, 8}) {
    for (int mn = 0; mn < 2; ++mn) {
      for (int rep = 0; rep < 2; ++rep) {
        if (mn) rate<true><<<148, 128, smem>>>(iters, pc, d);
        else rate<false><<<148, 128, smem>>>(iters, pc, d);
      }
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
      }
      long long h[148];
      cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (long long v : h) avg += v;
      avg /= 148;
      printf("%s operands, %d MMAs per commit: %.1f cycles per M128xN256xK16 MMA "
             "(tensor floor 128)\n",
             mn ? "MN-major" : "K-major", pc, avg / (iters * pc));
    }
  }
  return 0;
}
