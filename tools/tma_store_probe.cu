// Microbenchmark: TMA tensor-store throughput from shared memory into a
// [rows][256] bf16 matrix (the layout of a 256-channel NTHWC activation),
// as a function of the box width (32 channels / 64 B rows with SW64, or
// 64 channels / 128 B rows with SW128) and the number of stores in flight.
// Also a plain st.global baseline.  148 CTAs x 8 epilogue-like warps.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O2 \
//        -I paper_1910_00932_b200/csrc tools/tma_store_probe.cu -o tools/tma_store_probe -lcuda
#include <cuda.h>
#include <cstdio>
#include <vector>

#include "tc_common.cuh"

using namespace tsm;

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

constexpr int C = 256;

// Each CTA writes row blocks of 128 rows x 256 channels; `grp` threads
// groups of 128 threads each own a stripe of column boxes.
template <int BOXC>
__global__ void __launch_bounds__(256, 1)
    store_kernel(const __grid_constant__ CUtensorMap map, int row_blocks, int inflight) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  constexpr int BOXB = 128 * BOXC * 2;
  const int grp = threadIdx.x / 128;
  const bool leader = (threadIdx.x % 128) == 0;
  uint8_t* buf = sm + grp * 4 * BOXB;
  for (int i = threadIdx.x % 128; i < 4 * BOXB / 16; i += 128)
    reinterpret_cast<uint4*>(buf)[i] = make_uint4(i, i, i, i);
  tc::fence_proxy_async();
  __syncthreads();
  int seq = 0;
  for (int rb = blockIdx.x; rb < row_blocks; rb += gridDim.x) {
    for (int cb = grp; cb < C / BOXC; cb += 2, ++seq) {
      if (leader) {
        tc::bulk_wait_read_n(inflight - 1);
        if (BOXC == 32) tc::tma_store_2d(&map, buf + (seq % inflight) * BOXB, cb * BOXC, rb * 128);
        else tc::tma_store_2d(&map, buf + (seq % inflight) * BOXB, cb * BOXC, rb * 128);
        tc::bulk_commit();
      }
      __syncwarp();
    }
  }
  if (leader) tc::bulk_wait<0>();
}


// Load + store (the residual epilogue's pattern): each group TMA-loads a box
// from `src` into a slot, waits, and TMA-stores it to `dst` (same coordinates).
template <int BOXC>
__global__ void __launch_bounds__(256, 1)
    copy_kernel(const __grid_constant__ CUtensorMap msrc, const __grid_constant__ CUtensorMap mdst,
                int row_blocks) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  constexpr int BOXB = 128 * BOXC * 2;
  constexpr int SL = 4;  // slots per group
  __shared__ __align__(8) uint64_t bar[2][SL];
  const int grp = threadIdx.x / 128;
  const bool leader = (threadIdx.x % 128) == 0;
  uint8_t* buf = sm + grp * SL * BOXB;
  if (leader)
    for (int i = 0; i < SL; ++i) tc::mbar_init(&bar[grp][i], 1);
  tc::fence_barrier_init();
  __syncthreads();
  if (!leader) return;
  // sequence of this group's boxes
  const int per_rb = C / BOXC / 2;
  int n = 0;
  for (int rb = blockIdx.x; rb < row_blocks; rb += gridDim.x) n += per_rb;
  auto coord = [&](int L, int& cb, int& rb) {
    rb = blockIdx.x + (L / per_rb) * gridDim.x;
    cb = grp + 2 * (L % per_rb);
  };
  for (int L = 0; L < SL && L < n; ++L) {
    int cb, rb;
    coord(L, cb, rb);
    tc::mbar_arrive_expect_tx(&bar[grp][L], BOXB);
    tc::tma_load_2d(buf + L * BOXB, &msrc, &bar[grp][L], cb * BOXC, rb * 128);
  }
  for (int L = 0; L < n; ++L) {
    const int sl = L % SL;
    tc::mbar_wait(&bar[grp][sl], (L / SL) & 1);
    int cb, rb;
    coord(L, cb, rb);
    tc::tma_store_2d(&mdst, buf + sl * BOXB, cb * BOXC, rb * 128);
    tc::bulk_commit();
    if (L + SL < n) {
      tc::bulk_wait_read<0>();  // slot read by the store before it is reloaded
      int cb2, rb2;
      coord(L + SL, cb2, rb2);
      tc::mbar_arrive_expect_tx(&bar[grp][sl], BOXB);
      tc::tma_load_2d(buf + sl * BOXB, &msrc, &bar[grp][sl], cb2 * BOXC, rb2 * 128);
    }
  }
  tc::bulk_wait<0>();
}

__global__ void stg_kernel(uint4* out, long long n16) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n16;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = make_uint4((uint32_t)i, 0, 0, 0);
}

int main() {
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<EncodeTiledFn>(fn);
  const long long rows = 64LL * 8 * 56 * 56;  // 1.6 M rows x 256 ch = 822 MB
  void* out;
  cudaMalloc(&out, rows * C * 2);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return rows * C * 2 * 5 / (ms * 1e-3) / 1e9;
  };
  const int blocks = (int)(rows / 128);
  for (int boxc : {32, 64}) {
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)C * 2};
    cuuint32_t box[2] = {(cuuint32_t)boxc, 128};
    cuuint32_t es[2] = {1, 1};
    CUresult r = encode(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, out, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE,
                        boxc == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); return 1; }
    const int smem = 2 * 4 * 128 * boxc * 2 + 1024;
    if (boxc == 32) cudaFuncSetAttribute(store_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    else cudaFuncSetAttribute(store_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int inflight : {1, 2, 4}) {
      double gbs = timeit([&] {
        if (boxc == 32) store_kernel<32><<<148, 256, smem>>>(map, blocks, inflight);
        else store_kernel<64><<<148, 256, smem>>>(map, blocks, inflight);
      });
      cudaError_t e = cudaGetLastError();
      printf("TMA store box %2d ch (%3d B rows), %d in flight per group: %7.0f GB/s %s\n", boxc,
             boxc * 2, inflight, gbs, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  void* src;
  cudaMalloc(&src, rows * C * 2);
  cudaMemset(src, 0, rows * C * 2);
  for (int boxc : {32, 64}) {
    CUtensorMap ms, md;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)C * 2};
    cuuint32_t box[2] = {(cuuint32_t)boxc, 128};
    cuuint32_t es[2] = {1, 1};
    const auto sw = boxc == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
    encode(&ms, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    encode(&md, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, out, dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = 2 * 4 * 128 * boxc * 2 + 1024;
    if (boxc == 32) cudaFuncSetAttribute(copy_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    else cudaFuncSetAttribute(copy_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    double gbs = 2 * timeit([&] {
      if (boxc == 32) copy_kernel<32><<<148, 256, smem>>>(ms, md, blocks);
      else copy_kernel<64><<<148, 256, smem>>>(ms, md, blocks);
    });
    cudaError_t e = cudaGetLastError();
    printf("TMA load+store box %2d ch (%3d B rows), 4 slots per group: %7.0f GB/s (read+write) %s\n",
           boxc, boxc * 2, gbs, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  double gbs = timeit([&] { stg_kernel<<<148 * 8, 256>>>((uint4*)out, rows * C * 2 / 16); });
  printf("st.global.v4 baseline: %7.0f GB/s\n", gbs);
  return 0;
}
