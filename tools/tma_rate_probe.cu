// Probe: per-SM TMA load throughput against box shape, for the operand
// boxes the conv engine issues — [rows][64 channels] bf16 tiles (128-byte
// rows) out of an NTHWC activation with C channels per pixel (rows C*2 bytes
// apart).  Every CTA (one per SM) streams its own slice of a tensor larger
// than L2 through an S-stage ring (no MMA): reported are bytes per SM-cycle
// and TB/s for the whole chip, for 64-, 128- and 256-row boxes.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O2 \
//        -I paper_1910_00932_b200/csrc tools/tma_rate_probe.cu -o tools/tma_rate_probe -lcuda
#include <cuda.h>
#include <cstdio>
#include <cstdlib>

#include "tc_common.cuh"

using namespace tsm;

constexpr int kStages = 6;

__global__ void __launch_bounds__(32, 1)
    stream(const __grid_constant__ CUtensorMap map, int rows_box, int boxes_per_stage,
           int iters, int64_t rows_total, int cboxes, long long* out) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (tc::smem_u32(raw) & 1023u)) & 1023u);
  __shared__ __align__(8) uint64_t full[kStages];
  const int stage_bytes = rows_box * 128 * boxes_per_stage;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) tc::mbar_init(&full[s], 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    // this SM's rows: a contiguous slice, walked box by box
    const int64_t slice = rows_total / gridDim.x;
    int64_t row = slice * blockIdx.x;
    int cb = 0;
    for (int it = 0; it < iters + kStages; ++it) {
      const int s = it % kStages;
      if (it >= kStages) tc::mbar_wait(&full[s], ((it / kStages) - 1) & 1);
      if (it < iters) {
        tc::mbar_arrive_expect_tx(&full[s], stage_bytes);
        for (int b = 0; b < boxes_per_stage; ++b) {
          tc::tma_load_2d(sm + s * stage_bytes + b * rows_box * 128, &map, &full[s], cb * 64,
                          (int)row);
          if (++cb == cboxes) {
            cb = 0;
            row += rows_box;
            if (row + rows_box > slice * (blockIdx.x + 1)) row = slice * blockIdx.x;
          }
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                             const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                             const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  EncodeFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int64_t bytes = (argc > 1 ? atoll(argv[1]) : 1024) << 20;  // MiB: 1024 > L2, 64 < L2
  void* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  long long* d;
  cudaMalloc(&d, sms * sizeof(long long));
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int C : {256, 1024}) {
    const int64_t rows = bytes / (C * 2);
    for (int rb : {64, 128, 256}) {
      for (int bps : {1, 2, 4}) {
        if (rb * 128 * bps * kStages > 196 * 1024) continue;
        CUtensorMap map;
        cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)rows};
        cuuint64_t strides[1] = {(cuuint64_t)C * 2};
        cuuint32_t box[2] = {64, (cuuint32_t)rb}, es[2] = {1, 1};
        enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int stage_bytes = rb * 128 * bps;
        const int iters = (int)((1ll << 29) / sms / stage_bytes);
        const int smem = stage_bytes * kStages + 1024;
        for (int rep = 0; rep < 2; ++rep)
          stream<<<sms, 32, smem>>>(map, rb, bps, iters, rows, C / 64, d);
        if (cudaDeviceSynchronize() != cudaSuccess) {
          printf("error\n");
          return 1;
        }
        long long h[256];
        cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
        const double bpc = (double)iters * stage_bytes / mx;
        printf("C=%4d box %3d rows x 128 B, %d boxes/stage (%3d KB): %6.1f B/cycle/SM, "
               "%5.2f TB/s chip, %5.0f cycles per box\n",
               C, rb, bps, stage_bytes / 1024, bpc, bpc * sms * clk * 1e3 / 1e12,
               mx / ((double)iters * bps));
      }
    }
  }
  return 0;
}
