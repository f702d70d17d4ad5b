// Whole-bottleneck fusion for the identity-skip residual-shift unit of res2
// (c_in = c_out = 256, width 64, shift 1/8: F = B = 32, stride 1) — SURVEY
// §8(f) f2.  One persistent kernel computes, per 16 x 8-pixel tile of one
// frame,
//
//   r1 = relu(conv1x1(shift(x)) + b1)     on the 18 x 10 halo of the tile
//   r2 = relu(conv3x3(r1) + b2)           r1 never leaves shared memory
//   y  = relu(conv1x1(r2) + b3 + x)       r2 stays on chip for conv3
//
// (run_unit, net.cpp:85-126, for the unit expand_layer builds, arch.cpp:
// 278-323).  HBM traffic per pixel: x once (256 ch) and y once (256 ch),
// plus the activations the backward saves (r1, r2 and the three ReLU
// bitmasks) — against x twice (conv1 and the residual), r1 and r2 each
// written and read back, y written, for the three-kernel sequence.
//
// Operands (all tcgen05, bf16 x bf16 -> fp32 in TMEM):
//   conv1  A = the shifted x halo: eight 32-channel TMA boxes of 10 x 18
//          pixels, channels [0,32) at frame t-1, [32,64) at t+1, the rest
//          at t, from a 5-D map (C, W, H, T, N) so frames outside the clip
//          and pixels outside the image are TMA zero fill (the reference's
//          +0.0 boundary, kernels.cpp:108-115); the 180 halo rows are two
//          M = 128 MMA tiles (rows 180..255 are ignored).  B = W1, resident.
//          Halo pixels outside the image are set to 0 in the epilogue (they
//          are conv2's zero padding, not relu(b1)).
//   conv2  A = the r1 halo tile in shared memory, one descriptor per tap
//          (start row r * 10 + s, 8-row groups 10 rows apart) as in
//          halo_conv.cuh; B = the W2 tap, streamed through the operand ring.
//   conv3  A = the r2 tile in shared memory; B = W3, resident; the residual
//          (unshifted x at the tile, eight 32-channel boxes streamed through
//          the ring) enters the accumulator as identity k-blocks, like the
//          unfused conv3 (tc_gemm.cuh res_kb), so the epilogue has no
//          residual stream.
//
// The summation order of every output equals the unfused path's (conv1's K
// in channel order, conv2 tap-major, conv3 then the identity blocks): the
// fused unit is bitwise identical to tsm_block_fwd's three kernels.
//
// Warp roles: w0 TMA producer, w1 TMEM allocator + MMA issuer, w2..w9
// epilogue (two groups of four warps).  Per CTA the tiles are pipelined:
// the MMA issues conv2(i), conv1(i+1), conv3(i); the epilogue runs
// epi2(i), epi1(i+1), epi3(i).  Every accumulator and on-chip buffer is free
// by issue order, so only five MMA<->epilogue barriers are needed: conv1(i+1)
// is issued after conv2(i), which waited for epi1(i) to finish reading D1;
// conv2(i+1) waits for epi1(i+1), which the epilogue runs after epi2(i) (D2
// read); conv3(i+1) waits for epi2(i+1), run after epi3(i) (D3 read); and
// the r1 / r2 tiles are rewritten only after an accumulator that was issued
// after their last reader completed (MMAs complete in issue order).
#pragma once
#include "tc_common.cuh"

namespace tsm {
namespace fused {

constexpr int kThreads = 320;       // w0 TMA, w1 MMA, w2..w9 epilogue
constexpr int kEpiThreads = 256;
constexpr int kTH = 16, kTW = 8;    // output tile: 16 rows x 8 columns = 128 pixels
constexpr int kHP = kTW + 2, kHR = kTH + 2;  // halo pitch (10) / rows (18)
constexpr int kHalo = kHP * kHR;    // 180 halo pixels
constexpr int kC = 256, kWd = 64;   // unit channels / width
constexpr int kSlotBytes = 12 * 1024;   // ring slot: a 32-ch halo box (11.25 KB),
                                        // a W2 tap (8 KB) or a 32-ch centre box (8 KB)
constexpr int kHaloSlabBytes = kHalo * 64;  // 11520
constexpr int kCentreSlabBytes = 128 * 64;  // 8192
constexpr int kTapBytes = 64 * 128;         // W2 tap [64 co][64 ci] SW128
constexpr int kW1Bytes = 64 * kC * 2;       // [64 co][256 ci] as four [64][64] SW128 blocks
constexpr int kW3Bytes = kC * kWd * 2;      // [256 co][64 ci] SW128
constexpr int kIdentBytes = 64 * 64 * 2;
constexpr int kR1Bytes = kHalo * 128;       // r1 halo tile [180][64] SW128
constexpr int kR1Alloc = 23 * 1024;
constexpr int kR2Bytes = 128 * 128;         // r2 tile [128][64] SW128
constexpr int kStageOut = 128 * 64;         // y sub-tile [128][32] SW64
constexpr int kMaxSlots = 8;
constexpr int kSmemLimit = 227 * 1024;

struct Params {
  int tiles_y, tiles_x, total;  // tiles per frame row / column, total tiles
  int T, H, W;                  // frames per clip, extent
  const float *b1, *b2, *b3;
  __nv_bfloat16* r1;            // saved activation [frames][H][W][64]
  uint32_t *r1_bits, *r2_bits, *y_bits;  // [pixels][2], [pixels][2], [pixels][8]
  int slots;                    // ring depth
};

// smem layout (offsets from the 1 KiB-aligned base)
struct Layout {
  static constexpr int W1 = 0;
  static constexpr int W3 = W1 + kW1Bytes;                 // 32 KB
  static constexpr int IDENT = W3 + kW3Bytes;              // 64 KB
  static constexpr int R2 = IDENT + kIdentBytes;           // 72 KB
  static constexpr int OUT = R2 + kR2Bytes;                // 88 KB: [2 groups][8 KB]
  static constexpr int RING = OUT + 2 * kStageOut;         // 104 KB
  // the ring is followed by the r1 halo tile: conv1's second M tile reads
  // 256 rows of a 180-row halo box, i.e. up to 4.75 KB past the last slot
  __host__ __device__ static int r1(int slots) { return RING + slots * kSlotBytes; }
  __host__ __device__ static int bias(int slots) { return r1(slots) + kR1Alloc; }   // b1, b2, b3 fp32
  __host__ __device__ static int bars(int slots) { return bias(slots) + (64 + 64 + 256) * 4; }
  __host__ __device__ static int bytes(int slots) { return bars(slots) + 512 + 1024; }
};

__device__ __forceinline__ uint32_t sw64(int r, int c) {
  return (uint32_t)(r * 64 + ((c ^ ((r >> 1) & 3)) << 4));
}
__device__ __forceinline__ uint32_t sw128(int r, int c) {
  return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4));
}

__global__ void __launch_bounds__(kThreads, 1)
    bottleneck_fwd_kernel(const __grid_constant__ CUtensorMap map_x5,   // x (C,W,H,T,N) box {32,10,18,1,1}
                          const __grid_constant__ CUtensorMap map_xc5,  // x (C,W,H,T,N) box {32,8,16,1,1}
                          const __grid_constant__ CUtensorMap map_w1,   // W1 [64][256] box {64,64}
                          const __grid_constant__ CUtensorMap map_w2,   // W2 [64][9*64] box {64,64}
                          const __grid_constant__ CUtensorMap map_w3,   // W3 [256][64] box {64,256}
                          const __grid_constant__ CUtensorMap map_r2,   // r2 (64,W,H,F) box {64,8,16,1}
                          const __grid_constant__ CUtensorMap map_y,    // y (256,W,H,F) box {32,8,16,1}
                          const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  const int S = p.slots;
  uint8_t* ring = smem + Layout::RING;
  uint8_t* r1s = smem + Layout::r1(S);
  uint8_t* r2s = smem + Layout::R2;
  float* bias_s = reinterpret_cast<float*>(smem + Layout::bias(S));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Layout::bars(S));
  uint64_t* full = bars;                 // [kMaxSlots]
  uint64_t* empty = full + kMaxSlots;    // [kMaxSlots]
  uint64_t* wbar = empty + kMaxSlots;    // resident weights landed
  uint64_t* d1_full = wbar + 1;          // conv1 accumulators ready (MMA -> epilogue)
  uint64_t* d2_full = d1_full + 1;
  uint64_t* d3_full = d2_full + 1;
  uint64_t* r1_ready = d3_full + 1;      // r1 halo tile written (epilogue -> MMA)
  uint64_t* r2_ready = r1_ready + 1;     // r2 tile written
  uint32_t* tslot = reinterpret_cast<uint32_t*>(r2_ready + 1);
  const uint32_t warp = tc::warp_id();

  if (warp == 0 && tc::lane_id() == 0) {
    tc::tma_prefetch(&map_x5);
    tc::tma_prefetch(&map_xc5);
    tc::tma_prefetch(&map_w2);
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(wbar, 1);
    tc::mbar_init(d1_full, 1);
    tc::mbar_init(d2_full, 1);
    tc::mbar_init(d3_full, 1);
    tc::mbar_init(r1_ready, kEpiThreads / 32);
    tc::mbar_init(r2_ready, kEpiThreads / 32);
    tc::fence_barrier_init();
  }
  if (warp >= 2) {
    // identity B operand [64 n][64 k] SW128 (row n = 128 B, chunk c at c ^ (n & 7))
    uint8_t* ident = smem + Layout::IDENT;
    for (int i = threadIdx.x - 64; i < kIdentBytes / 16; i += kEpiThreads) {
      const int n = i >> 3, c = (i & 7) ^ (n & 7);
      uint4 v = make_uint4(0, 0, 0, 0);
      if (c == (n >> 3)) {
        uint32_t* w = reinterpret_cast<uint32_t*>(&v);
        const int e = n & 7;
        w[e >> 1] = (e & 1) ? 0x3F800000u : 0x00003F80u;
      }
      *reinterpret_cast<uint4*>(ident + i * 16) = v;
    }
    tc::fence_proxy_async();
  }
  if (warp == 1) tc::tmem_alloc<512>(tslot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;
  tc::pdl_wait();  // (PDL) global memory only after the predecessor completed
  tc::pdl_launch_dependents();
  if (warp >= 2) {  // biases -> shared memory (read by the epilogue only)
    for (int i = threadIdx.x - 64; i < 64 + 64 + 256; i += kEpiThreads)
      bias_s[i] = i < 64 ? __ldg(p.b1 + i) : i < 128 ? __ldg(p.b2 + i - 64) : __ldg(p.b3 + i - 128);
    tc::named_bar(4, kEpiThreads);
  }
  // TMEM columns: D1 (two M tiles) [0,128), D2 [128,192), D3 [256,512)
  constexpr uint32_t kD1 = 0, kD2 = 128, kD3 = 256;

  auto decode = [&](int tile, int& f, int& ty, int& tx) {
    tx = tile % p.tiles_x;
    const int rest = tile / p.tiles_x;
    ty = rest % p.tiles_y;
    f = rest / p.tiles_y;
  };
  const int tile0 = blockIdx.x, tstep = gridDim.x;
  const int ntiles = tile0 < p.total ? (p.total - tile0 + tstep - 1) / tstep : 0;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (tc::elect_one()) {
      uint8_t* w1s = smem + Layout::W1;
      uint8_t* w3s = smem + Layout::W3;
      tc::mbar_arrive_expect_tx(wbar, kW1Bytes + kW3Bytes);
      for (int j = 0; j < 4; ++j) tc::tma_load_2d(w1s + j * 8192, &map_w1, wbar, j * 64, 0);
      tc::tma_load_2d(w3s, &map_w3, wbar, 0, 0);
      int slot = 0;
      uint32_t phase = 0;
      auto next_slot = [&]() -> uint8_t* {
        tc::mbar_wait(&empty[slot], phase ^ 1);
        return ring + slot * kSlotBytes;
      };
      auto advance = [&]() {
        if (++slot == S) {
          slot = 0;
          phase ^= 1;
        }
      };
      auto halo = [&](int tile) {  // conv1 A: eight 32-channel halo boxes, shifted
        int f, ty, tx;
        decode(tile, f, ty, tx);
        const int n = f / p.T, t = f - n * p.T;
        for (int j = 0; j < 8; ++j) {
          uint8_t* dst = next_slot();
          tc::mbar_arrive_expect_tx(&full[slot], kHaloSlabBytes);
          const int dt = j == 0 ? -1 : (j == 1 ? 1 : 0);  // [0,32): t-1, [32,64): t+1
          tc::tma_load_5d(dst, &map_x5, &full[slot], j * 32, tx * kTW - 1, ty * kTH - 1, t + dt, n);
          advance();
        }
      };
      if (ntiles > 0) halo(tile0);
      for (int it = 0; it < ntiles; ++it) {
        const int tile = tile0 + it * tstep;
        for (int tap = 0; tap < 9; ++tap) {  // conv2 B: the W2 taps
          uint8_t* dst = next_slot();
          tc::mbar_arrive_expect_tx(&full[slot], kTapBytes);
          tc::tma_load_2d(dst, &map_w2, &full[slot], tap * 64, 0);
          advance();
        }
        if (it + 1 < ntiles) halo(tile + tstep);
        int f, ty, tx;
        decode(tile, f, ty, tx);
        const int n = f / p.T, t = f - n * p.T;
        for (int j = 0; j < 8; ++j) {  // conv3 residual: x at the tile, unshifted
          uint8_t* dst = next_slot();
          tc::mbar_arrive_expect_tx(&full[slot], kCentreSlabBytes);
          tc::tma_load_5d(dst, &map_xc5, &full[slot], j * 32, tx * kTW, ty * kTH, t, n);
          advance();
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    constexpr uint32_t id64 = tc::idesc_bf16(128, 64, false, false);
    constexpr uint32_t id256 = tc::idesc_bf16(128, 256, false, false);
    const uint32_t w1a = tc::smem_u32(smem + Layout::W1), w3a = tc::smem_u32(smem + Layout::W3);
    const uint32_t ida = tc::smem_u32(smem + Layout::IDENT), r1a = tc::smem_u32(r1s),
                   r2a = tc::smem_u32(r2s), ringa = tc::smem_u32(ring);
    tc::mbar_wait(wbar, 0);
    int slot = 0;
    uint32_t phase = 0;
    auto take = [&]() -> uint32_t {
      tc::mbar_wait(&full[slot], phase);
      tc::tc_fence_after();
      return ringa + slot * kSlotBytes;
    };
    auto release = [&]() {
      if (tc::elect_one()) tc::mma_commit(&empty[slot]);
      __syncwarp();
      if (++slot == S) {
        slot = 0;
        phase ^= 1;
      }
    };
    auto commit = [&](uint64_t* bar) {
      if (tc::elect_one()) tc::mma_commit(bar);
      __syncwarp();
    };
    auto conv1 = [&]() {
      // K = 256 in channel order: slab j holds channels [32 j, 32 j + 32)
      // (SW64 rows of 64 B); two M tiles (halo rows 0..127, 128..255)
      for (int j = 0; j < 8; ++j) {
        const uint32_t a = take();
        if (tc::elect_one()) {
#pragma unroll
          for (int q = 0; q < 2; ++q) {  // UMMA_K = 16 channels = 32 bytes
            const int kk = j * 2 + q;     // k-step over the 256 channels
            const uint64_t bd =
                tc::smem_desc(w1a + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024, tc::kSw128);
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
              const uint64_t ad = tc::smem_desc(a + mt * 128 * 64 + q * 32, 16, 512, tc::kSw64);
              tc::mma_bf16(tmem + kD1 + mt * 64, ad, bd, id64, kk > 0 ? 1u : 0u);
            }
          }
        }
        __syncwarp();
        release();
      }
      commit(d1_full);
    };
    auto conv2 = [&](int it) {
      tc::mbar_wait(r1_ready, it & 1);
      tc::tc_fence_after();
      for (int tap = 0; tap < 9; ++tap) {
        const uint32_t b = take();
        const int r = tap / 3, s = tap % 3;
        if (tc::elect_one()) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint64_t ad = tc::smem_desc(r1a + (r * kHP + s) * 128 + q * 32, 16, kHP * 128,
                                              tc::kSw128);
            const uint64_t bd = tc::smem_desc(b + q * 32, 16, 1024, tc::kSw128);
            tc::mma_bf16(tmem + kD2, ad, bd, id64, (tap > 0 || q > 0) ? 1u : 0u);
          }
        }
        __syncwarp();
        release();
      }
      commit(d2_full);
    };
    auto conv3 = [&](int it) {
      tc::mbar_wait(r2_ready, it & 1);
      tc::tc_fence_after();
      if (tc::elect_one()) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint64_t ad = tc::smem_desc(r2a + q * 32, 16, 1024, tc::kSw128);
          const uint64_t bd = tc::smem_desc(w3a + q * 32, 16, 1024, tc::kSw128);
          tc::mma_bf16(tmem + kD3, ad, bd, id256, q > 0 ? 1u : 0u);
        }
      }
      __syncwarp();
      // residual: D3[:, 64 c + n] += x[:, 64 c + k] I[n][k], slab j = channels [32 j, +32)
      for (int j = 0; j < 8; ++j) {
        const uint32_t a = take();
        if (tc::elect_one()) {
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const uint64_t ad = tc::smem_desc(a + q * 32, 16, 512, tc::kSw64);
            const uint64_t bd = tc::smem_desc(ida + ((j & 1) * 2 + q) * 32, 16, 1024, tc::kSw128);
            tc::mma_bf16(tmem + kD3 + (j >> 1) * 64, ad, bd, id64, 1u);
          }
        }
        __syncwarp();
        release();
      }
      commit(d3_full);
    };
    if (ntiles > 0) conv1();
    for (int it = 0; it < ntiles; ++it) {
      conv2(it);
      if (it + 1 < ntiles) conv1();
      conv3(it);
    }
  } else {
    // ===================== epilogue (two groups of four warps) =====================
    const int grp = (int)(warp - 2) >> 2;
    const int q = warp & 3;  // TMEM lane quarter
    const int lane = tc::lane_id();
    const int lrow = q * 32 + lane;
    const bool leader = ((warp - 2) & 3) == 0 && lane == 0;
    const bool all_leader = warp == 2 && lane == 0;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    uint8_t* ob = smem + Layout::OUT + grp * kStageOut;
    const float* b1 = bias_s;
    const float* b2 = bias_s + 64;
    const float* b3 = bias_s + 128;
    auto arrive_warp = [&](uint64_t* bar) {
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(bar);
    };
    // epi1: r1 = relu(D1 + b1) on the halo (0 outside the image) -> r1 tile in
    // smem (conv2's A) + the tile's centre pixels to global (saved) + bits
    auto epi1 = [&](int it, int tile) {
      int f, ty, tx;
      decode(tile, f, ty, tx);
      tc::mbar_wait(d1_full, it & 1);
      tc::tc_fence_after();
      const int hp = grp * 128 + lrow;  // halo pixel (M tile grp, row lrow)
      uint32_t raw[4][16];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        tc::tmem_ld_32x32b_x16(tmem + lane_base + kD1 + grp * 64 + c * 16, raw[c]);
      tc::tmem_ld_wait();
      if (hp < kHalo) {
        const int hr = hp / kHP, hc = hp - hr * kHP;
        const int ph = ty * kTH - 1 + hr, pw = tx * kTW - 1 + hc;
        const bool inside = ph >= 0 && ph < p.H && pw >= 0 && pw < p.W;
        uint32_t o[32];
#pragma unroll
        for (int c = 0; c < 4; ++c)
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float a = __uint_as_float(raw[c][2 * i]) + b1[c * 16 + 2 * i];
            const float b = __uint_as_float(raw[c][2 * i + 1]) + b1[c * 16 + 2 * i + 1];
            o[c * 8 + i] = inside ? tc::pack_bf16(fmaxf(a, 0.f), fmaxf(b, 0.f)) : 0u;
          }
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<uint4*>(r1s + sw128(hp, c)) =
              make_uint4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
        const bool centre = hr >= 1 && hr <= kTH && hc >= 1 && hc <= kTW;
        if (centre && inside) {
          const long long pix = ((long long)f * p.H + ph) * p.W + pw;
          uint4* dst = reinterpret_cast<uint4*>(p.r1 + pix * 64);
#pragma unroll
          for (int c = 0; c < 8; ++c)
            dst[c] = make_uint4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
          uint32_t lo[16], hi[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            lo[i] = o[i];
            hi[i] = o[16 + i];
          }
          p.r1_bits[pix * 2] = tc::relu_bits16(lo);
          p.r1_bits[pix * 2 + 1] = tc::relu_bits16(hi);
        }
      }
      tc::fence_proxy_async();  // r1 tile: generic writes -> async-proxy (MMA) reads
      tc::tc_fence_before();
      arrive_warp(r1_ready);
    };
    // epi2: r2 = relu(D2 + b2) -> r2 tile (conv3's A, and stored by TMA) + bits
    auto epi2 = [&](int it, int tile) {
      int f, ty, tx;
      decode(tile, f, ty, tx);
      tc::mbar_wait(d2_full, it & 1);
      tc::tc_fence_after();
      uint32_t raw0[16], raw1[16];
      tc::tmem_ld_32x32b_x16(tmem + lane_base + kD2 + grp * 32, raw0);
      tc::tmem_ld_32x32b_x16(tmem + lane_base + kD2 + grp * 32 + 16, raw1);
      tc::tmem_ld_wait();
      uint32_t o[16];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        o[i] = tc::pack_bf16(fmaxf(__uint_as_float(raw0[2 * i]) + b2[grp * 32 + 2 * i], 0.f),
                             fmaxf(__uint_as_float(raw0[2 * i + 1]) + b2[grp * 32 + 2 * i + 1], 0.f));
        o[8 + i] = tc::pack_bf16(fmaxf(__uint_as_float(raw1[2 * i]) + b2[grp * 32 + 16 + 2 * i], 0.f),
                                 fmaxf(__uint_as_float(raw1[2 * i + 1]) + b2[grp * 32 + 17 + 2 * i], 0.f));
      }
      const int ph = ty * kTH + (lrow >> 3), pw = tx * kTW + (lrow & 7);
      if (ph < p.H && pw < p.W)
        p.r2_bits[(((long long)f * p.H + ph) * p.W + pw) * 2 + grp] = tc::relu_bits16(o);
      // the previous tile's r2 store must have finished reading the tile
      if (all_leader) tc::bulk_wait_read<0>();
      tc::named_bar(1, kEpiThreads);
#pragma unroll
      for (int c = 0; c < 4; ++c)
        *reinterpret_cast<uint4*>(r2s + sw128(lrow, grp * 4 + c)) =
            make_uint4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
      tc::fence_proxy_async();
      tc::tc_fence_before();
      tc::named_bar(1, kEpiThreads);
      if (all_leader) {
        tc::tma_store_4d(&map_r2, r2s, 0, tx * kTW, ty * kTH, f);
        tc::bulk_commit();
      }
      arrive_warp(r2_ready);
    };
    // epi3: y = relu(D3 + b3) (the residual is already in D3) -> TMA stores of
    // 32-channel sub-tiles + bits; group grp owns channels [128 grp, +128)
    auto epi3 = [&](int it, int tile) {
      int f, ty, tx;
      decode(tile, f, ty, tx);
      tc::mbar_wait(d3_full, it & 1);
      tc::tc_fence_after();
      const int ph = ty * kTH + (lrow >> 3), pw = tx * kTW + (lrow & 7);
      const bool inside = ph < p.H && pw < p.W;
      const long long pix = ((long long)f * p.H + ph) * p.W + pw;
#pragma unroll 1
      for (int u = 0; u < 4; ++u) {
        const int col = grp * 128 + u * 32;
        uint32_t raw0[16], raw1[16];
        tc::tmem_ld_32x32b_x16(tmem + lane_base + kD3 + col, raw0);
        tc::tmem_ld_32x32b_x16(tmem + lane_base + kD3 + col + 16, raw1);
        tc::tmem_ld_wait();
        uint32_t o[16];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          o[i] = tc::pack_bf16(fmaxf(__uint_as_float(raw0[2 * i]) + b3[col + 2 * i], 0.f),
                               fmaxf(__uint_as_float(raw0[2 * i + 1]) + b3[col + 2 * i + 1], 0.f));
          o[8 + i] =
              tc::pack_bf16(fmaxf(__uint_as_float(raw1[2 * i]) + b3[col + 16 + 2 * i], 0.f),
                            fmaxf(__uint_as_float(raw1[2 * i + 1]) + b3[col + 17 + 2 * i], 0.f));
        }
        if (inside) p.y_bits[pix * 8 + col / 32] = tc::relu_bits16(o);
        if (leader) tc::bulk_wait_read<0>();  // the staging tile's last store has read it
        tc::named_bar(2 + grp, 128);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          *reinterpret_cast<uint4*>(ob + sw64(lrow, c)) =
              make_uint4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
        tc::fence_proxy_async();
        tc::named_bar(2 + grp, 128);
        if (leader) {
          tc::tma_store_4d(&map_y, ob, col, tx * kTW, ty * kTH, f);
          tc::bulk_commit();
        }
      }
    };
    if (ntiles > 0) epi1(0, tile0);
    for (int it = 0; it < ntiles; ++it) {
      const int tile = tile0 + it * tstep;
      epi2(it, tile);
      if (it + 1 < ntiles) epi1(it + 1, tile + tstep);
      epi3(it, tile);
    }
    if (leader || all_leader) tc::bulk_wait<0>();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(tmem);
}

}  // namespace fused
}  // namespace tsm
