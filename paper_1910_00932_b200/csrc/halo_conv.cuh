// Halo-tile 3x3 stride-1 convolutions for 64 -> 64 channel layers (the
// TSM-R50 res2 conv2: 56x56 pixels, the stage where im2col TMA traffic —
// nine 128-byte window rows per pixel — bounds the generic GEMM).
//
// One TMA box brings a pixel tile plus its one-pixel halo into shared
// memory (128-byte swizzled rows, one pixel = 64 channels per row).  Every
// filter tap is then a tcgen05 descriptor into that tile: the tap offset is
// a start-address offset of (r * pitch + s) rows and the stride between
// 8-pixel core groups (SBO) is the halo pitch.  tcgen05 applies the 128B
// swizzle on absolute shared-memory address bits, so descriptors may start
// at any 128-byte row (verified by tools/halo_probe.cu).
//
//   halo_conv_kernel<KH,C> y = act(conv(x, W) + bias) [* (mask > 0)]
//                        (forward, and dgrad with the tap-flipped W^T)
//                        tile = 16 x 8 output pixels, halo 18 x 10,
//                        weights (9 x 64 x 64) resident in shared memory.
//   wgrad3x3_c64_kernel  D[tap*64 + ci][co] = sum_p x(p + tap)[ci] dY(p)[co]
//                        per 8 x 8 output patch: halo 10 x 10 of x (MN-major
//                        A, taps paired into 128-row M tiles) and the dY
//                        patch (MN-major B).  All 576 rows live in five
//                        TMEM accumulators; the spare 64 rows of the fifth
//                        tile multiply a constant all-ones slab, giving the
//                        bias gradient sum_p dY(p)[co] from the same MMAs.
//                        K (patches) is split over the CTAs; fp32 partials
//                        are reduced in a fixed order (deterministic).
// Reference semantics: kernels.cpp:171-200 (forward), 246-280 (grad_x),
// 282-325 (grad_w, grad_b).
#pragma once
#include "pool_bwd.cuh"
#include "tc_common.cuh"

namespace tsm {
namespace halo {

constexpr int kThreads = 320;  // w0 TMA, w1 MMA, w2-9 epilogue (2 groups x 4 warps)
constexpr int kEpiThreads = 256;
constexpr int kRowB = 128;  // one pixel: 64 bf16 channels
constexpr int kSmemLimit = 227 * 1024;

// forward / dgrad: KH x KH taps (offsets -KH/2 .. KH-1-KH/2) over C-channel
// pixels, 64 output channels.  <3, 64>: the 64-wide 3x3 convs; <4, 16>: the
// space-to-depth stem (a 7x7 / stride-2 conv as 4x4 / stride-1, 32-byte
// pixel rows with the 32-byte swizzle).
constexpr int kTH = 16, kTW = 8;                  // output tile (pixels)
constexpr int kSub = 128 * 64;                    // [128 rows][32 ch] bf16 sub-tile
template <int KH, int C>
struct HaloCfg {
  static constexpr int RB = C * 2;                          // pixel row bytes
  static constexpr int PAD = KH / 2;                        // window origin offset
  static constexpr int HP = kTW + KH - 1, HR = kTH + KH - 1;  // halo pitch / rows
  static constexpr int HALO = HP * HR * RB;
  static constexpr int STRIDE = (HALO + 1023) / 1024 * 1024;  // 1 KiB aligned stages
  static constexpr int TAP = 64 * RB;                      // one tap's weights [64][C]
  static constexpr int WBYTES = KH * KH * TAP;              // resident weights
  static constexpr uint32_t SW = RB == 128 ? tc::kSw128 : RB == 64 ? tc::kSw64 : tc::kSw32;
};

// weight gradient: KH x KW taps over 64-channel pixels, 8 x 8 output patches.
// <3, 3>: the 64-wide 3x3 convs; <4, 1>: the space-to-depth stem after its
// four horizontal taps are folded into 64 channels (head_kernels: stem_x4).
constexpr int kPW = 8;                            // output patch 8 x 8
constexpr int kDyBytes = 64 * kRowB;              // 8192
constexpr int kOnesBytes = 13 * 1024;
constexpr int kMaxStages = 10;
template <int KH, int KW>
struct WgradCfg {
  static constexpr int TAPS = KH * KW;
  static constexpr int MT = (TAPS + 1) / 2;          // 128-row M tiles (tap pairs)
  static constexpr bool ONES = TAPS % 2 == 1;        // last pair's slab b: all-ones (db)
  static constexpr int P = kPW + KW - 1, R = kPW + KH - 1;  // halo pitch / rows
  static constexpr int HALO = P * R * kRowB;
  static constexpr int HSTRIDE = (HALO + 1023) / 1024 * 1024;
  static constexpr int STAGE = HSTRIDE + kDyBytes;
  static_assert(MT * 64 <= 512, "TMEM columns");
};

struct FwdParams {
  int tiles_y, tiles_x, total;
  const float* bias;
  int relu, has_mask, stages;
  int H, W;
  uint32_t* bits_out;         // nullable: ReLU bitmask of the output, [pixel][2] words
  const uint32_t* mask_bits;  // nullable: bitmask replacing the bf16 mask tile
};

struct WgradParams {
  int patches_y, patches_x, total;
  float* ws;     // [grid][576][64] fp32 partials
  float* db_ws;  // [grid][64] (nullable)
  int stages;
};

// pointer arithmetic (not an integer round trip) keeps the result a known
// shared-space pointer: LDS/STS instead of generic LD/ST
__device__ __forceinline__ uint8_t* align1k(uint8_t* p) {
  return p + ((1024u - (tc::smem_u32(p) & 1023u)) & 1023u);
}

// (frame, tile row, tile column) of a persistent CTA's tiles, advanced by the
// grid stride with carries instead of a division per tile.
struct TileCursor {
  int tx, ty, f, dx, dy, df;
  __device__ __forceinline__ void init(int tile, int stride, int tiles_x, int tiles_y) {
    tx = tile % tiles_x;
    ty = (tile / tiles_x) % tiles_y;
    f = tile / tiles_x / tiles_y;
    dx = stride % tiles_x;
    dy = (stride / tiles_x) % tiles_y;
    df = stride / tiles_x / tiles_y;
  }
  __device__ __forceinline__ void next(int tiles_x, int tiles_y) {
    tx += dx;
    const int cx = tx >= tiles_x;
    tx -= cx * tiles_x;
    ty += dy + cx;
    const int cy = ty >= tiles_y;
    ty -= cy * tiles_y;
    f += df + cy;
  }
};

// 16-byte chunk c of row r inside a [128][64 B] SW64-swizzled sub-tile.
__device__ __forceinline__ uint32_t sw64(int r, int c) {
  return (uint32_t)(r * 64 + ((c ^ ((r >> 1) & 3)) << 4));
}

// ---------------------------------------------------------------------------
template <int KH, int C>
__global__ void __launch_bounds__(kThreads, 1)
    halo_conv_kernel(const __grid_constant__ CUtensorMap map_x,
                       const __grid_constant__ CUtensorMap map_w,
                       const __grid_constant__ CUtensorMap map_out,
                       const __grid_constant__ CUtensorMap map_mask, const FwdParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  uint8_t* sw = smem;
  using HC = HaloCfg<KH, C>;
  uint8_t* halo = sw + HC::WBYTES;
  uint8_t* epi = halo + p.stages * HC::STRIDE;  // [grp][2 out sub-tiles, mask sub-tile]
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages], tfull[2], tempty[2],
      wbar, mbar[2];
  __shared__ uint32_t tslot;
  const uint32_t warp = tc::warp_id();
  const int S = p.stages;

  if (warp == 0 && tc::lane_id() == 0) {
    tc::tma_prefetch(&map_x);
    tc::tma_prefetch(&map_w);
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], kEpiThreads);
      tc::mbar_init(&mbar[a], 1);
    }
    tc::mbar_init(&wbar, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<128>(&tslot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  tc::pdl_wait();  // (PDL) global memory only after the predecessor completed
  tc::pdl_launch_dependents();
  const uint32_t tmem = tslot;

  if (warp == 0) {
    if (tc::elect_one()) {
      tc::mbar_arrive_expect_tx(&wbar, HC::WBYTES);
      for (int t = 0; t < KH * KH; ++t)
        tc::tma_load_2d(sw + t * HC::TAP, &map_w, &wbar, t * C, 0);
      int stage = 0;
      uint32_t phase = 0;
      TileCursor cur;
      cur.init(blockIdx.x, gridDim.x, p.tiles_x, p.tiles_y);
      for (int tile = blockIdx.x; tile < p.total;
           tile += gridDim.x, cur.next(p.tiles_x, p.tiles_y)) {
        tc::mbar_wait(&empty[stage], phase ^ 1);
        tc::mbar_arrive_expect_tx(&full[stage], HC::HALO);
        tc::tma_load_4d(halo + stage * HC::STRIDE, &map_x, &full[stage], 0,
                        cur.tx * kTW - HC::PAD, cur.ty * kTH - HC::PAD, cur.f);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = tc::idesc_bf16(128, 64, false, false);
    tc::mbar_wait(&wbar, 0);
    const uint32_t w0 = tc::smem_u32(sw), h0 = tc::smem_u32(halo);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < p.total; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      tc::mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
      tc::tc_fence_after();
      tc::mbar_wait(&full[stage], phase);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint32_t hs = h0 + stage * HC::STRIDE;
#pragma unroll
        for (int t = 0; t < KH * KH; ++t) {
          const int r = t / KH, s = t - KH * (t / KH);
#pragma unroll
          for (int j = 0; j < C / 16; ++j) {  // UMMA_K = 16 channels = 32 bytes
            const uint64_t ad = tc::smem_desc(hs + (r * HC::HP + s) * HC::RB + j * 32, 16,
                                              HC::HP * HC::RB, HC::SW);
            const uint64_t bd =
                tc::smem_desc(w0 + t * HC::TAP + j * 32, 16, 8 * HC::RB, HC::SW);
            tc::mma_bf16(tmem + acc * 64, ad, bd, idesc, (t > 0 || j > 0) ? 1u : 0u);
          }
        }
        tc::mma_commit(&empty[stage]);
        tc::mma_commit(&tfull[acc]);
      }
      __syncwarp();
      if (++stage == S) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else {
    // epilogue: group g owns channels [32 g, 32 g + 32); warp w reads TMEM
    // lanes (w % 4) * 32 .. +32 = tile rows (pixel i * 8 + j of the 16 x 8 tile)
    // Mask tile in by TMA, output staged (SW64) and stored by TMA: the
    // epilogue's global traffic stays off the L1/LSU path the N = 64 MMAs'
    // shared-memory operand reads contend on.
    const int grp = (int)(warp - 2) >> 2;
    const int q = warp & 3;
    const int lrow = q * 32 + tc::lane_id();
    const bool leader = ((warp - 2) & 3) == 0 && tc::lane_id() == 0;
    // two output staging sub-tiles per group (tile parity): a tile's store
    // may still be reading one while the next tile fills the other
    uint8_t* ob0 = epi + grp * 3 * kSub;
    uint8_t* mb = ob0 + 2 * kSub;
    float bias[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) bias[i] = p.bias ? __ldg(p.bias + grp * 32 + i) : 0.f;
    int it = 0;
    const int ti = lrow >> 3, tj = lrow & 7;  // pixel (ti, tj) of the 16 x 8 tile
    const bool need_pix = p.bits_out != nullptr || p.mask_bits != nullptr;
    TileCursor cur;
    cur.init(blockIdx.x, gridDim.x, p.tiles_x, p.tiles_y);
    for (int tile = blockIdx.x; tile < p.total;
         tile += gridDim.x, ++it, cur.next(p.tiles_x, p.tiles_y)) {
      const int f = cur.f, ty = cur.ty, tx = cur.tx;
      uint8_t* ob = ob0 + (it & 1) * kSub;
      const int ph = ty * kTH + ti, pw = tx * kTW + tj;
      const long long pix = (need_pix && ph < p.H && pw < p.W)
                                ? ((long long)f * p.H + ph) * p.W + pw : -1;
      // bitmask word issued before the accumulator wait (latency hidden)
      const uint32_t mbits = (p.mask_bits && pix >= 0) ? __ldg(p.mask_bits + pix * 2 + grp) : 0u;
      if (leader && p.has_mask) {
        tc::mbar_arrive_expect_tx(&mbar[grp], kSub);
        tc::tma_load_4d(mb, &map_mask, &mbar[grp], grp * 32, tx * kTW, ty * kTH, f);
      }
      const int acc = it & 1;
      tc::mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc::tc_fence_after();
      uint32_t raw0[16], raw1[16];
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + acc * 64 + grp * 32;
      tc::tmem_ld_32x32b_x16(ta, raw0);
      tc::tmem_ld_32x32b_x16(ta + 16, raw1);
      tc::tmem_ld_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&tempty[acc]);
      float v[32];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        v[i] = __uint_as_float(raw0[i]) + bias[i];
        v[16 + i] = __uint_as_float(raw1[i]) + bias[16 + i];
      }
      if (p.relu) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
      }
      if (p.has_mask) {
        tc::mbar_wait(&mbar[grp], it & 1);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint4 mm = *reinterpret_cast<const uint4*>(mb + sw64(lrow, c));
          const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&mm);
#pragma unroll
          for (int i = 0; i < 8; ++i) v[8 * c + i] = __bfloat162float(e[i]) > 0.f ? v[8 * c + i] : 0.f;
        }
      }
      uint32_t o[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) o[j] = tc::pack_bf16(v[2 * j], v[2 * j + 1]);
      if (p.mask_bits) {
#pragma unroll
        for (int j = 0; j < 16; ++j) o[j] &= tc::bits_keep(mbits, j);
      }
      if (p.bits_out && pix >= 0) p.bits_out[pix * 2 + grp] = tc::relu_bits16(o);
      // the store two tiles back (same staging sub-tile) must have finished
      // reading it
      if (leader) tc::bulk_wait_read<1>();
      tc::named_bar(1 + grp, 128);
#pragma unroll
      for (int c = 0; c < 4; ++c)
        *reinterpret_cast<uint4*>(ob + sw64(lrow, c)) =
            make_uint4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
      tc::fence_proxy_async();
      tc::named_bar(1 + grp, 128);
      if (leader) {
        tc::tma_store_4d(&map_out, ob, grp * 32, tx * kTW, ty * kTH, f);
        tc::bulk_commit();
      }
    }
    if (leader) tc::bulk_wait<0>();
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<128>(tmem);
}

// ---------------------------------------------------------------------------
template <int KH, int KW>
__global__ void __launch_bounds__(kThreads, 1)
    wgrad_halo_kernel(const __grid_constant__ CUtensorMap map_x,
                      const __grid_constant__ CUtensorMap map_dy, const WgradParams p) {
  using WC = WgradCfg<KH, KW>;
  constexpr int NROW = WC::TAPS * 64;  // D rows that are weight gradients
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  const int S = p.stages;
  uint8_t* ones = smem + S * WC::STAGE;
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages], tfull;
  __shared__ uint32_t tslot;
  const uint32_t warp = tc::warp_id();
  // contiguous patch range of this CTA (fixed partition -> deterministic)
  const int b0 = (int)((long long)p.total * blockIdx.x / gridDim.x);
  const int b1 = (int)((long long)p.total * (blockIdx.x + 1) / gridDim.x);

  if (warp == 0 && tc::lane_id() == 0) {
    tc::tma_prefetch(&map_x);
    tc::tma_prefetch(&map_dy);
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(&tfull, 1);
    tc::fence_barrier_init();
  }
  if (WC::ONES && warp >= 2) {
    // all-ones bf16 slab (swizzle-invariant) for the bias-gradient rows
    const uint4 one = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
    for (int i = threadIdx.x - 64; i < kOnesBytes / 16; i += kEpiThreads)
      reinterpret_cast<uint4*>(ones)[i] = one;
    tc::fence_proxy_async();
  }
  if (warp == 1) tc::tmem_alloc<512>(&tslot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  tc::pdl_wait();  // (PDL) global memory only after the predecessor completed
  tc::pdl_launch_dependents();
  const uint32_t tmem = tslot;

  auto decode = [&](int b, int& f, int& py, int& px) {
    px = b % p.patches_x;
    const int rest = b / p.patches_x;
    py = rest % p.patches_y;
    f = rest / p.patches_y;
  };

  if (warp == 0) {
    if (tc::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int b = b0; b < b1; ++b) {
        int f, py, px;
        decode(b, f, py, px);
        tc::mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* st = smem + stage * WC::STAGE;
        tc::mbar_arrive_expect_tx(&full[stage], WC::HALO + kDyBytes);
        tc::tma_load_4d(st, &map_x, &full[stage], 0, px * kPW - KW / 2, py * kPW - KH / 2, f);
        tc::tma_load_4d(st + WC::HSTRIDE, &map_dy, &full[stage], 0, px * kPW, py * kPW, f);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = tc::idesc_bf16(128, 64, true, true);
    const uint32_t s0 = tc::smem_u32(smem), o0 = tc::smem_u32(ones);
    int stage = 0;
    uint32_t phase = 0;
    for (int b = b0; b < b1; ++b) {
      tc::mbar_wait(&full[stage], phase);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint32_t hs = s0 + stage * WC::STAGE, ds = hs + WC::HSTRIDE;
#pragma unroll
        for (int mt = 0; mt < WC::MT; ++mt) {
          const int ta = 2 * mt, tb = 2 * mt + 1;
          const int ra = ta / KW, sa = ta % KW;
          uint32_t lbo;
          if (tb < WC::TAPS) {
            lbo = (uint32_t)(((tb / KW - ra) * WC::P + (tb % KW - sa)) * kRowB);
          } else {
            // slab b of k-step j starts at ones + 2j * pitch rows
            lbo = o0 - hs - (uint32_t)((ra * WC::P + sa) * kRowB);
          }
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint64_t ad = tc::smem_desc(hs + ((2 * j + ra) * WC::P + sa) * kRowB, lbo,
                                              WC::P * kRowB, tc::kSw128);
            const uint64_t bd = tc::smem_desc(ds + j * 16 * kRowB, 8192, 1024, tc::kSw128);
            tc::mma_bf16(tmem + mt * 64, ad, bd, idesc, (b > b0 || j > 0) ? 1u : 0u);
          }
        }
        tc::mma_commit(&empty[stage]);
        if (b == b1 - 1) tc::mma_commit(&tfull);
      }
      __syncwarp();
      if (++stage == S) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else {
    // epilogue: rows mt*128 + lane-row of D -> ws[cta][row][co] (rows < NROW),
    // row NROW (first ones row, odd tap counts) -> db_ws[cta][co]
    const int grp = (int)(warp - 2) >> 2;
    const int q = warp & 3;
    const int lrow = q * 32 + tc::lane_id();
    const bool has_k = b1 > b0;
    if (has_k) {
      tc::mbar_wait(&tfull, 0);
      tc::tc_fence_after();
    }
    float* wsb = p.ws + (long long)blockIdx.x * NROW * 64;
#pragma unroll 1
    for (int mt = 0; mt < WC::MT; ++mt) {
      const int row = mt * 128 + lrow;
      uint32_t raw0[16], raw1[16];
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + mt * 64 + grp * 32;
      tc::tmem_ld_32x32b_x16(ta, raw0);
      tc::tmem_ld_32x32b_x16(ta + 16, raw1);
      tc::tmem_ld_wait();
      float* dst = nullptr;
      if (row < NROW) dst = wsb + (long long)row * 64 + grp * 32;
      else if (WC::ONES && row == NROW && p.db_ws)
        dst = p.db_ws + (long long)blockIdx.x * 64 + grp * 32;
      if (dst) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float4 a, c;
          a.x = has_k ? __uint_as_float(raw0[4 * i + 0]) : 0.f;
          a.y = has_k ? __uint_as_float(raw0[4 * i + 1]) : 0.f;
          a.z = has_k ? __uint_as_float(raw0[4 * i + 2]) : 0.f;
          a.w = has_k ? __uint_as_float(raw0[4 * i + 3]) : 0.f;
          c.x = has_k ? __uint_as_float(raw1[4 * i + 0]) : 0.f;
          c.y = has_k ? __uint_as_float(raw1[4 * i + 1]) : 0.f;
          c.z = has_k ? __uint_as_float(raw1[4 * i + 2]) : 0.f;
          c.w = has_k ? __uint_as_float(raw1[4 * i + 3]) : 0.f;
          reinterpret_cast<float4*>(dst)[i] = a;
          reinterpret_cast<float4*>(dst)[4 + i] = c;
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------------------
// Stem conv (space-to-depth 4x4 / s1 over 16-channel pixels, 64 outputs) and
// the 3x3 / s2 / pad 1 max pool in one kernel: the 822 MB stem output of a
// 64-clip step never leaves the SM.  A tile is 16 x 16 stem pixels at origin
// (14 ty - 1, 14 tx - 1) — two 16 x 8 MMA sub-tiles on one 19 x 19 halo —
// whose 3x3 windows hold exactly the 7 x 7 pooled pixels (7 ty + i,
// 7 tx + j); the border row / column is recomputed by the neighbour tile.
// The epilogue rounds the stem to bf16 into a swizzled [16][16][64] shared
// tile (double-buffered across tiles), then pools from it with the same
// scan order and compare / select code as maxpool_fwd_kernel: output and
// argmax bitwise equal to the stem kernel followed by the pool kernel.
constexpr int kSPT = 16;                             // stem tile edge
constexpr int kSPHP = kSPT + 3;                      // halo pitch / rows (19)
constexpr int kSPHalo = kSPHP * kSPHP * 32;          // 11552 B
constexpr int kSPStride = (kSPHalo + 1023) / 1024 * 1024;
constexpr int kSPW = 16 * 64 * 32;                   // 16 taps x [64][16] bf16
constexpr int kSPTile = kSPT * kSPT * 128;           // [16][16][64] bf16
constexpr int kSPEpi = 512;                          // 4 groups x 4 warps (16 channels each)
constexpr int kSPThreads = 64 + kSPEpi;

struct StemPoolParams {
  int tiles_y, tiles_x, total, stages;
  const float* bias;
  int H, W, Ho, Wo;  // stem extent, pooled extent
  uint4* y;          // [frames][Ho][Wo][64] bf16
  uint2* arg;        // [frames][Ho][Wo][64] uint8 (tap 0..8)
};

__global__ void __launch_bounds__(kSPThreads, 1)
    stem_pool_kernel(const __grid_constant__ CUtensorMap map_x,
                     const __grid_constant__ CUtensorMap map_w, const StemPoolParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  uint8_t* sw = smem;
  uint8_t* halo = sw + kSPW;
  uint8_t* st = halo + p.stages * kSPStride;  // 2 stem tiles
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages], tfull[2], tempty[2], wbar;
  __shared__ uint32_t tslot;
  const uint32_t warp = tc::warp_id();
  const int S = p.stages;
  if (warp == 0 && tc::lane_id() == 0) {
    tc::tma_prefetch(&map_x);
    tc::tma_prefetch(&map_w);
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], kSPEpi);
    }
    tc::mbar_init(&wbar, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<256>(&tslot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  tc::pdl_wait();
  tc::pdl_launch_dependents();
  const uint32_t tmem = tslot;

  if (warp == 0) {
    if (tc::elect_one()) {
      tc::mbar_arrive_expect_tx(&wbar, kSPW);
      for (int t = 0; t < 16; ++t) tc::tma_load_2d(sw + t * 2048, &map_w, &wbar, t * 16, 0);
      int stage = 0;
      uint32_t phase = 0;
      TileCursor cur;
      cur.init(blockIdx.x, gridDim.x, p.tiles_x, p.tiles_y);
      for (int tile = blockIdx.x; tile < p.total;
           tile += gridDim.x, cur.next(p.tiles_x, p.tiles_y)) {
        tc::mbar_wait(&empty[stage], phase ^ 1);
        tc::mbar_arrive_expect_tx(&full[stage], kSPHalo);
        // halo origin = tile origin (14 t - 1) - 2 (the s2d conv's window offset)
        tc::tma_load_4d(halo + stage * kSPStride, &map_x, &full[stage], 0, 14 * cur.tx - 3,
                        14 * cur.ty - 3, cur.f);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = tc::idesc_bf16(128, 64, false, false);
    tc::mbar_wait(&wbar, 0);
    const uint32_t w0 = tc::smem_u32(sw), h0 = tc::smem_u32(halo);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int tile = blockIdx.x; tile < p.total; tile += gridDim.x, ++it) {
      const int acc = it & 1;
      tc::mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
      tc::tc_fence_after();
      tc::mbar_wait(&full[stage], phase);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint32_t hs = h0 + stage * kSPStride;
#pragma unroll
        for (int sb = 0; sb < 2; ++sb) {
#pragma unroll
          for (int t = 0; t < 16; ++t) {
            const int r = t >> 2, c = t & 3;
            const uint64_t ad =
                tc::smem_desc(hs + (r * kSPHP + c + 8 * sb) * 32, 16, kSPHP * 32, tc::kSw32);
            const uint64_t bd = tc::smem_desc(w0 + t * 2048, 16, 8 * 32, tc::kSw32);
            tc::mma_bf16(tmem + acc * 128 + sb * 64, ad, bd, idesc, t > 0 ? 1u : 0u);
          }
        }
        tc::mma_commit(&empty[stage]);
        tc::mma_commit(&tfull[acc]);
      }
      __syncwarp();
      if (++stage == S) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else {
    // epilogue: group g owns channels [16 g, 16 g + 16); warp w reads TMEM
    // lanes (w % 4) * 32 .. +32 = sub-tile pixel (i, j) = (lrow / 8, lrow % 8)
    // (16 warps: the pool below is issue-bound and needs the parallelism)
    const int grp = (int)(warp - 2) >> 2;
    const int q = warp & 3;
    const int lrow = q * 32 + tc::lane_id();
    const int et = (int)threadIdx.x - 64;  // 0..511
    const int ti = lrow >> 3, tj = lrow & 7;
    float bias[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) bias[i] = p.bias ? __ldg(p.bias + grp * 16 + i) : 0.f;
    int it = 0;
    TileCursor cur;
    cur.init(blockIdx.x, gridDim.x, p.tiles_x, p.tiles_y);
    for (int tile = blockIdx.x; tile < p.total;
         tile += gridDim.x, ++it, cur.next(p.tiles_x, p.tiles_y)) {
      const int acc = it & 1;
      uint8_t* tb = st + (it & 1) * kSPTile;
      tc::mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc::tc_fence_after();
      uint32_t raw[2][16];
#pragma unroll
      for (int sb = 0; sb < 2; ++sb)
        tc::tmem_ld_32x32b_x16(tmem + ((uint32_t)(q * 32) << 16) + acc * 128 + sb * 64 + grp * 16,
                               raw[sb]);
      tc::tmem_ld_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&tempty[acc]);
#pragma unroll
      for (int sb = 0; sb < 2; ++sb) {
        uint32_t o[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          o[k] = tc::pack_bf16(__uint_as_float(raw[sb][2 * k]) + bias[2 * k],
                               __uint_as_float(raw[sb][2 * k + 1]) + bias[2 * k + 1]);
        const int pix = ti * kSPT + 8 * sb + tj;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int ch = grp * 2 + k;  // 16-byte chunk (8 channels) of the 128-byte pixel
          *reinterpret_cast<uint4*>(tb + pix * 128 + ((ch ^ (pix & 7)) << 4)) =
              make_uint4(o[4 * k], o[4 * k + 1], o[4 * k + 2], o[4 * k + 3]);
        }
      }
      tc::named_bar(1, kSPEpi);  // the stem tile is complete
      // pool: 7 x 7 pixels x 8 chunks of 8 channels
      const int r0 = 14 * cur.ty - 1, c0 = 14 * cur.tx - 1;
      // interior tiles (no padded tap in any window): unchecked, unrolled
      const bool inner = r0 >= 0 && c0 >= 0 && r0 + 15 <= p.H && c0 + 15 <= p.W &&
                         7 * cur.ty + 7 <= p.Ho && 7 * cur.tx + 7 <= p.Wo;
      for (int item = et; item < 7 * 7 * 8; item += kSPEpi) {
        const int pi = item / 56, rem = item - pi * 56, pj = rem >> 3, ck = rem & 7;
        const int ho = 7 * cur.ty + pi, wo = 7 * cur.tx + pj;
        uint32_t best[4], barg[4];
        auto tap = [&](int dh, int dw, bool seed) {
          const int pix = (2 * pi + dh) * kSPT + 2 * pj + dw;
          const uint4 v = *reinterpret_cast<const uint4*>(tb + pix * 128 + ((ck ^ (pix & 7)) << 4));
          const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
          const uint32_t tt = (uint32_t)(dh * 3 + dw) * 0x00010001u;
          if (seed) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              best[k] = vw[k];
              barg[k] = tt;
            }
          } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const uint32_t m = __hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&vw[k]),
                                             *reinterpret_cast<const __nv_bfloat162*>(&best[k]));
              best[k] = (vw[k] & m) | (best[k] & ~m);
              barg[k] = (tt & m) | (barg[k] & ~m);
            }
          }
        };
        if (inner) {
#pragma unroll
          for (int t = 0; t < 9; ++t) tap(t / 3, t % 3, t == 0);
        } else {
          if (ho >= p.Ho || wo >= p.Wo) continue;
          bool first = true;
#pragma unroll
          for (int dh = 0; dh < 3; ++dh) {
            const int h = r0 + 2 * pi + dh;
            if (h < 0 || h >= p.H) continue;
#pragma unroll
            for (int dw = 0; dw < 3; ++dw) {
              const int w = c0 + 2 * pj + dw;
              if (w < 0 || w >= p.W) continue;
              tap(dh, dw, first);
              first = false;
            }
          }
        }
        const long long o = (((long long)cur.f * p.Ho + ho) * p.Wo + wo) * 8 + ck;
        __stcs(p.y + o, make_uint4(best[0], best[1], best[2], best[3]));
        __stcs(p.arg + o, make_uint2(__byte_perm(barg[0], barg[1], 0x6420),
                                     __byte_perm(barg[2], barg[3], 0x6420)));
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<256>(tmem);
}

// ---------------------------------------------------------------------------
// Stem weight gradient with the max-pool backward fused into its dY operand:
// wgrad_halo_kernel<4, 1> whose 8 x 8-pixel dY patches are not loaded from a
// stored stem-output gradient but gathered from the pooled gradient and the
// argmax bytes by the (otherwise idle until the end) epilogue warps — two
// groups of 4 warps taking alternate patches, each thread one 2 x 2 block x 8
// channels (poolbwd::block2x2, the pool kernels' routing and order, so the
// bf16 operand is bitwise the stored one).  The 822 MB stem gradient of a
// 64-clip step is neither written nor read.  `full` completes on the x halo
// bytes (producer) plus one arrival of the group that wrote the patch.
struct StemWgradPoolParams {
  WgradParams w;
  const uint4* gy;   // pooled gradient [frames][Ho][Wo][64] bf16
  const uint2* arg;  // argmax bytes [frames][Ho][Wo][64]
  int Ho, Wo, H, W;  // pooled / stem extents (H = 2 Ho, W = 2 Wo)
};

constexpr int kSWGroups = 4;                       // dY-producer / epilogue groups of 4 warps
constexpr int kSWThreads = 64 + 128 * kSWGroups;

__global__ void __launch_bounds__(kSWThreads, 1)
    stem_wgrad_pool_kernel(const __grid_constant__ CUtensorMap map_s,
                           const __grid_constant__ CUtensorMap map_gy,
                           const __grid_constant__ CUtensorMap map_arg,
                           const StemWgradPoolParams sp) {
  constexpr int KH = 4, KW = 1;
  using WC = WgradCfg<KH, KW>;
  // per stage: the x4 halo (built here), dY, and the raw s2d halo it is
  // built from: 11 rows x 11 pixels x 16 channels (TMA, no swizzle)
  constexpr int kSRows = kPW + KH - 1, kSCols = kPW + 3;  // 11 x 11
  constexpr int kSBytes = kSRows * kSCols * 32;           // 3872
  // and the patch's 5 x 5 pool windows of the pooled gradient (bf16) and
  // the argmax bytes, staged by TMA so the routing reads shared memory
  constexpr int kGyOff = 3968, kGyBytes = 25 * 128, kArgOff = kGyOff + kGyBytes,
                kArgBytes = 25 * 64;
  constexpr int kStage = WC::STAGE + 9216;
  static_assert(kArgOff + kArgBytes <= 9216, "stem wgrad stage");
  constexpr int NROW = WC::TAPS * 64;
  static_assert(!WC::ONES, "the stem's bias gradient comes from the ones channel");
  const WgradParams& p = sp.w;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  const int S = p.stages;
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages], sfull[kMaxStages], tfull;
  __shared__ uint32_t tslot;
  const uint32_t warp = tc::warp_id();
  const int b0 = (int)((long long)p.total * blockIdx.x / gridDim.x);
  const int b1 = (int)((long long)p.total * (blockIdx.x + 1) / gridDim.x);

  if (warp == 0 && tc::lane_id() == 0) {
    tc::tma_prefetch(&map_s);
    tc::tma_prefetch(&map_gy);
    tc::tma_prefetch(&map_arg);
    for (int s = 0; s < S; ++s) {
      tc::mbar_init(&full[s], 1);   // the group that built the stage's operands
      tc::mbar_init(&empty[s], 1);
      tc::mbar_init(&sfull[s], 1);  // raw s2d halo landed
    }
    tc::mbar_init(&tfull, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<512>(&tslot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  tc::pdl_wait();
  tc::pdl_launch_dependents();
  const uint32_t tmem = tslot;

  auto decode = [&](int b, int& f, int& py, int& px) {
    px = b % p.patches_x;
    const int rest = b / p.patches_x;
    py = rest % p.patches_y;
    f = rest / p.patches_y;
  };

  if (warp == 0) {
    if (tc::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int b = b0; b < b1; ++b) {
        int f, py, px;
        decode(b, f, py, px);
        tc::mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* raw = smem + stage * kStage + WC::STAGE;
        tc::mbar_arrive_expect_tx(&sfull[stage], kSBytes + kGyBytes + kArgBytes);
        // x4 pixel (h, w) = s2d pixels (h, w - 2 .. w + 1): origin w - 2, h - 2
        tc::tma_load_4d(raw, &map_s, &sfull[stage], 0, px * kPW - 2, py * kPW - KH / 2, f);
        // pool windows 4 py .. 4 py + 4 x 4 px .. 4 px + 4 (out of range: zeros,
        // never routed)
        tc::tma_load_4d(raw + kGyOff, &map_gy, &sfull[stage], 0, 4 * px, 4 * py, f);
        tc::tma_load_4d(raw + kArgOff, &map_arg, &sfull[stage], 0, 4 * px, 4 * py, f);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = tc::idesc_bf16(128, 64, true, true);
    const uint32_t s0 = tc::smem_u32(smem);
    int stage = 0;
    uint32_t phase = 0;
    for (int b = b0; b < b1; ++b) {
      tc::mbar_wait(&full[stage], phase);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint32_t hs = s0 + stage * kStage, ds = hs + WC::HSTRIDE;
#pragma unroll
        for (int mt = 0; mt < WC::MT; ++mt) {
          const int ta = 2 * mt, tb = 2 * mt + 1;
          const int ra = ta / KW, sa = ta % KW;
          const uint32_t lbo = (uint32_t)(((tb / KW - ra) * WC::P + (tb % KW - sa)) * kRowB);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint64_t ad = tc::smem_desc(hs + ((2 * j + ra) * WC::P + sa) * kRowB, lbo,
                                              WC::P * kRowB, tc::kSw128);
            const uint64_t bd = tc::smem_desc(ds + j * 16 * kRowB, 8192, 1024, tc::kSw128);
            tc::mma_bf16(tmem + mt * 64, ad, bd, idesc, (b > b0 || j > 0) ? 1u : 0u);
          }
        }
        tc::mma_commit(&empty[stage]);
        if (b == b1 - 1) tc::mma_commit(&tfull);
      }
      __syncwarp();
      if (++stage == S) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else {
    const int grp = (int)(warp - 2) >> 2;
    const int gt = (int)threadIdx.x - 64 - 128 * grp;  // 0..127 within the group
    // ---- dY producer: group g writes patches b0 + g, b0 + g + kSWGroups, ... ----
    // (the patch's pool windows arrive with its raw s2d halo on sfull)
    {
      const int blk = gt >> 3, ck = gt & 7;         // 2 x 2 block (4 x 4 per patch), chunk
      const int by = blk >> 2, bx = blk & 3;
      for (int b = b0 + grp; b < b1; b += kSWGroups) {
        const int k = b - b0, stage = k % S;
        const uint32_t phase = (uint32_t)((k / S) & 1);
        int f, py, px;
        decode(b, f, py, px);
        const int a = 4 * py + by, bb = 4 * px + bx;  // window of the block's top-left pixel
        uint4 v[4] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0),
                      make_uint4(0, 0, 0, 0)};
        uint8_t* hsb = smem + stage * kStage;
        const uint8_t* raw = hsb + WC::STAGE;
        tc::mbar_wait(&empty[stage], phase ^ 1);
        tc::mbar_wait(&sfull[stage], phase);
        if (a < sp.Ho && bb < sp.Wo) {
          poolbwd::Block2x2 kb;
          const uint4* gw = reinterpret_cast<const uint4*>(raw + kGyOff);
          const uint2* aw = reinterpret_cast<const uint2*>(raw + kArgOff);
          const int o00 = (by * 5 + bx) * 8 + ck;
          kb.right = bb + 1 < sp.Wo;
          kb.down = a + 1 < sp.Ho;
          kb.a00 = aw[o00];
          kb.g00 = gw[o00];
          kb.a01 = kb.a10 = kb.a11 = make_uint2(0xFFFFFFFFu, 0xFFFFFFFFu);  // no tap matches
          kb.g01 = kb.g10 = kb.g11 = make_uint4(0, 0, 0, 0);
          if (kb.right) {
            kb.a01 = aw[o00 + 8];
            kb.g01 = gw[o00 + 8];
          }
          if (kb.down) {
            kb.a10 = aw[o00 + 40];
            kb.g10 = gw[o00 + 40];
            if (kb.right) {
              kb.a11 = aw[o00 + 48];
              kb.g11 = gw[o00 + 48];
            }
          }
          poolbwd::route2x2(kb, v);
        }
        uint8_t* ds = hsb + WC::HSTRIDE;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int r = (2 * by + (q >> 1)) * kPW + 2 * bx + (q & 1);  // patch pixel row
          *reinterpret_cast<uint4*>(ds + r * kRowB + ((ck ^ (r & 7)) << 4)) = v[q];
        }
        // x4 halo: row r = h * 8 + w (128 B, 128-byte swizzle), chunk 2t + i =
        // s2d pixel (h, w + t) channels 8i..8i+7 of the raw halo
        for (int e = gt; e < kSRows * kPW * 8; e += 128) {
          const int r = e >> 3, c = e & 7, h = r >> 3, w = r & 7;
          const uint4 v4 = *reinterpret_cast<const uint4*>(raw + (h * kSCols + w + (c >> 1)) * 32 +
                                                           (c & 1) * 16);
          *reinterpret_cast<uint4*>(hsb + r * kRowB + ((c ^ (r & 7)) << 4)) = v4;
        }
        tc::fence_proxy_async();
        tc::named_bar(1 + grp, 128);
        if (gt == 0) tc::mbar_arrive(&full[stage]);
      }
    }
    // ---- epilogue: rows mt*128 + lane-row of D -> ws[cta][row][co] ----
    const int q = warp & 3;
    const int lrow = q * 32 + tc::lane_id();
    const bool has_k = b1 > b0;
    if (has_k) {
      tc::mbar_wait(&tfull, 0);
      tc::tc_fence_after();
    }
    float* wsb = p.ws + (long long)blockIdx.x * NROW * 64;
#pragma unroll 1
    for (int mt = 0; mt < WC::MT; ++mt) {
      const int row = mt * 128 + lrow;
      uint32_t raw0[16];  // 16 columns per group
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + mt * 64 + grp * 16;
      tc::tmem_ld_32x32b_x16(ta, raw0);
      tc::tmem_ld_wait();
      if (row < NROW) {
        float* dst = wsb + (long long)row * 64 + grp * 16;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float4 a;
          a.x = has_k ? __uint_as_float(raw0[4 * i + 0]) : 0.f;
          a.y = has_k ? __uint_as_float(raw0[4 * i + 1]) : 0.f;
          a.z = has_k ? __uint_as_float(raw0[4 * i + 2]) : 0.f;
          a.w = has_k ? __uint_as_float(raw0[4 * i + 3]) : 0.f;
          reinterpret_cast<float4*>(dst)[i] = a;
        }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<512>(tmem);
}

}  // namespace halo
}  // namespace tsm
