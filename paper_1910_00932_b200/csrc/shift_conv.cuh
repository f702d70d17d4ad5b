// Fused temporal shift + 1x1 conv for 64 -> 64 channels with narrow shift
// groups (the TSM-R50 res2.0 conv1: F = B = 8 of 64 channels, 56 x 56).
//
// The generic GEMM loads the shifted operand as 8-channel slabs, i.e. TMA
// boxes of 16-byte rows (eight requests per pixel).  Here a 16 x 8 pixel
// tile is loaded as three full 128-byte-row boxes of a 5-D map (C, W, H, T,
// N): frame t, t - 1 and t + 1 (out-of-clip frames zero-filled by TMA: the
// shift's zero boundary, kernels.cpp:127-157).  Only the first 16-channel
// K chunk mixes sources, so it becomes up to three MMAs — the t - 1 tile
// against the weights of channels [0, F), the t + 1 tile against [F, F+B),
// the t tile against [F+B, 16) — built once per CTA as masked copies of the
// resident weight slab; chunks 1..3 are plain MMAs on the t tile.
//
// DG (input gradient of that conv, adjoint shift + skip, kernels.cpp:
// 127-157): dx[t] = mask * (dy[t] W0 + dy[t+1] Wn + dy[t-1] Wp + skip[t]),
// the adjoint shift moving the output channels [0, F) from frame t + 1 and
// [F, F+B) from t - 1; Wn / Wp / W0 are the dgrad weights with every output
// channel outside the group zeroed (three masked copies, built once per CTA),
// so each source tile is a full K = 64 GEMM (12 MMAs per tile against an
// HBM time of ~4x that).  The skip gradient comes in by TMA per group one
// tile ahead (double-buffered).
//
//   warp 0: TMA producer (weights once, three boxes per tile)
//   warp 1: MMA issuer (tcgen05, accumulator double-buffered in TMEM)
//   warps 2..9: weight-mask build (once), then the halo kernels' epilogue:
//            bias, ReLU, ReLU bitmask, bf16 staging, TMA store.
#pragma once
#include "halo_conv.cuh"

namespace tsm {
namespace halo {

constexpr int kS1Tile = kTW * kTH * kRowB;  // 16 KB: 128 pixels x 64 channels
constexpr int kS1Stage = 3 * kS1Tile;       // frames t, t - 1, t + 1

struct Shift1Params {
  int tiles_y, tiles_x, total, stages;
  int T;                // frames per clip
  int F, B;             // shift groups: [0, F) from t - 1, [F, F + B) from t + 1
  const float* bias;
  int relu, H, W;
  uint32_t* bits_out;         // nullable (forward): ReLU bitmask of the output, [pixel][2]
  const uint32_t* mask_bits;  // nullable (DG): input-side ReLU mask, [pixel][2] words
  int has_res;                // DG: add the skip gradient (map_res)
};

template <bool DG>
__global__ void __launch_bounds__(kThreads, 1)
    shift1x1_kernel(const __grid_constant__ CUtensorMap map_x,
                    const __grid_constant__ CUtensorMap map_w,
                    const __grid_constant__ CUtensorMap map_out,
                    const __grid_constant__ CUtensorMap map_res, const Shift1Params p) {
  constexpr int kW = 64 * kRowB;                       // one [64][64] weight slab
  constexpr int kWBytes = DG ? 4 * kW : 2 * kW;        // loaded + variants
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  uint8_t* sw = smem;                 // [64][64] weights as loaded, SW128
  uint8_t* sv = sw + kW;              // fwd: chunk-0 variants [Wm | Wp | W0 | 0];
                                      // DG: masked copies W0, Wn, Wp
  uint8_t* tiles = smem + kWBytes;    // [stages][3 tiles]
  uint8_t* epi = tiles + p.stages * kS1Stage;  // [grp][2 staging (+ 2 skip) sub-tiles]
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages], tfull[2], tempty[2],
      wbar, rbar[2][2];
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
      tc::mbar_init(&rbar[a][0], 1);
      tc::mbar_init(&rbar[a][1], 1);
    }
    tc::mbar_init(&wbar, 1);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<128>(&tslot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  tc::pdl_wait();
  tc::pdl_launch_dependents();
  const uint32_t tmem = tslot;

  if (warp == 0) {
    if (tc::elect_one()) {
      tc::mbar_arrive_expect_tx(&wbar, kW);
      tc::tma_load_2d(sw, &map_w, &wbar, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      TileCursor cur;
      cur.init(blockIdx.x, gridDim.x, p.tiles_x, p.tiles_y);
      for (int tile = blockIdx.x; tile < p.total;
           tile += gridDim.x, cur.next(p.tiles_x, p.tiles_y)) {
        const int n = cur.f / p.T, t = cur.f - n * p.T;
        const int x0 = cur.tx * kTW, y0 = cur.ty * kTH;
        tc::mbar_wait(&empty[stage], phase ^ 1);
        tc::mbar_arrive_expect_tx(&full[stage], kS1Stage);
        uint8_t* d = tiles + stage * kS1Stage;
        // [frame t | t - 1 | t + 1]
        tc::tma_load_5d(d, &map_x, &full[stage], 0, x0, y0, t, n);
        tc::tma_load_5d(d + kS1Tile, &map_x, &full[stage], 0, x0, y0, t - 1, n);
        tc::tma_load_5d(d + 2 * kS1Tile, &map_x, &full[stage], 0, x0, y0, t + 1, n);
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = tc::idesc_bf16(128, 64, false, false);
    // the weight variants are built by the epilogue warps (named barrier 3)
    tc::named_bar(3, 32 + kEpiThreads);
    tc::tc_fence_after();
    const uint32_t w0 = tc::smem_u32(sw), v0 = tc::smem_u32(sv), t0 = tc::smem_u32(tiles);
    const bool use_m = p.F > 0, use_p = p.B > 0;
    const bool use_0 = DG ? p.F + p.B < 64 : p.F + p.B < 16;
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
        const uint32_t a = t0 + stage * kS1Stage;
        const uint32_t d = tmem + acc * 64;
        auto adesc = [&](uint32_t base) {
          return tc::smem_desc(base, 16, kTW * kRowB, tc::kSw128);
        };
        auto bdesc = [&](uint32_t base) { return tc::smem_desc(base, 16, 8 * kRowB, tc::kSw128); };
        uint32_t accum = 0;
        if constexpr (DG) {
          // (tile, weights): (t, W0), (t + 1, Wn), (t - 1, Wp)
          auto gemm = [&](uint32_t at, uint32_t wv) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              tc::mma_bf16(d, adesc(at + j * 32), bdesc(wv + j * 32), idesc, accum);
              accum = 1;
            }
          };
          if (use_0) gemm(a, v0);
          if (use_m) gemm(a + 2 * kS1Tile, v0 + kW);
          if (use_p) gemm(a + kS1Tile, v0 + 2 * kW);
        } else {
          if (use_m) {
            tc::mma_bf16(d, adesc(a + kS1Tile), bdesc(v0), idesc, accum);
            accum = 1;
          }
          if (use_p) {
            tc::mma_bf16(d, adesc(a + 2 * kS1Tile), bdesc(v0 + 32), idesc, accum);
            accum = 1;
          }
          if (use_0) {
            tc::mma_bf16(d, adesc(a), bdesc(v0 + 64), idesc, accum);
            accum = 1;
          }
#pragma unroll
          for (int j = 1; j < 4; ++j)
            tc::mma_bf16(d, adesc(a + j * 32), bdesc(w0 + j * 32), idesc, 1u);
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
    tc::mbar_wait(&wbar, 0);
    if constexpr (DG) {
      // masked copies: variant v keeps output-channel rows co of its group
      // (W0: [F+B, 64), Wn: [0, F), Wp: [F, F+B)); rows are whole 128-byte
      // swizzled lines, so a row copy keeps the swizzle
      for (int i = threadIdx.x - 64; i < 3 * 64 * 8; i += kEpiThreads) {
        const int v = i >> 9, co = (i >> 3) & 63, c = i & 7;
        const int lo = v == 0 ? p.F + p.B : (v == 1 ? 0 : p.F);
        const int hi = v == 0 ? 64 : (v == 1 ? p.F : p.F + p.B);
        const int off = co * kRowB + c * 16;
        const uint4 val = (co >= lo && co < hi) ? *reinterpret_cast<const uint4*>(sw + off)
                                                : make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(sv + v * kW + off) = val;
      }
    } else {
      // chunk-0 variants [Wm | Wp | W0 | 0] in one 64-channel slab (same
      // SW128 layout): K element k of variant v keeps channel k - 16 v of
      // row co iff it lies in the variant's shift group
      for (int i = threadIdx.x - 64; i < 64 * 8; i += kEpiThreads) {
        const int co = i >> 3, c = i & 7;  // 16-byte chunk c (K 8c .. 8c + 7) of row co
        const int v = c >> 1, k0 = 8 * (c & 1);  // variant, channel offset inside chunk 0
        uint4 val = make_uint4(0, 0, 0, 0);
        if (v < 3) {
          const int lo = v == 0 ? 0 : (v == 1 ? p.F : p.F + p.B);
          const int hi = v == 0 ? p.F : (v == 1 ? p.F + p.B : 16);
          if (k0 >= lo && k0 + 8 <= hi)  // groups are multiples of 8 channels
            val = *reinterpret_cast<const uint4*>(sw + co * kRowB + (((c & 1) ^ (co & 7)) << 4));
        }
        *reinterpret_cast<uint4*>(sv + co * kRowB + ((c ^ (co & 7)) << 4)) = val;
      }
    }
    tc::fence_proxy_async();
    tc::named_bar(3, 32 + kEpiThreads);

    // epilogue: group g owns channels [32 g, 32 g + 32); warp w reads TMEM
    // lanes (w % 4) * 32 .. +32 = tile pixel (lrow / 8, lrow % 8)
    const int grp = (int)(warp - 2) >> 2;
    const int q = warp & 3;
    const int lrow = q * 32 + tc::lane_id();
    const bool leader = ((warp - 2) & 3) == 0 && tc::lane_id() == 0;
    uint8_t* ob0 = epi + grp * (DG ? 4 : 2) * kSub;
    uint8_t* rb0 = ob0 + 2 * kSub;  // (DG) skip-gradient sub-tiles, one tile ahead
    float bias[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) bias[i] = p.bias ? __ldg(p.bias + grp * 32 + i) : 0.f;
    const int ti = lrow >> 3, tj = lrow & 7;
    const bool need_pix = p.bits_out != nullptr || p.mask_bits != nullptr;
    int it = 0;
    TileCursor cur, nxt;
    cur.init(blockIdx.x, gridDim.x, p.tiles_x, p.tiles_y);
    nxt = cur;
    const bool skip = DG && p.has_res;
    auto load_skip = [&](int slot, const TileCursor& c) {
      tc::mbar_arrive_expect_tx(&rbar[grp][slot], kSub);
      tc::tma_load_4d(rb0 + slot * kSub, &map_res, &rbar[grp][slot], grp * 32, c.tx * kTW,
                      c.ty * kTH, c.f);
    };
    if (skip && leader && (int)blockIdx.x < p.total) load_skip(0, cur);
    for (int tile = blockIdx.x; tile < p.total;
         tile += gridDim.x, ++it, cur.next(p.tiles_x, p.tiles_y)) {
      uint8_t* ob = ob0 + (it & 1) * kSub;
      // the next tile's skip sub-tile: its slot was last read in tile it - 1
      // (before this group's named barriers there)
      nxt.next(p.tiles_x, p.tiles_y);
      if (skip && leader && tile + (int)gridDim.x < p.total) load_skip((it + 1) & 1, nxt);
      const int ph = cur.ty * kTH + ti, pw = cur.tx * kTW + tj;
      const long long pix = (need_pix && ph < p.H && pw < p.W)
                                ? ((long long)cur.f * p.H + ph) * p.W + pw : -1;
      const uint32_t mbits = (p.mask_bits && pix >= 0) ? __ldg(p.mask_bits + pix * 2 + grp) : 0u;
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
      if (skip) {
        const uint8_t* rb = rb0 + (it & 1) * kSub;
        tc::mbar_wait(&rbar[grp][it & 1], (it >> 1) & 1);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint4 rr = *reinterpret_cast<const uint4*>(rb + sw64(lrow, c));
          const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&rr);
#pragma unroll
          for (int i = 0; i < 8; ++i) v[8 * c + i] += __bfloat162float(e[i]);
        }
      }
      if (p.relu) {
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
      }
      uint32_t o[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) o[j] = tc::pack_bf16(v[2 * j], v[2 * j + 1]);
      if (p.mask_bits) {
#pragma unroll
        for (int j = 0; j < 16; ++j) o[j] &= tc::bits_keep(mbits, j);
      }
      if (p.bits_out && pix >= 0) p.bits_out[pix * 2 + grp] = tc::relu_bits16(o);
      // the store two tiles back (same staging sub-tile) must have finished;
      // (DG) every thread has read the skip sub-tile before it is reloaded
      if (leader) tc::bulk_wait_read<1>();
      tc::named_bar(1 + grp, 128);
#pragma unroll
      for (int c = 0; c < 4; ++c)
        *reinterpret_cast<uint4*>(ob + sw64(lrow, c)) =
            make_uint4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
      tc::fence_proxy_async();
      tc::named_bar(1 + grp, 128);
      if (leader) {
        tc::tma_store_4d(&map_out, ob, grp * 32, cur.tx * kTW, cur.ty * kTH, cur.f);
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
// Weight (and bias) gradient of the same conv: dW[co][ci] = sum_p dY(p)[co]
// shift(x)(p)[ci].  Per 8 x 8 patch (K = 64 pixels, MN-major operands) the
// frame tiles x(t), x(t-1), x(t+1) and dY(t) come in as 128-byte-row boxes
// (out-of-clip frames zero-filled); two M = 128 MMAs per K step accumulate
// D0 = [x(t) | x(t-1)]^T dY and D1 = [x(t+1) | 1]^T dY in TMEM over the
// CTA's patches — the all-ones rows give the bias gradient —
// and the CTA's 256 x 64 fp32 partial goes to ws.  wgrad_shift1_reduce sums
// the partials in CTA order (deterministic) and keeps each input channel's
// live row: ci < F from x(t-1), F <= ci < F+B from x(t+1), the rest x(t).
constexpr int kS1Patch = kPW * kPW * kRowB;  // 8 KB: 64 pixels x 64 channels
constexpr int kS1WStage = 4 * kS1Patch;      // x(t), x(t-1), x(t+1), dY

struct Shift1WgradParams {
  int patches_y, patches_x, total, stages, T;
  float* ws;  // [grid][256][64]
};

__global__ void __launch_bounds__(kThreads, 1)
    wgrad_shift1_kernel(const __grid_constant__ CUtensorMap map_x,
                        const __grid_constant__ CUtensorMap map_dy, const Shift1WgradParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  const int S = p.stages;
  uint8_t* ones = smem + S * kS1WStage;
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages], tfull;
  __shared__ uint32_t tslot;
  const uint32_t warp = tc::warp_id();
  // patches blockIdx.x + k * gridDim.x: the CTAs sweep one window of
  // consecutive patches, so a frame tile read as x(t +- 1) by one CTA is
  // still in L2 when another reads it as x(t) (a contiguous range per CTA
  // re-fetched each frame three times from HBM: 118 us)
  const int b0 = (int)blockIdx.x, bstep = (int)gridDim.x;

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
  if (warp >= 2) {  // all-ones bf16 tile (swizzle-invariant) for the bias rows
    const uint4 one = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
    for (int i = threadIdx.x - 64; i < kS1Patch / 16; i += kEpiThreads)
      reinterpret_cast<uint4*>(ones)[i] = one;
    tc::fence_proxy_async();
  }
  if (warp == 1) tc::tmem_alloc<128>(&tslot);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  tc::pdl_wait();
  tc::pdl_launch_dependents();
  const uint32_t tmem = tslot;

  if (warp == 0) {
    if (tc::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int b = b0; b < p.total; b += bstep) {
        const int px = b % p.patches_x, rest = b / p.patches_x;
        const int py = rest % p.patches_y, f = rest / p.patches_y;
        const int n = f / p.T, t = f - n * p.T;
        tc::mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* st = smem + stage * kS1WStage;
        tc::mbar_arrive_expect_tx(&full[stage], kS1WStage);
        const int x0 = px * kPW, y0 = py * kPW;
        tc::tma_load_5d(st, &map_x, &full[stage], 0, x0, y0, t, n);
        tc::tma_load_5d(st + kS1Patch, &map_x, &full[stage], 0, x0, y0, t - 1, n);
        tc::tma_load_5d(st + 2 * kS1Patch, &map_x, &full[stage], 0, x0, y0, t + 1, n);
        tc::tma_load_5d(st + 3 * kS1Patch, &map_dy, &full[stage], 0, x0, y0, t, n);
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
    for (int b = b0; b < p.total; b += bstep) {
      tc::mbar_wait(&full[stage], phase);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint32_t st = s0 + stage * kS1WStage, ds = st + 3 * kS1Patch;
        const uint32_t xp = st + 2 * kS1Patch;
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // 16 pixels (two patch rows) per K step
          const uint32_t acc = (b > b0 || j > 0) ? 1u : 0u;
          const uint64_t bd = tc::smem_desc(ds + j * 16 * kRowB, 8192, 8 * kRowB, tc::kSw128);
          // M atoms at LBO: x(t) | x(t-1), then x(t+1) | ones
          const uint64_t a0 = tc::smem_desc(st + j * 16 * kRowB, kS1Patch, 8 * kRowB, tc::kSw128);
          const uint64_t a1 = tc::smem_desc(xp + j * 16 * kRowB, o0 - xp, 8 * kRowB, tc::kSw128);
          tc::mma_bf16(tmem, a0, bd, idesc, acc);
          tc::mma_bf16(tmem + 64, a1, bd, idesc, acc);
        }
        tc::mma_commit(&empty[stage]);
        if (b + bstep >= p.total) tc::mma_commit(&tfull);
      }
      __syncwarp();
      if (++stage == S) {
        stage = 0;
        phase ^= 1;
      }
    }
  } else {
    // rows mt * 128 + lane-row of D -> ws[cta][row][co]
    const int grp = (int)(warp - 2) >> 2;
    const int q = warp & 3;
    const int lrow = q * 32 + tc::lane_id();
    const bool has_k = b0 < p.total;
    if (has_k) {
      tc::mbar_wait(&tfull, 0);
      tc::tc_fence_after();
    }
    float* wsb = p.ws + (long long)blockIdx.x * 256 * 64;
#pragma unroll 1
    for (int mt = 0; mt < 2; ++mt) {
      uint32_t raw0[16], raw1[16];
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + mt * 64 + grp * 32;
      tc::tmem_ld_32x32b_x16(ta, raw0);
      tc::tmem_ld_32x32b_x16(ta + 16, raw1);
      tc::tmem_ld_wait();
      float* dst = wsb + (long long)(mt * 128 + lrow) * 64 + grp * 32;
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
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc<128>(tmem);
}

// dw[co][ci] = sum over CTAs of ws[cta][row(ci)][co]; db[co] from the first
// all-ones row (192).  Block = 32 outputs (consecutive co) x 8 warps: warp w
// sums CTAs c = w mod 8 in order, then warp 0 adds the eight partials in
// order (deterministic; 130 blocks keep the 9.7 MB of partials streaming).
__global__ void __launch_bounds__(256)
    wgrad_shift1_reduce_kernel(const float* __restrict__ ws, float* __restrict__ dw,
                               float* __restrict__ db, int grid, int F, int B) {
  __shared__ float part[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.x * 32 + lane;
  int row, co;
  float* out = nullptr;
  if (i < 64 * 64) {
    const int ci = i >> 6;
    co = i & 63;
    row = ci < F ? 64 + ci : (ci < F + B ? 128 + ci : ci);
    out = dw + co * 64 + ci;
  } else {
    co = (i - 64 * 64) & 63;
    row = 192;
    if (i < 64 * 64 + 64 && db) out = db + co;
  }
  const float* src = ws + (long long)row * 64 + co;
  float acc = 0.f;
  for (int c = w; c < grid; c += 8) acc += __ldg(src + (long long)c * 256 * 64);
  part[w][lane] = acc;
  __syncthreads();
  if (w == 0 && out) {
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) sum += part[j][lane];
    *out = sum;
  }
}

}  // namespace halo
}  // namespace tsm
