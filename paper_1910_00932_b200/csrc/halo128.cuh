// Halo-tile 3x3 stride-1 convolution for 128 -> 128 channels (the TSM-R50
// res3 conv2 forward and its stride-1 input gradient, 28 x 28 pixels).
//
// The im2col GEMM re-reads every input pixel nine times through TMA (one
// 16 KB im2col box per tap and 64-channel slab); here one 18 x 10-pixel halo
// per 16 x 8 output tile (two 64-channel TMA boxes, 46 KB) is loaded once and
// the nine taps are descriptor offsets into it, as in halo_conv_kernel.  The
// 288 KB of weights do not fit in shared memory beside the halo ring, so they
// stream through a ring of weight tiles (18 per output tile, L2 resident).
// M = 128 pixels per CTA, N = 128 output channels, K = 9 taps x 128.
//
// CG = 2 (default): a CTA pair (2-CTA cluster) shares one M = 256 MMA; each
// CTA holds the halo of its own output tile and half of every weight tile
// ([64 co][64 ci]) at the same shared-memory offsets, so the weight stream
// per CTA halves (190 KB of TMA intake per 128-pixel tile instead of 334 KB
// single, 432 KB for the im2col pair).  The leader (rank 0) issues the MMAs,
// its full barriers count both CTAs' bytes and its commits arrive on both
// CTAs' barriers.  The pair walks tiles 2 u + rank; an odd last tile pairs
// with a padding tile that loads a valid halo and stores nothing.
//
//   warp 0: TMA producer (halo ring of 2, weight ring of p.bstages)
//   warp 1: MMA issuer (tcgen05, accumulator double-buffered in TMEM)
//   warps 2..9: epilogue, two groups of 64 output channels: bias, ReLU,
//            optional ReLU bitmask of the output / input mask, bf16 staging,
//            TMA store per 32-channel sub-tile.
#pragma once
#include "halo_conv.cuh"

namespace tsm {
namespace halo {

constexpr int kH128HP = kTW + 2, kH128HR = kTH + 2;           // 10 x 18 halo
constexpr int kH128SlabBytes = kH128HP * kH128HR * 128;       // 23040 (64 channels)
constexpr int kH128SlabStride = (kH128SlabBytes + 1023) / 1024 * 1024;
constexpr int kH128HaloStride = 2 * kH128SlabStride;          // both channel halves
constexpr int kH128BBytes = 128 * 128;                        // [128 co][64 ci] bf16
constexpr int kH128MaxBs = 16;

struct Halo128Params {
  int tiles_y, tiles_x, total, bstages;
  const float* bias;
  int relu, H, W;
  uint32_t* bits_out;         // nullable: ReLU bitmask of the output, [pixel][4] words
  const uint32_t* mask_bits;  // nullable: input-side ReLU mask (dgrad), [pixel][4] words
};

template <int CG>
__global__ void __launch_bounds__(kThreads, 1)
    halo128_kernel(const __grid_constant__ CUtensorMap map_x,
                   const __grid_constant__ CUtensorMap map_w,
                   const __grid_constant__ CUtensorMap map_out, const Halo128Params p) {
  constexpr bool PAIR = CG == 2;
  constexpr int kBCta = kH128BBytes / CG;  // weight bytes per CTA and stage
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  uint8_t* halo = smem;                                  // [2][2 slabs]
  uint8_t* bring = halo + 2 * kH128HaloStride;           // [bstages][kBCta]
  uint8_t* epi = bring + p.bstages * kBCta;              // [grp][2 slots][8 KB]
  __shared__ __align__(8) uint64_t hfull[2], hempty[2], bfull[kH128MaxBs], bempty[kH128MaxBs],
      tfull[2], tempty[2];
  __shared__ uint32_t tslot;
  const uint32_t warp = tc::warp_id();
  const int BS = p.bstages;
  const uint32_t rank = PAIR ? tc::cluster_rank() : 0;
  const int units = (p.total + CG - 1) / CG;
  const int u0 = PAIR ? (int)tc::cluster_id_x() : (int)blockIdx.x;
  const int ustep = PAIR ? (int)tc::num_clusters_x() : (int)gridDim.x;

  if (warp == 0 && tc::lane_id() == 0) {
    tc::tma_prefetch(&map_x);
    tc::tma_prefetch(&map_w);
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&hfull[s], 1);
      tc::mbar_init(&hempty[s], 1);
    }
    for (int s = 0; s < BS; ++s) {
      tc::mbar_init(&bfull[s], 1);
      tc::mbar_init(&bempty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], CG * (kEpiThreads / 32));  // one arrival per epilogue warp
    }
    tc::fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (PAIR) tc::tmem_alloc_cg2<256>(&tslot);
    else tc::tmem_alloc<256>(&tslot);
  }
  tc::tc_fence_before();
  if constexpr (PAIR) tc::cluster_sync();  // the peer's barriers are initialised
  else __syncthreads();
  tc::tc_fence_after();
  tc::pdl_wait();
  tc::pdl_launch_dependents();
  const uint32_t tmem = tslot;

  if (warp == 0) {
    if (tc::elect_one()) {
      int hs = 0, bs = 0;
      uint32_t hph = 0, bph = 0;
      TileCursor cur;
      cur.init(CG * u0 + (int)rank, CG * ustep, p.tiles_x, p.tiles_y);
      for (int u = u0; u < units; u += ustep, cur.next(p.tiles_x, p.tiles_y)) {
        const bool pad = CG * u + (int)rank >= p.total;
        tc::mbar_wait(&hempty[hs], hph ^ 1);
        if (rank == 0) tc::mbar_arrive_expect_tx(&hfull[hs], CG * 2 * kH128SlabBytes);
        uint8_t* h = halo + hs * kH128HaloStride;
        const int cx = pad ? -1 : cur.tx * kTW - 1, cy = pad ? -1 : cur.ty * kTH - 1,
                  cf = pad ? 0 : cur.f;
        for (int j = 0; j < 2; ++j) {
          if constexpr (PAIR)
            tc::tma_load_4d_cg2(h + j * kH128SlabStride, &map_x, tc::mapa(&hfull[hs], 0), 64 * j,
                                cx, cy, cf);
          else
            tc::tma_load_4d(h + j * kH128SlabStride, &map_x, &hfull[hs], 64 * j, cx, cy, cf);
        }
        if (++hs == 2) {
          hs = 0;
          hph ^= 1;
        }
        for (int t = 0; t < 9; ++t)
          for (int j = 0; j < 2; ++j) {
            tc::mbar_wait(&bempty[bs], bph ^ 1);
            if (rank == 0) tc::mbar_arrive_expect_tx(&bfull[bs], kH128BBytes);
            if constexpr (PAIR)
              tc::tma_load_2d_cg2(bring + bs * kBCta, &map_w, tc::mapa(&bfull[bs], 0),
                                  t * 128 + j * 64, 64 * (int)rank);
            else
              tc::tma_load_2d(bring + bs * kBCta, &map_w, &bfull[bs], t * 128 + j * 64, 0);
            if (++bs == BS) {
              bs = 0;
              bph ^= 1;
            }
          }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16(128 * CG, 128, false, false);
      const uint32_t h0 = tc::smem_u32(halo), b0 = tc::smem_u32(bring);
      auto commit = [&](uint64_t* bar) {
        if constexpr (PAIR) tc::mma_commit_cg2(bar, 0x3);  // both CTAs' barriers
        else tc::mma_commit(bar);
      };
      int hs = 0, bs = 0;
      uint32_t hph = 0, bph = 0;
      int it = 0;
      for (int u = u0; u < units; u += ustep, ++it) {
        const int acc = it & 1;
        tc::mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        tc::mbar_wait(&hfull[hs], hph);
        tc::tc_fence_after();
        const uint32_t hb = h0 + hs * kH128HaloStride;
        for (int t = 0; t < 9; ++t) {
          const int r = t / 3, s = t - 3 * (t / 3);
          for (int j = 0; j < 2; ++j) {
            tc::mbar_wait(&bfull[bs], bph);
            tc::tc_fence_after();
            if (tc::elect_one()) {
              const uint32_t ab = hb + j * kH128SlabStride + (r * kH128HP + s) * 128;
              const uint32_t bb = b0 + bs * kBCta;
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                const uint64_t ad = tc::smem_desc(ab + kk * 32, 16, kH128HP * 128, tc::kSw128);
                const uint64_t bd = tc::smem_desc(bb + kk * 32, 16, 8 * 128, tc::kSw128);
                if constexpr (PAIR)
                  tc::mma_bf16_cg2(tmem + acc * 128, ad, bd, idesc, (t | j | kk) ? 1u : 0u);
                else
                  tc::mma_bf16(tmem + acc * 128, ad, bd, idesc, (t | j | kk) ? 1u : 0u);
              }
              commit(&bempty[bs]);
              if (t == 8 && j == 1) {
                commit(&hempty[hs]);
                commit(&tfull[acc]);
              }
            }
            __syncwarp();
            if (++bs == BS) {
              bs = 0;
              bph ^= 1;
            }
          }
        }
        if (++hs == 2) {
          hs = 0;
          hph ^= 1;
        }
      }
    }
  } else {
    // epilogue: group g owns output channels [64 g, 64 g + 64) = sub-tiles
    // 2g, 2g + 1 of 32 channels; warp w reads TMEM lanes (w % 4) * 32 .. +32
    // = tile pixel (lrow / 8, lrow % 8)
    const int grp = (int)(warp - 2) >> 2;
    const int q = warp & 3;
    const int lrow = q * 32 + tc::lane_id();
    const bool leader = ((warp - 2) & 3) == 0 && tc::lane_id() == 0;
    uint8_t* ob0 = epi + grp * 2 * kSub;
    const int ti = lrow >> 3, tj = lrow & 7;
    const bool need_pix = p.bits_out != nullptr || p.mask_bits != nullptr;
    __shared__ float bias_s[128];
    if (lrow < 64) bias_s[grp * 64 + lrow] = p.bias ? __ldg(p.bias + grp * 64 + lrow) : 0.f;
    tc::named_bar(1 + grp, 128);
    int it = 0;
    TileCursor cur;
    cur.init(CG * u0 + (int)rank, CG * ustep, p.tiles_x, p.tiles_y);
    for (int u = u0; u < units; u += ustep, ++it, cur.next(p.tiles_x, p.tiles_y)) {
      const bool pad = CG * u + (int)rank >= p.total;  // uniform over the CTA
      const int ph = cur.ty * kTH + ti, pw = cur.tx * kTW + tj;
      const long long pix = (need_pix && !pad && ph < p.H && pw < p.W)
                                ? ((long long)cur.f * p.H + ph) * p.W + pw : -1;
      uint32_t mbits[2] = {0u, 0u};
      if (p.mask_bits && pix >= 0) {
        mbits[0] = __ldg(p.mask_bits + pix * 4 + 2 * grp);
        mbits[1] = __ldg(p.mask_bits + pix * 4 + 2 * grp + 1);
      }
      const int acc = it & 1;
      tc::mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc::tc_fence_after();
      uint32_t raw[2][32];
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + acc * 128 + (2 * grp + v) * 32;
        tc::tmem_ld_32x32b_x16(ta, *reinterpret_cast<uint32_t(*)[16]>(&raw[v][0]));
        tc::tmem_ld_32x32b_x16(ta + 16, *reinterpret_cast<uint32_t(*)[16]>(&raw[v][16]));
      }
      tc::tmem_ld_wait();
      tc::tc_fence_before();
      __syncwarp();
      if (tc::lane_id() == 0) {
        if constexpr (PAIR) tc::mbar_arrive_cluster(tc::mapa(&tempty[acc], 0));
        else tc::mbar_arrive(&tempty[acc]);
      }
      if (pad) continue;
#pragma unroll
      for (int v = 0; v < 2; ++v) {
        const int sub = 2 * grp + v;
        float y[32];
#pragma unroll
        for (int i = 0; i < 32; ++i)
          y[i] = __uint_as_float(raw[v][i]) + bias_s[sub * 32 + i];
        if (p.relu) {
#pragma unroll
          for (int i = 0; i < 32; ++i) y[i] = fmaxf(y[i], 0.f);
        }
        uint32_t o[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) o[j] = tc::pack_bf16(y[2 * j], y[2 * j + 1]);
        if (p.mask_bits) {
#pragma unroll
          for (int j = 0; j < 16; ++j) o[j] &= tc::bits_keep(mbits[v], j);
        }
        if (p.bits_out && pix >= 0) p.bits_out[pix * 4 + sub] = tc::relu_bits16(o);
        uint8_t* ob = ob0 + v * kSub;
        // the store two sub-tiles back (same slot) must have finished reading it
        if (leader) tc::bulk_wait_read<1>();
        tc::named_bar(1 + grp, 128);
#pragma unroll
        for (int c = 0; c < 4; ++c)
          *reinterpret_cast<uint4*>(ob + sw64(lrow, c)) =
              make_uint4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
        tc::fence_proxy_async();
        tc::named_bar(1 + grp, 128);
        if (leader) {
          tc::tma_store_4d(&map_out, ob, sub * 32, cur.tx * kTW, cur.ty * kTH, cur.f);
          tc::bulk_commit();
        }
      }
    }
    if (leader) tc::bulk_wait<0>();
  }
  tc::tc_fence_before();
  if constexpr (PAIR) {
    tc::cluster_sync();  // both CTAs are done with the pair's TMEM and shared memory
    tc::tc_fence_after();
    if (warp == 1) tc::tmem_dealloc_cg2<256>(tmem);
  } else {
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc<256>(tmem);
  }
}

}  // namespace halo
}  // namespace tsm

namespace tsm {
namespace halo {

// ---------------------------------------------------------------------------
// Weight (+ bias) gradient of the same 3x3 / 128-channel conv (res3 conv2):
// dW[co][r][s][ci] = sum_p x(p + (r - 1, s - 1))[ci] dY(p)[co].  The CTAs
// form three groups, group r owning kernel row r: per 8 x 8 output patch it
// loads the 10 x 8 window of x rows r - 1 .. r + 6 (two 64-channel slabs =
// the two M atoms of a 128-row operand) and the dY patch (two 64-channel
// slabs = the two N atoms of N = 128), and the three taps s are descriptor
// offsets into the window: D_s[ci][co] += x_s^T dY over 4 K steps of 16
// pixels.  Group 0 adds an all-ones M tile whose rows give the bias
// gradient.  N = 128 instead of the 64-channel kernel's 64 halves the
// shared-memory operand bytes per MMA.  CTA i of a group takes patches
// i, i + G, ... (the three groups sweep the same patches together, so the
// x / dY tiles are read from HBM once); fp32 partials per CTA, reduced in a
// fixed order by wgrad_halo128_reduce_kernel (deterministic).
constexpr int kW128P = kPW + 2;                        // window pitch (10 pixels)
constexpr int kW128Slab = kW128P * kPW * kRowB;        // 10 x 8 pixels x 64 ch = 10240
constexpr int kW128Stage = 2 * kW128Slab + 2 * kDyBytes;  // 36864
constexpr int kW128Rows = 3 * 128 + 1;                 // per-CTA partial rows (+ db)

struct Wgrad128Params {
  int patches_y, patches_x, total, stages, gctas;
  float* ws;  // [grid][kW128Rows][128]
};

__global__ void __launch_bounds__(kThreads, 1)
    wgrad_halo128_kernel(const __grid_constant__ CUtensorMap map_x,
                         const __grid_constant__ CUtensorMap map_dy, const Wgrad128Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  const int S = p.stages;
  uint8_t* ones = smem + S * kW128Stage;  // [2 atoms][64 px][64] all-ones bf16
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages], tfull;
  __shared__ uint32_t tslot;
  const uint32_t warp = tc::warp_id();
  const int grp_r = (int)blockIdx.x / p.gctas;          // kernel row of this CTA group
  const int b0 = (int)blockIdx.x - grp_r * p.gctas, bstep = p.gctas;

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
  if (warp >= 2) {
    const uint4 one = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
    for (int i = threadIdx.x - 64; i < 2 * kDyBytes / 16; i += kEpiThreads)
      reinterpret_cast<uint4*>(ones)[i] = one;
    tc::fence_proxy_async();
  }
  if (warp == 1) tc::tmem_alloc<512>(&tslot);
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
        tc::mbar_wait(&empty[stage], phase ^ 1);
        uint8_t* st = smem + stage * kW128Stage;
        tc::mbar_arrive_expect_tx(&full[stage], kW128Stage);
        const int x0 = px * kPW, y0 = py * kPW;
        for (int j = 0; j < 2; ++j) {
          tc::tma_load_4d(st + j * kW128Slab, &map_x, &full[stage], 64 * j, x0 - 1,
                          y0 - 1 + grp_r, f);
          tc::tma_load_4d(st + 2 * kW128Slab + j * kDyBytes, &map_dy, &full[stage], 64 * j, x0,
                          y0, f);
        }
        if (++stage == S) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = tc::idesc_bf16(128, 128, true, true);
    const uint32_t s0 = tc::smem_u32(smem), o0 = tc::smem_u32(ones);
    int stage = 0;
    uint32_t phase = 0;
    for (int b = b0; b < p.total; b += bstep) {
      tc::mbar_wait(&full[stage], phase);
      tc::tc_fence_after();
      if (tc::elect_one()) {
        const uint32_t xs = s0 + stage * kW128Stage, ds = xs + 2 * kW128Slab;
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // 16 pixels (two patch rows) per K step
          const uint32_t acc = (b > b0 || j > 0) ? 1u : 0u;
          const uint64_t bd = tc::smem_desc(ds + j * 16 * kRowB, kDyBytes, 8 * kRowB, tc::kSw128);
#pragma unroll
          for (int s = 0; s < 3; ++s) {
            const uint64_t ad = tc::smem_desc(xs + (2 * j * kW128P + s) * kRowB, kW128Slab,
                                              kW128P * kRowB, tc::kSw128);
            tc::mma_bf16(tmem + s * 128, ad, bd, idesc, acc);
          }
          if (grp_r == 0) {
            const uint64_t od =
                tc::smem_desc(o0 + j * 16 * kRowB, kDyBytes, 8 * kRowB, tc::kSw128);
            tc::mma_bf16(tmem + 3 * 128, od, bd, idesc, acc);
          }
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
    // D_s rows = ci (TMEM lanes), columns = co: ws[cta][s * 128 + ci][co];
    // the ones tile's row 0 -> ws[cta][384][co]; group g takes columns
    // [64 g, 64 g + 64)
    const int grp = (int)(warp - 2) >> 2;
    const int q = warp & 3;
    const int lrow = q * 32 + tc::lane_id();
    const bool has_k = b0 < p.total;
    if (has_k) {
      tc::mbar_wait(&tfull, 0);
      tc::tc_fence_after();
    }
    float* wsb = p.ws + (long long)blockIdx.x * kW128Rows * 128;
    const int ntiles = grp_r == 0 ? 4 : 3;
#pragma unroll 1
    for (int s = 0; s < ntiles; ++s) {
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        const int c0 = grp * 64 + h * 32;
        uint32_t raw0[16], raw1[16];
        const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + s * 128 + c0;
        tc::tmem_ld_32x32b_x16(ta, raw0);
        tc::tmem_ld_32x32b_x16(ta + 16, raw1);
        tc::tmem_ld_wait();
        if (s == 3 && lrow != 0) continue;
        float* dst = wsb + (long long)(s * 128 + (s == 3 ? 0 : lrow)) * 128 + c0;
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

// dw[co][r][s][ci] = sum over the CTAs of group r (in order) of
// ws[cta][s * 128 + ci][co]; db[co] = sum over group 0 of ws[cta][384][co].
__global__ void __launch_bounds__(256)
    wgrad_halo128_reduce_kernel(const float* __restrict__ ws, float* __restrict__ dw,
                                float* __restrict__ db, int gctas) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;  // (tap, ci, co), co fastest
  if (i >= 9 * 128 * 128 + 128) return;
  int r, row, co;
  float* out;
  if (i < 9 * 128 * 128) {
    co = i & 127;
    const int ci = (i >> 7) & 127, tap = i >> 14;
    r = tap / 3;
    row = (tap - 3 * r) * 128 + ci;
    out = dw + ((long long)co * 9 + tap) * 128 + ci;
  } else {
    if (!db) return;
    co = i - 9 * 128 * 128;
    r = 0;
    row = 3 * 128;
    out = db + co;
  }
  const float* src = ws + ((long long)r * gctas * kW128Rows + row) * 128 + co;
  float a[4] = {0.f, 0.f, 0.f, 0.f};
  int c = 0;
  for (; c + 4 <= gctas; c += 4) {
#pragma unroll
    for (int j = 0; j < 4; ++j) a[j] += __ldg(src + (long long)(c + j) * kW128Rows * 128);
  }
  for (int j = 0; c < gctas; ++c, ++j) a[j] += __ldg(src + (long long)c * kW128Rows * 128);
  *out = (a[0] + a[1]) + (a[2] + a[3]);
}

}  // namespace halo
}  // namespace tsm
