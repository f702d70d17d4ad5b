// Persistent, warp-specialized tcgen05 GEMM for the TSM bottleneck convs.
//
//   D[M, N] = sum_k A[M, K] * B[N, K]      bf16 x bf16 -> fp32 in TMEM
//
// Activations live channels-last per frame ("NTHWC": rows = pixels of
// N*T frames, channels contiguous).  Every conv of the block is one of:
//   * 1x1 forward   M = pixels, N = C_out, K = C_in    A = act (K-major)
//   * 3x3 forward   M = pixels, N = C_out, K = 9*C_in  A = im2col(act)
//   * dgrad         same shapes with dY as A and W^T / flipped W as B
//   * wgrad         M = C_out,  N = C_in(*9), K = pixels (both MN-major)
//
// Operands are staged by TMA in "slabs": one TMA box of [rows][KC] bf16
// (KC = 8/16/32/64 channels -> no / 32B / 64B / 128B swizzle).  A K-major
// stage (BK = 64) is 64/KC slabs side by side along K; an MN-major stage is
// MN/KC slabs along M (or N) with 64 K-rows each.  Each slab is its own TMA
// box with its own coordinates — this is what lets the temporal shift ride in
// the loads: a slab whose channels lie in the shifted group [0,F) is fetched
// from row r - H*W (frame t-1) and [F,F+B) from r + H*W (frame t+1) of a 3-D
// tensor map (C, T*H*W, clips); rows outside the clip are out of bounds and
// TMA zero-fills them, which is exactly the reference's +0.0 boundary
// (kernels.cpp:108-115).  The shifted activation is never materialised.
//
// Warp roles (6 warps): w0 TMA producer, w1 TMEM allocator + MMA issuer
// (one elected thread), w2..w5 epilogue.  Tiles are distributed round-robin
// over a persistent grid; the smem ring (runtime depth) runs across tile
// boundaries and the TMEM accumulator is double-buffered, so the epilogue of
// tile i overlaps the main loop of tile i+1.
//
// bf16 epilogue (TMA path): per 32-column sub-tile the epilogue warps load
// the accumulator from TMEM, add bias / ReLU, add the residual and apply the
// ReLU-backward mask — both prefetched by TMA into a 2-slot smem ring — then
// stage bf16 into swizzled smem and write it with a TMA store.  The adjoint
// temporal shift of the dgrad of the shifted conv is a per-group row offset
// (-H*W / +H*W) on the 3-D store map: rows leaving the clip are clipped by
// TMA, and the vacated boundary frame is filled by shift_out_boundary().
#pragma once

#include <type_traits>

#include "tc_common.cuh"

namespace tsm {
namespace gemm {

constexpr int BM = 128;
constexpr int BK = 64;
// w0 TMA, w1 MMA, w2.. epilogue (kGroups groups of 4 warps, one per TMEM
// lane quarter each), then 2 bias-gradient warps.  The memory-bound GEMMs
// are bound by the epilogue's per-sub-tile latency chain, so more groups =
// more sub-tiles in flight per SM.
#ifndef TSM_EPI_GROUPS
#define TSM_EPI_GROUPS 3
#endif
constexpr int kGroups = TSM_EPI_GROUPS;
constexpr int kEpiThreads = 128 * kGroups;
constexpr int kBiasWarp0 = 2 + 4 * kGroups;
constexpr int kThreads = 64 + kEpiThreads + 64;
constexpr int kBarBias = kGroups + 1;   // named barrier: all epilogue threads (bias staging)
constexpr int kBarDb = kGroups + 2;     // named barrier: the two bias-gradient warps
constexpr int kMaxStages = 8;
constexpr int EC = 32;                  // epilogue sub-tile columns (64 B rows, SW64)
constexpr int kSubBytes = BM * EC * 2;  // 8 KiB
constexpr int kIdentBytes = 64 * 64 * 2;  // identity operand of the fused residual
constexpr int kSmemLimit = 227 * 1024;

enum LoadMode : int {
  LOAD_ACT3D = 0,   // 3-D map (C, rows_per_clip, clips), optional group row offsets
  LOAD_W2D = 1,     // 2-D map (K, rows): plain matrix, row-major [rows][K]
  LOAD_IM2COL = 2,  // 4-D im2col map (C, W, H, frames)
};

enum MapMode : int {
  MAP_CLIP = 0,    // M tiles enumerate (clip, 128-row block) of an ACT3D operand
  MAP_LINEAR = 1,  // M tiles enumerate 128-row blocks of [0, M_total)
};

enum EpiMode : int {
  EPI_BF16 = 0,  // out bf16 [rows][ldo] (+bias, relu, residual, mask, adjoint-shift rows)
  EPI_F32 = 1,   // out fp32 [split][M][N] partial tile (wgrad), optional transpose
};

struct OpLoad {
  int mode;
  // ACT3D: channel-group row offsets (temporal shift): channels [0,g0) read
  // row + off0, [g0,g1) read row + off1, the rest read row.
  int g0, g1, off0, off1;
  // ACT3D: rows per clip; IM2COL: output geometry for pixel -> coordinates.
  int rows_per_clip;
  int w_out, h_out, stride, pad;  // IM2COL: wo/ho extents, conv stride, padding
  int c_in;                       // IM2COL / W2D tap_map: channels per tap (K decomposition)
  int taps_w;                     // IM2COL: filter width (tap -> (r, s))
  // W2D: K index (tap * c_in + c) reads column (tap_map[tap] * c_in + c),
  // 4-bit entries (the sub-pixel dgrad classes pick 1-4 of the 9 taps).
  unsigned long long tap_map;
  // IM2COL: vtaps > 0 lists the taps explicitly, 2 bits each (r | s << 1,
  // offsets 0 / 1): the merged sub-pixel dgrad's 9 virtual taps.
  int vtaps, vtap_rs;
  // ACT3D, virtual channels (shift splits narrower than a slab, F + B <= vg):
  // virtual channel v < vg reads real channel v at row + off0, vg <= v < 2 vg
  // reads channel v - vg at row + off1, v >= 2 vg reads v - 2 vg at the row
  // itself.  The GEMM's other operand zeroes the columns that must not count
  // (expanded weights) or the caller picks the rows that do (weight gradient).
  int vg;
};

struct Params {
  // problem
  int m_tiles, n_tiles, k_blocks, splits;  // splits > 1: K range split (EPI_F32)
  int stages;                              // smem ring depth (runtime)
  // Residual in the MMA: res_kb extra k-blocks per tile multiply 64-channel
  // slabs of the residual (map_res, loaded like A through `r`) by a 64x64
  // identity into TMEM columns [64 j, 64 j + 64) — the residual is then
  // already in the accumulator and the epilogue has no residual stream.
  int res_kb;
  OpLoad r;
  int out_slots;                           // TMA epilogue staging buffers per group (1, 2)
  int map_mode;
  int tiles_per_clip, rows_per_clip;  // MAP_CLIP
  // MAP_CLIP clip remainders: tiles m >= rem_tiles0 (rem_rows > 0 enables) gather the
  // last rem_rows rows of rem_clips clips each (A through map_res, output
  // through map_mask, both boxed {KC, rem_rows, rem_clips}); n_clips clips.
  int rem_tiles0, rem_rows, rem_clips, n_clips;
  // K-side clip remainders (MN-major ACT3D operands): k-blocks kb >= krem0
  // (krem_rows > 0 enables) gather the last krem_rows rows of krem_clips
  // clips each, A through map_res and B through map_mask.
  int krem0, krem_rows, krem_clips;
  int m_total;                        // MAP_LINEAR
  int kb_per_clip;                    // MN-major ACT3D K decomposition
  // Interleaved split-K (k_ilv > 0): split s takes the k_ilv-block chunks
  // s, s + splits, s + 2 splits, ...; the splits then sweep one window of
  // K together, so rows one split reads at a frame offset (shifted
  // operands) are still in L2 when another split reads them unshifted.
  int k_ilv;
  OpLoad a, b;
  // epilogue
  int epi;
  int n_total;  // valid N columns
  const float* bias;
  const __nv_bfloat16* residual;  // same layout as out
  const __nv_bfloat16* mask;      // relu-backward mask (same layout as out): out *= mask > 0
  __nv_bfloat16* out;
  int ldo;
  int relu;
  int tma_out;  // bf16 epilogue through TMA (maps out/res/mask) instead of direct stores
  // ReLU bitmasks, [rows][ldo / 32] words, bit j of word w = column 32 w + j:
  // bits_out (forward) records out > 0; mask_bits (backward) replaces the
  // bf16 `mask` (out *= bit).  16x less traffic than a bf16 mask.
  uint32_t* bits_out;
  const uint32_t* mask_bits;
  int bits_ld;
  // adjoint temporal shift on the output rows (dgrad of the shifted conv):
  // columns [0,sg0) of row (t) land in row (t-1), [sg0,sg1) in row (t+1);
  // the vacated boundary rows receive +0.0 (kernels.cpp:127-157).
  int shift_out, sg0, sg1, hw, frames;
  // strided scatter of output rows (dgrad of a strided 1x1 projection): row
  // (f, ho, wo) of the Ho x Wo grid lands at (f, ho*ss + oh, wo*ss + ow) of
  // a Hi x Wi grid (rows no launch writes are pre-zeroed by the caller).
  int scatter, sc_wo, sc_ho, sc_stride, sc_wi, sc_hi, sc_oh, sc_ow;
  // Row-aligned M tiles for the sub-pixel scatter (m_rows > 0): tile m
  // covers class rows [m * m_rows, + m_rows) = sc_rows whole rows of sc_wo
  // pixels (the MMA's last BM - m_rows rows are computed and dropped), so a
  // staged sub-tile is one box of the 5-D class map map_out (C, 2, Wo, 2,
  // frames * Ho) at (col, ow, 0, oh, m * sc_rows) — one TMA store instead of
  // per-thread scattered rows.
  int m_rows, sc_rows, sc_tma;
  // Merged sub-pixel classes (cls_n > 0): the tile walk's N axis carries
  // cls_n classes (rotated by the M tile so a CTA's tiles cycle through
  // them); class c takes k-blocks [cls_kb[c], cls_kb[c+1]) and scatters to
  // (2 ho + cls_oh[c], 2 wo + cls_ow[c]).
  int cls_n, cls_kb[5], cls_oh[4], cls_ow[4];
  // scatter only: out[row] = bf16(out[row] + value) (read-modify-write of
  // rows another launch wrote; no pre-zeroing)
  int acc_out;
  float* out_f32;
  int transpose_f32;  // write out_f32[N][M] instead of [M][N]
  // Fused bias gradient (wgrad only): the epilogue warps also consume every
  // smem stage and sum the dY slab per output channel over the tile's pixel
  // rows -> db_part[split][c_out] (reduced over splits in a fixed order).
  // db_mode 1: dY is the A operand (co = m*BM + i, summed by n == 0 tiles);
  // db_mode 2: dY is the B operand (co = i < BN, summed by m == 0 tiles).
  int db_mode;
  float* db_part;
  int db_c;  // c_out
};

// ---------------------------------------------------------------------------
// Stage geometry (compile-time)

// CG = 2: a CTA pair (cta_group::2) computes a 256 x BN tile; each CTA
// stages its own 128 rows of A and BN / 2 rows of B.
// BKT: K per stage.  64 everywhere except the MN-major weight gradients of
// CTA pairs, which stage 128 pixel rows per box: TMA throughput per byte
// grows with the box (tools/tma_rate_probe.cu: L2-resident 64-row boxes
// ~170-250 cycles each, 128-row boxes ~250).
template <int BN, int KCA, int KCB, bool AMN, bool BMN, int CG = 1, int BKT = BK>
struct Cfg {
  static constexpr int BNL = BN / CG;  // B rows (N) staged by one CTA
  static constexpr int A_SLABS = AMN ? BM / KCA : BKT / KCA;
  static constexpr int A_ROWS = AMN ? BKT : BM;
  static constexpr int A_SLAB_BYTES = A_ROWS * KCA * 2;
  static constexpr int B_SLABS = BMN ? BNL / KCB : BKT / KCB;
  static constexpr int B_ROWS = BMN ? BKT : BNL;
  static constexpr int B_SLAB_BYTES = B_ROWS * KCB * 2;
  static constexpr int A_BYTES = A_SLABS * A_SLAB_BYTES;  // = BM*BK*2
  static constexpr int B_BYTES = B_SLABS * B_SLAB_BYTES;  // = BNL*BK*2
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int RES_PER_STAGE = STAGE_BYTES / A_BYTES;  // residual tiles per stage
  static constexpr int TMEM_COLS = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128
                                   : 2 * BN <= 256 ? 256 : 512;
  static constexpr int BAR_BYTES = 512;  // mbarriers (full, empty, tfull, tempty, resbar, consumed) + TMEM slot
  static_assert(A_BYTES == BM * BKT * 2 && B_BYTES == BNL * BKT * 2, "slab tiling");
  static_assert(BKT == BK || (AMN && BMN), "K per stage other than 64: MN-major operands only");
  static_assert(CG == 1 || CG == 2, "CTA pairs or single CTAs");
  static_assert(BN % EC == 0, "epilogue sub-tiles");
  // epilogue smem, per epilogue group: 2 staging buffers + 2 residual + 2
  // mask slots (as needed)
  static int epi_bytes(bool res, bool mask, bool tma_out, int out_slots = 2) {
    return tma_out ? kGroups * kSubBytes * (out_slots + (res ? 2 : 0) + (mask ? 2 : 0)) : 0;
  }
  static int stages_for_limit(int limit, int epi, int extra) {
    int s = (limit - 1024 - BAR_BYTES - epi - extra) / STAGE_BYTES;
    return s > kMaxStages ? kMaxStages : s;
  }
  static int stages_for(int epi) {
    int s = (kSmemLimit - 2048 - BAR_BYTES - epi) / STAGE_BYTES;  // 1 KiB static smem
    return s > kMaxStages ? kMaxStages : s;
  }
  static int smem_bytes(int stages, int epi, int extra = 0) {
    return stages * STAGE_BYTES + epi + extra + 1024 + BAR_BYTES;
  }
};

// UMMA smem descriptor for k-step j (16 K-elements) of one operand stage.
template <int KC, bool MN, int ROWS, int SLAB_BYTES>
__device__ __forceinline__ uint64_t operand_desc(uint32_t base, int j) {
  constexpr uint32_t layout = tc::swizzle_for_row_bytes(KC * 2);
  if constexpr (!MN) {
    // K-major: slabs tile K.  Rows of KC*2 bytes; 8-row groups at SBO.
    if constexpr (KC == 8) {
      // no swizzle: core matrices 8 rows x 16 B; the two K halves of one
      // UMMA_K=16 step are adjacent slabs (LBO = slab stride).
      return tc::smem_desc(base + (2 * j) * SLAB_BYTES, SLAB_BYTES, 128, layout);
    } else {
      const int k_el = j * 16;
      const uint32_t addr = base + (k_el / KC) * SLAB_BYTES + (k_el % KC) * 2;
      return tc::smem_desc(addr, 16, 8 * KC * 2, layout);
    }
  } else {
    // MN-major: slabs tile M/N (KC channels each, LBO apart), 64 K-rows.
    // k-step j covers K-rows [16j, 16j+16).
    if constexpr (KC == 8) {
      // interleave: SBO = MN-block (slab) stride, LBO = 8-row K-group stride.
      return tc::smem_desc(base + j * 16 * 16, 128, SLAB_BYTES, layout);
    } else {
      return tc::smem_desc(base + j * 16 * KC * 2, SLAB_BYTES, 8 * KC * 2, layout);
    }
  }
}

// Producer: issue one slab.  `chan` indexes the operand's channel axis and
// (clip,row) / pixel its row axis.
// TMA loads of one operand stage: CG = 2 completes on the pair leader's
// barrier (cta_group::2 form), CG = 1 on this CTA's.
template <int CG>
__device__ __forceinline__ void ld2(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                    int c1) {
  if constexpr (CG == 2) tc::tma_load_2d_cg2(dst, map, tc::mapa(bar, 0), c0, c1);
  else tc::tma_load_2d(dst, map, bar, c0, c1);
}
template <int CG>
__device__ __forceinline__ void ld3(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                    int c1, int c2) {
  if constexpr (CG == 2) tc::tma_load_3d_cg2(dst, map, tc::mapa(bar, 0), c0, c1, c2);
  else tc::tma_load_3d(dst, map, bar, c0, c1, c2);
}
template <int CG>
__device__ __forceinline__ void ldi(void* dst, const CUtensorMap* map, uint64_t* bar, int c,
                                    int w, int h, int n, uint16_t ow, uint16_t oh) {
  if constexpr (CG == 2) tc::tma_load_im2col_4d_cg2(dst, map, tc::mapa(bar, 0), c, w, h, n, ow, oh);
  else tc::tma_load_im2col_4d(dst, map, bar, c, w, h, n, ow, oh);
}

template <int CG = 1>
__device__ __forceinline__ void load_slab(const OpLoad& L, const CUtensorMap* map, void* dst,
                                          uint64_t* bar, int chan, int clip, int row) {
  if (L.mode == LOAD_ACT3D) {
    if (L.vg) {
      const int grp = chan < L.vg ? 0 : (chan < 2 * L.vg ? 1 : 2);
      ld3<CG>(dst, map, bar, chan - grp * L.vg, row + (grp == 0 ? L.off0 : grp == 1 ? L.off1 : 0),
              clip);
      return;
    }
    const int off = chan < L.g0 ? L.off0 : (chan < L.g1 ? L.off1 : 0);
    ld3<CG>(dst, map, bar, chan, row + off, clip);
  } else if (L.mode == LOAD_W2D) {
    if (L.tap_map) {
      const int tap = chan / L.c_in, c = chan - tap * L.c_in;
      chan = (int)((L.tap_map >> (4 * tap)) & 15) * L.c_in + c;
    }
    ld2<CG>(dst, map, bar, chan, row);
  } else {
    // IM2COL: (clip, row) -> flattened output pixel (frame, ho, wo); `chan`
    // = K index (tap * c_in + c).
    const int tap = chan / L.c_in, c = chan - tap * L.c_in;
    const int r = tap / L.taps_w, s = tap - r * L.taps_w;
    const int hw = L.w_out * L.h_out;
    const int pix = clip * L.rows_per_clip + row;
    const int f = pix / hw, rem = pix - f * hw;
    const int ho = rem / L.w_out, wo = rem - ho * L.w_out;
    ldi<CG>(dst, map, bar, c, wo * L.stride - L.pad, ho * L.stride - L.pad, f, (uint16_t)s,
            (uint16_t)r);
  }
}

// Window origin of flattened output pixel `pix` (frame, ho, wo) for an
// im2col operand: one set of divisions per tile / k-block, not per slab.
struct PixOrigin {
  int w, h, f;
};
__device__ __forceinline__ PixOrigin pix_origin(const OpLoad& L, int pix) {
  const int hw = L.w_out * L.h_out;
  const int f = pix / hw, rem = pix - f * hw;
  const int ho = rem / L.w_out, wo = rem - ho * L.w_out;
  return {wo * L.stride - L.pad, ho * L.stride - L.pad, f};
}

// Walks the K index (tap * c_in + c) of an im2col operand without divisions.
struct TapCursor {
  int c, r, s, t;
  __device__ __forceinline__ void set_rs(const OpLoad& L) {
    const int e = (L.vtap_rs >> (2 * t)) & 3;
    r = e & 1;
    s = e >> 1;
  }
  __device__ __forceinline__ void init(const OpLoad& L, int chan) {
    t = chan / L.c_in;
    c = chan - t * L.c_in;
    if (L.vtaps) {
      set_rs(L);
    } else {
      r = t / L.taps_w;
      s = t - r * L.taps_w;
    }
  }
  __device__ __forceinline__ void advance(const OpLoad& L, int delta) {
    c += delta;
    while (c >= L.c_in) {
      c -= L.c_in;
      ++t;
      if (L.vtaps) {
        set_rs(L);
      } else if (++s == L.taps_w) {
        s = 0;
        ++r;
      }
    }
  }
};

// 16-byte chunk c of row r inside a [128][64 B] SW64-swizzled sub-tile.
__device__ __forceinline__ uint32_t sw64_off(int r, int c) {
  return (uint32_t)(r * 64 + ((c ^ ((r >> 1) & 3)) << 4));
}

// (n, m unit, split) of the tiles tile0, tile0 + step, ... with n fastest:
// the carries replace three integer divisions per tile and role.
struct TileWalk {
  int n, mu, sp, dn, dmu, dsp, nt, mus;
  __device__ __forceinline__ TileWalk(int tile, int step, int n_tiles, int m_units)
      : nt(n_tiles), mus(m_units) {
    n = tile % nt;
    mu = (tile / nt) % mus;
    sp = tile / nt / mus;
    dn = step % nt;
    dmu = (step / nt) % mus;
    dsp = step / nt / mus;
  }
  __device__ __forceinline__ void next() {
    n += dn;
    const int cn = n >= nt;
    n -= cn * nt;
    mu += dmu + cn;
    const int cm = mu >= mus;
    mu -= cm * mus;
    sp += dsp + cm;
  }
};

template <int BN, int KCA, int KCB, bool AMN, bool BMN, int CG = 1, int BKT = BK>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                   const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_out,
                   const __grid_constant__ CUtensorMap map_res,
                   const __grid_constant__ CUtensorMap map_mask, const Params p) {
  using C = Cfg<BN, KCA, KCB, AMN, BMN, CG, BKT>;
  constexpr bool PAIR = CG == 2;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1 KiB alignment by pointer arithmetic on the __shared__ array (not an
  // integer round trip), so every derived pointer stays a known shared-space
  // pointer and compiles to LDS/STS instead of generic LD/ST
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  const int STAGES = p.stages;
  const bool tma_epi = p.epi == EPI_BF16 && p.tma_out;
  const bool has_res = tma_epi && p.residual != nullptr;
  const bool has_mask = tma_epi && p.mask != nullptr;
  // identity B operand of the residual k-blocks: 64 x 64 bf16, K-major SW128
  uint8_t* ident = smem + STAGES * C::STAGE_BYTES;
  uint8_t* epi = ident + (p.res_kb ? kIdentBytes : 0);
  uint8_t* out_buf = epi;                                            // [group][2][8 KiB]
  uint8_t* res_buf = out_buf + p.out_slots * kGroups * kSubBytes;         // [group][2][8 KiB]
  uint8_t* mask_buf = res_buf + (has_res ? 2 * kGroups * kSubBytes : 0);  // [group][2][8 KiB]
  uint8_t* epi_end =
      epi + (tma_epi ? kGroups * kSubBytes * (p.out_slots + (has_res ? 2 : 0) + (has_mask ? 2 : 0)) : 0);
  float* bias_s = reinterpret_cast<float*>(epi_end);  // TMA epilogue: [n_tiles * BN]
  uint8_t* bar_base = epi_end + ((tma_epi && p.bias) ? p.n_tiles * BN * 4 : 0);
  uint64_t* full = reinterpret_cast<uint64_t*>(bar_base);
  uint64_t* empty = full + kMaxStages;
  uint64_t* tfull = empty + kMaxStages;  // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint64_t* resbar = tempty + 2;         // [group][2]
  // pairs with a fused bias gradient: the MMA's commit of a stage (both
  // CTAs), after which the bias warps read it and release it on `empty`
  uint64_t* consumed = resbar + 2 * kGroups;  // [kMaxStages]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(consumed + kMaxStages);

  const uint32_t warp = tc::warp_id();
  // CTA pairs enumerate (m pair, n, split) tiles over the clusters; the CTA
  // of rank r takes 128-row tile m = 2 * pair + r (m == m_tiles: a padding
  // tile that loads a valid tile and stores nothing)
  const uint32_t rank = PAIR ? tc::cluster_rank() : 0;
  const int m_units = PAIR ? (p.m_tiles + 1) / 2 : p.m_tiles;
  const int nt_walk = p.n_tiles * (p.cls_n ? p.cls_n : 1);
  const int total_tiles = m_units * nt_walk * p.splits;
  const int tile0 = PAIR ? (int)tc::cluster_id_x() : (int)blockIdx.x;
  const int tstep = PAIR ? (int)tc::num_clusters_x() : (int)gridDim.x;
  const int kb_per_split = (p.k_blocks + p.splits - 1) / p.splits;

  if (warp == 0 && tc::lane_id() == 0) {
    tc::tma_prefetch(&map_a);
    tc::tma_prefetch(&map_b);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      // + the bias-grad reader; pairs: the reader alone (it follows `consumed`)
      tc::mbar_init(&empty[s], p.db_mode ? (PAIR ? 1 : 2) : 1);
      tc::mbar_init(&consumed[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      // pairs: one arrival per epilogue warp of both CTAs (on the leader's)
      tc::mbar_init(&tempty[a], PAIR ? 2 * (kEpiThreads / 32) : kEpiThreads);
    }
    for (int a = 0; a < 2 * kGroups; ++a) tc::mbar_init(&resbar[a], 1);
    tc::fence_barrier_init();
  }
  if (p.res_kb && warp >= 2) {
    // B[n][k] = (n == k): row n = 128 B, 16-byte chunk c at c ^ (n & 7)
    for (int i = threadIdx.x - 64; i < kIdentBytes / 16; i += kThreads - 64) {
      const int n = i >> 3, c = (i & 7) ^ (n & 7);  // chunk i&7 holds k = 8c..8c+7
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
  if (warp == 1) {
    if constexpr (PAIR) tc::tmem_alloc_cg2<C::TMEM_COLS>(tmem_slot);
    else tc::tmem_alloc<C::TMEM_COLS>(tmem_slot);
  }
  tc::tc_fence_before();
  if constexpr (PAIR) tc::cluster_sync();  // the peer's barriers are initialised
  else __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // (PDL) everything above overlapped the previous kernel's tail; global
  // memory is touched only from here on
  tc::pdl_wait();
  tc::pdl_launch_dependents();

  // tile -> (m, n, split) for the tile0 + k * tstep walk of every role,
  // advanced with carries (no divisions per tile)
  auto decode = [&](const TileWalk& w, int& m, int& n, int& split) {
    n = w.n;
    m = w.mu;
    split = w.sp;
    if (p.cls_n) {  // split = the sub-pixel class
      const int cr = w.n / p.n_tiles;
      n = w.n - cr * p.n_tiles;
      split = (cr + w.mu) % p.cls_n;
    }
    if constexpr (PAIR) m = 2 * m + (int)rank;
  };
  // the accumulator stage has been read: hand it back to the MMA issuer
  auto release_acc = [&](int acc) {
    tc::tc_fence_before();
    if constexpr (PAIR) {
      __syncwarp();
      if (tc::lane_id() == 0) tc::mbar_arrive_cluster(tc::mapa(&tempty[acc], 0));
    } else {
      tc::mbar_arrive(&tempty[acc]);
    }
  };
  auto k_range = [&](int split, int& kb0, int& kb1) {
    if (p.cls_n) {
      kb0 = p.cls_kb[split];
      kb1 = p.cls_kb[split + 1];
      return;
    }
    if (p.k_ilv) {  // virtual range [0, k-blocks of this split's chunks)
      const int Q = p.k_ilv, nch = (p.k_blocks + Q - 1) / Q;
      const int mine = split < nch ? (nch - split + p.splits - 1) / p.splits : 0;
      const bool has_last = mine > 0 && (nch - 1 - split) % p.splits == 0;
      kb0 = 0;
      kb1 = mine * Q - (has_last ? nch * Q - p.k_blocks : 0);
      return;
    }
    kb0 = split * kb_per_split;
    kb1 = min(p.k_blocks, kb0 + kb_per_split);
  };

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (tc::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      TileWalk tw(tile0, tstep, nt_walk, m_units);
      for (int tile = tile0; tile < total_tiles; tile += tstep, tw.next()) {
        int m, n, split, kb0, kb1;
        decode(tw, m, n, split);
        k_range(split, kb0, kb1);
        if constexpr (PAIR) m = min(m, p.m_tiles - 1);  // padding tile: load a valid one
        // M-side row coordinates of this tile (K-major operands).
        int m_clip = 0, m_row = m * (p.m_rows ? p.m_rows : BM);
        const bool m_rem = p.rem_rows && m >= p.rem_tiles0;
        if (m_rem) {
          m_clip = (m - p.rem_tiles0) * p.rem_clips;
          m_row = p.tiles_per_clip * BM;
        } else if (p.map_mode == MAP_CLIP) {
          m_clip = m / p.tiles_per_clip;
          m_row = (m - m_clip * p.tiles_per_clip) * BM;
        }
        // im2col operands: per-tile pixel origin (K-major A) and per-slab
        // tap offsets (MN-major B, slabs span N), hoisted out of the K loop.
        PixOrigin a_org{0, 0, 0};
        TapCursor a_cur{0, 0, 0};
        if (!AMN && p.a.mode == LOAD_IM2COL) {
          a_org = pix_origin(p.a, m_clip * p.a.rows_per_clip + m_row);
          a_cur.init(p.a, kb0 * BK);
        }
        // per-slab tap cursors for MN-major im2col operands (slabs span M/N)
        constexpr int kAIm = AMN && C::A_SLABS <= 8 ? C::A_SLABS : 1;
        TapCursor a_tap[kAIm];
        const bool a_im2col_mn = AMN && p.a.mode == LOAD_IM2COL;
        if (a_im2col_mn) {
#pragma unroll
          for (int j = 0; j < kAIm; ++j) a_tap[j].init(p.a, m * BM + j * KCA);
        }
        constexpr int kBIm = BMN && C::B_SLABS <= 8 ? C::B_SLABS : 1;
        TapCursor b_tap[kBIm];
        const bool b_im2col = BMN && p.b.mode == LOAD_IM2COL;
        if (b_im2col) {
#pragma unroll
          for (int j = 0; j < kBIm; ++j) b_tap[j].init(p.b, n * BN + (int)rank * C::BNL + j * KCB);
        }
        // K-side (clip, k-block in clip) of MN-major operands (K = pixels),
        // one division per tile, then stepped
        // real k-block (interleaved: the first of this split's chunk) and
        // the blocks left in the chunk
        int kreal = p.k_ilv ? split * p.k_ilv : kb0;
        int kleft = p.k_ilv ? p.k_ilv : kb1 - kb0;
        int kc_clip = 0, kc_in = kreal;
        auto k_clip_of = [&]() {
          if (p.kb_per_clip > 0) {
            kc_clip = kreal / p.kb_per_clip;
            kc_in = kreal - kc_clip * p.kb_per_clip;
          } else {
            kc_in = kreal;
          }
        };
        k_clip_of();
        for (int kv = kb0; kv < kb1; ++kv) {
          const int kb = kreal;
          bool jumped = false;
          if (++kreal, --kleft == 0 && p.k_ilv) {  // next chunk of this split
            kreal += (p.splits - 1) * p.k_ilv;
            kleft = p.k_ilv;
            jumped = true;
          }
          tc::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * C::STAGE_BYTES;
          uint8_t* sb = sa + C::A_BYTES;
          // pairs: the leader's barrier expects both CTAs' bytes
          if (!PAIR) tc::mbar_arrive_expect_tx(&full[stage], C::STAGE_BYTES);
          else if (rank == 0) tc::mbar_arrive_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
          const bool k_rem = p.krem_rows && kb >= p.krem0;
          int k_clip = kc_clip, k_row = kc_in * BKT;
          if (k_rem) {
            k_clip = (kb - p.krem0) * p.krem_clips;
            k_row = p.kb_per_clip * BKT;
          } else if (++kc_in == p.kb_per_clip) {
            kc_in = 0;
            ++kc_clip;
          }
          if constexpr (!AMN) {
            if (p.a.mode == LOAD_IM2COL) {
#pragma unroll 1
              for (int j = 0; j < C::A_SLABS; ++j) {
                ldi<CG>(sa + j * C::A_SLAB_BYTES, &map_a, &full[stage], a_cur.c, a_org.w,
                        a_org.h, a_org.f, (uint16_t)a_cur.s, (uint16_t)a_cur.r);
                a_cur.advance(p.a, KCA);
              }
            } else {
#pragma unroll 1
              for (int j = 0; j < C::A_SLABS; ++j)
                load_slab<CG>(p.a, m_rem ? &map_res : &map_a, sa + j * C::A_SLAB_BYTES,
                              &full[stage], kb * BK + j * KCA, m_clip, m_row);
            }
          } else {
            if (a_im2col_mn) {
              const PixOrigin o = pix_origin(p.a, k_clip * p.a.rows_per_clip + k_row);
#pragma unroll
              for (int j = 0; j < kAIm; ++j)
                ldi<CG>(sa + j * C::A_SLAB_BYTES, &map_a, &full[stage], a_tap[j].c, o.w, o.h,
                        o.f, (uint16_t)a_tap[j].s, (uint16_t)a_tap[j].r);
            } else {
#pragma unroll 1
              for (int j = 0; j < C::A_SLABS; ++j)
                load_slab<CG>(p.a, k_rem ? &map_res : &map_a, sa + j * C::A_SLAB_BYTES,
                              &full[stage], m * BM + j * KCA, k_clip, k_row);
            }
          }
          if constexpr (!BMN) {
            // pairs: this CTA's half of the N tile (B rows)
#pragma unroll 1
            for (int j = 0; j < C::B_SLABS; ++j)
              load_slab<CG>(p.b, &map_b, sb + j * C::B_SLAB_BYTES, &full[stage],
                            kb * BK + j * KCB, 0, n * BN + (int)rank * C::BNL);
          } else {
            if (b_im2col) {
              const PixOrigin o = pix_origin(p.b, k_clip * p.b.rows_per_clip + k_row);
#pragma unroll
              for (int j = 0; j < kBIm; ++j)
                ldi<CG>(sb + j * C::B_SLAB_BYTES, &map_b, &full[stage], b_tap[j].c, o.w, o.h,
                        o.f, (uint16_t)b_tap[j].s, (uint16_t)b_tap[j].r);
            } else {
#pragma unroll 1
              for (int j = 0; j < C::B_SLABS; ++j)
                load_slab<CG>(p.b, k_rem ? &map_mask : &map_b, sb + j * C::B_SLAB_BYTES,
                              &full[stage], n * BN + (int)rank * C::BNL + j * KCB, k_clip,
                              k_row);
            }
          }
          if (jumped) k_clip_of();  // (the clip / row of the next chunk's first block)
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (!AMN && !PAIR) {
          // fused residual: A-shaped tiles of the residual (channels of this N
          // tile), C::RES_PER_STAGE of them packed into each stage so the
          // HBM-latency-bound residual stream keeps whole stages in flight
          for (int rk0 = 0; rk0 < p.res_kb; rk0 += C::RES_PER_STAGE) {
            const int nq = min(C::RES_PER_STAGE, p.res_kb - rk0);
            tc::mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sa = smem + stage * C::STAGE_BYTES;
            tc::mbar_arrive_expect_tx(&full[stage], nq * C::A_BYTES);
#pragma unroll 1
            for (int q = 0; q < nq; ++q)
#pragma unroll 1
              for (int j = 0; j < C::A_SLABS; ++j)
                load_slab(p.r, &map_res, sa + q * C::A_BYTES + j * C::A_SLAB_BYTES, &full[stage],
                          n * BN + (rk0 + q) * BK + j * KCA, m_clip, m_row);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (pair: the leader only) =====================
    constexpr uint32_t idesc = tc::idesc_bf16(BM * CG, BN, AMN, BMN);
    auto mma = [&](uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc_on) {
      if constexpr (PAIR) tc::mma_bf16_cg2(d, a, b, id, acc_on);
      else tc::mma_bf16(d, a, b, id, acc_on);
    };
    auto commit = [&](uint64_t* bar) {
      if constexpr (PAIR) tc::mma_commit_cg2(bar, 0x3);  // both CTAs' barriers
      else tc::mma_commit(bar);
    };
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    TileWalk tw(tile0, tstep, nt_walk, m_units);
    for (int tile = tile0; tile < total_tiles && (!PAIR || rank == 0);
         tile += tstep, ++it, tw.next()) {
      int m, n, split, kb0, kb1;
      decode(tw, m, n, split);
      k_range(split, kb0, kb1);
      const int acc = it & 1;
      tc::mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
      tc::tc_fence_after();
      const uint32_t tmem_d = tmem_base + acc * BN;
      for (int kb = kb0; kb < kb1; ++kb) {
        tc::mbar_wait(&full[stage], phase);
        tc::tc_fence_after();
        if (tc::elect_one()) {
          const uint32_t sa = tc::smem_u32(smem + stage * C::STAGE_BYTES);
          const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
          for (int j = 0; j < BKT / 16; ++j) {
            const uint64_t ad = operand_desc<KCA, AMN, C::A_ROWS, C::A_SLAB_BYTES>(sa, j);
            const uint64_t bd = operand_desc<KCB, BMN, C::B_ROWS, C::B_SLAB_BYTES>(sb, j);
            mma(tmem_d, ad, bd, idesc, (kb > kb0 || j > 0) ? 1u : 0u);
          }
          commit(PAIR && p.db_mode ? &consumed[stage] : &empty[stage]);
          if (kb == kb1 - 1 && p.res_kb == 0) commit(&tfull[acc]);
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if constexpr (!AMN && !PAIR) {
        // fused residual: D[:, 64 rk + i] += residual[:, n BN + 64 rk + i]
        constexpr uint32_t idesc64 = tc::idesc_bf16(BM, 64, false, false);
        for (int rk0 = 0; rk0 < p.res_kb; rk0 += C::RES_PER_STAGE) {
          const int nq = min(C::RES_PER_STAGE, p.res_kb - rk0);
          tc::mbar_wait(&full[stage], phase);
          tc::tc_fence_after();
          if (tc::elect_one()) {
            const uint32_t sb = tc::smem_u32(ident);
            for (int q = 0; q < nq; ++q) {
              const uint32_t sa = tc::smem_u32(smem + stage * C::STAGE_BYTES) + q * C::A_BYTES;
#pragma unroll
              for (int j = 0; j < BK / 16; ++j) {
                const uint64_t ad = operand_desc<KCA, false, C::A_ROWS, C::A_SLAB_BYTES>(sa, j);
                const uint64_t bd = operand_desc<64, false, 64, kIdentBytes>(sb, j);
                tc::mma_bf16(tmem_d + 64 * (rk0 + q), ad, bd, idesc64, 1u);
              }
            }
            tc::mma_commit(&empty[stage]);
            if (rk0 + nq == p.res_kb) tc::mma_commit(&tfull[acc]);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (kb1 <= kb0) {
        // empty K range (split beyond k_blocks): publish a zero tile
        if (tc::elect_one()) commit(&tfull[acc]);
        __syncwarp();
      }
    }
  } else if (warp >= kBiasWarp0) {
    // ===================== bias-gradient warps =====================
    // Every stage waits for these warps' arrival (the second on `empty`), so
    // they stay in lockstep with the producer — they must never run ahead:
    // an mbarrier parity wait cannot tell phase P from P-2.  For the tiles
    // that own the bias sum (n == 0 when dY is the A operand, m == 0 when it
    // is B) they also read the dY stage (MN-major [64 pixel rows][64 ch]
    // slabs, 128 B swizzle) with 16-byte loads.  Fixed-order reductions.
    if (p.db_mode) {
      const int bt = threadIdx.x - (64 + kEpiThreads);  // 0..63
      const bool on_a = p.db_mode == 1;
      const int nchunk = on_a ? BM / 8 : 8;  // 16-byte chunks across the dY channels
      const int cc = bt % nchunk, rg = bt / nchunk, nrg = 64 / nchunk;
      __shared__ float red[16][8];
      int stage = 0;
      uint32_t phase = 0;
      TileWalk tw(tile0, tstep, nt_walk, m_units);
      for (int tile = tile0; tile < total_tiles; tile += tstep, tw.next()) {
        int m, n, split, kb0, kb1;
        decode(tw, m, n, split);
        k_range(split, kb0, kb1);
        // (a pair's padding tile loads a copy of a valid tile: no sum)
        const bool sums = (on_a ? n == 0 : m == 0) && m < p.m_tiles;
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int kb = kb0; kb < kb1; ++kb) {
          // pairs: this CTA's stage is complete once the pair's MMA consumed it
          // (the leader's full barrier counted both CTAs' bytes)
          tc::mbar_wait(PAIR ? &consumed[stage] : &full[stage], phase);
          if (sums) {
            const uint8_t* slab = smem + stage * C::STAGE_BYTES + (on_a ? 0 : C::A_BYTES) +
                                  (cc >> 3) * (BKT * 64 * 2);
            const int c = cc & 7;
#pragma unroll 4
            for (int r = rg; r < BKT; r += nrg) {
              const uint4 v = *reinterpret_cast<const uint4*>(slab + r * 128 + ((c ^ (r & 7)) << 4));
              const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&v);
#pragma unroll
              for (int i = 0; i < 8; ++i) acc[i] += __bfloat162float(e[i]);
            }
          }
          tc::named_bar(kBarDb, 64);
          if (bt == 0) tc::mbar_arrive(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (sums) {
          // combine row groups: within each warp by shuffles, then the second warp -> the first
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], 16);
            if (!on_a) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], 8);
          }
          const int lane = bt & 31;
          if (warp == kBiasWarp0 + 1 && lane < nchunk)
#pragma unroll
            for (int i = 0; i < 8; ++i) red[lane][i] = acc[i];
          tc::named_bar(kBarDb, 64);
          if (warp == kBiasWarp0 && lane < nchunk) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int co = (on_a ? m * BM : 0) + lane * 8 + i;
              if (co < p.db_c) p.db_part[(long long)split * p.db_c + co] = acc[i] + red[lane][i];
            }
          }
          tc::named_bar(kBarDb, 64);
        }
      }
    }
  } else if (tma_epi) {
    // ===================== epilogue (warps 2..9), TMA path =====================
    // Compiled once per feature set (residual, bf16 mask, mask bits, bits
    // out, adjoint shift) used by the network, plus a runtime-flag fallback:
    // each hot loop then carries only its own work (the loop is latency-
    // and issue-sensitive; dead optional branches cost measurable time).
    uint8_t* const out_buf0 = out_buf;
    uint8_t* const res_buf0 = res_buf;
    uint8_t* const mask_buf0 = mask_buf;
    uint64_t* const resbar0 = resbar;
    auto tma_epilogue = [&](auto flags) {
      constexpr int EF = decltype(flags)::value;  // -1: runtime flags
      const bool E_RES = EF < 0 ? has_res : (EF & 1) != 0;
      const bool E_MASK = EF < 0 ? has_mask : (EF & 2) != 0;
      const bool E_MBITS = EF < 0 ? p.mask_bits != nullptr : (EF & 4) != 0;
      const bool E_BOUT = EF < 0 ? p.bits_out != nullptr : (EF & 8) != 0;
      const bool E_SHIFT = EF < 0 ? p.shift_out != 0 : (EF & 16) != 0;
      // strided row scatter (sub-pixel / strided-1x1 dgrad): no TMA box maps
      // the scattered rows, so the staged sub-tile is stored by the group's
      // threads, 4 lanes per 64-byte row segment
      const bool E_SCAT = EF < 0 ? p.scatter != 0 : (EF & 32) != 0;
      const bool E_ACC = EF < 0 ? p.acc_out != 0 : (EF & 64) != 0;
      // ===================== epilogue (warps 2..9), TMA path =====================
      // Two groups of 4 warps (one warp per TMEM lane quarter each) take
      // alternate 32-column sub-tiles, each with its own staging buffers,
      // residual/mask ring, mbarriers and named barrier.
      constexpr int NSUB = BN / EC;
      const int grp = (int)(warp - 2) >> 2;
      // Tile `it`: group grp takes sub-tiles s = s0 + kGroups * u with
      // s0 = (grp - it) mod kGroups — rotating the assignment over tiles
      // balances groups when kGroups does not divide NSUB (BN = 64 / 128).
      int gs_next = 0;  // this group's ring sequence number of its next sub-tile
      const int q = warp & 3;  // TMEM lane quarter this warp may access
      const int lrow = q * 32 + tc::lane_id();
      const bool leader = threadIdx.x == 64 + 128 * grp;
      const uint32_t bar_id = 1 + grp;
      const int OS = p.out_slots;  // 2: double-buffered staging; 1: K-heavy GEMMs keep the operand ring
      uint8_t* out_buf = out_buf0 + grp * OS * kSubBytes;
      uint8_t* res_buf = res_buf0 + grp * 2 * kSubBytes;
      uint8_t* mask_buf = mask_buf0 + grp * 2 * kSubBytes;
      uint64_t* resbar = resbar0 + grp * 2;
      const bool loads = E_RES || E_MASK;
      const uint32_t load_bytes = (E_RES ? kSubBytes : 0) + (E_MASK ? kSubBytes : 0);
      // bias -> shared memory once per CTA (an L2 round trip per sub-tile
      // otherwise sits on the epilogue's critical path)
      const bool has_bias = p.bias != nullptr;
      if (has_bias) {
        for (int i = threadIdx.x - 64; i < p.n_tiles * BN; i += kEpiThreads)
          bias_s[i] = i < p.n_total ? __ldg(p.bias + i) : 0.f;
        tc::named_bar(kBarBias, kEpiThreads);
      }
      int it = 0;
      const tc::FastDiv div_g((uint32_t)max(p.sc_wo * p.sc_ho, 1));
      const tc::FastDiv div_w((uint32_t)max(p.sc_wo, 1));
      TileWalk tw(tile0, tstep, nt_walk, m_units);
      for (int tile = tile0; tile < total_tiles; tile += tstep, ++it, tw.next()) {
        int m, n, split;
        decode(tw, m, n, split);
        int clip = 0, r0 = m * (p.m_rows ? p.m_rows : BM);
        const bool m_rem = p.rem_rows && m >= p.rem_tiles0;
        if (m_rem) {
          clip = (m - p.rem_tiles0) * p.rem_clips;
          r0 = p.tiles_per_clip * BM;
        } else if (p.map_mode == MAP_CLIP) {
          clip = m / p.tiles_per_clip;
          r0 = (m - clip * p.tiles_per_clip) * BM;
        }
        auto row_off = [&](int col) {
          if (!E_SHIFT) return 0;
          return col < p.sg0 ? -p.hw : (col < p.sg1 ? p.hw : 0);
        };
        auto issue_loads = [&](int sub, int slot) {
          const int col = n * BN + sub * EC;
          const int r = r0 + row_off(col);
          tc::mbar_arrive_expect_tx(&resbar[slot], load_bytes);
          if (p.map_mode == MAP_CLIP) {
            if (E_RES) tc::tma_load_3d(res_buf + slot * kSubBytes, &map_res, &resbar[slot], col, r, clip);
            if (E_MASK)
              tc::tma_load_3d(mask_buf + slot * kSubBytes, &map_mask, &resbar[slot], col, r, clip);
          } else {
            if (E_RES) tc::tma_load_2d(res_buf + slot * kSubBytes, &map_res, &resbar[slot], col, r);
            if (E_MASK) tc::tma_load_2d(mask_buf + slot * kSubBytes, &map_mask, &resbar[slot], col, r);
          }
        };
        const int s0 = (grp - it % kGroups + kGroups) % kGroups;
        const int NSUB_G = (NSUB - s0 + kGroups - 1) / kGroups;  // may be 0
        // group-local sub-tile u covers columns [(kGroups * u + s0) * EC, +EC)
        const int gs0 = gs_next;
        gs_next += NSUB_G;
        // (multiply-high divisions, m_total < 2^31: 64-bit divisions were a
        // quarter of the sub-pixel dgrad's issue slots)
        const int sc_oh = p.cls_n ? p.cls_oh[split] : p.sc_oh;
        const int sc_ow = p.cls_n ? p.cls_ow[split] : p.sc_ow;
        auto scat = [&](long long r) -> long long {
          if (r >= p.m_total) return -1;
          const uint32_t ru = (uint32_t)r;
          const uint32_t f = div_g.div(ru), rem = ru - f * div_g.d;
          const uint32_t a = div_w.div(rem), b = rem - a * div_w.d;
          return (long long)f * p.sc_hi * p.sc_wi +
                 (long long)((a * p.sc_stride + sc_oh) * p.sc_wi + b * p.sc_stride + sc_ow);
        };
        const int gt = (int)threadIdx.x - 64 - 128 * grp;  // thread within the group
        long long srow[4] = {-1, -1, -1, -1}, my_srow = -1;
        if (E_SCAT) {  // rows are the same for every sub-tile of the tile
          if (!p.sc_tma) {
#pragma unroll
            for (int k = 0; k < 4; ++k) srow[k] = scat((long long)r0 + (gt >> 2) + 32 * k);
          }
          my_srow = scat((long long)r0 + lrow);
        }
        if (PAIR && m >= p.m_tiles) gs_next = gs0;  // padding tile: no sub-tiles consumed
        if (leader && loads && !(PAIR && m >= p.m_tiles)) {
          if (NSUB_G > 0) issue_loads(s0, gs0 & 1);
          if (NSUB_G > 1) issue_loads(kGroups + s0, (gs0 + 1) & 1);
        }
        const int acc = it & 1;
        tc::mbar_wait(&tfull[acc], (it >> 1) & 1);
        tc::tc_fence_after();
        // more groups than sub-tiles (BN = 64), or a pair's padding tile:
        // nothing to store
        if (NSUB_G == 0 || (PAIR && m >= p.m_tiles)) {
          release_acc(acc);
          continue;
        }
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
        // row of this thread in the output (and mask) for sub-tile u; -1 if none
        auto out_row = [&](int u) -> long long {
          if (E_SCAT) return my_srow;
          if (m_rem) {  // row lrow % rem_rows of clip clip + lrow / rem_rows
            const int ci = clip + lrow / p.rem_rows;
            return ci < p.n_clips
                       ? (long long)ci * p.rows_per_clip + r0 + lrow % p.rem_rows : -1;
          }
          const int r = r0 + row_off(n * BN + (kGroups * u + s0) * EC) + lrow;
          if (p.map_mode == MAP_CLIP)
            return (r >= 0 && r < p.rows_per_clip) ? (long long)clip * p.rows_per_clip + r : -1;
          return r < p.m_total ? r : -1;
        };
        auto load_mbits = [&](int u) -> uint32_t {
          const long long row = out_row(u);
          return row >= 0 ? __ldg(p.mask_bits + row * p.bits_ld + (n * BN + (kGroups * u + s0) * EC) / 32)
                          : 0u;
        };
        uint32_t mbits_next = (E_MBITS && NSUB_G > 0) ? load_mbits(0) : 0u;
  #pragma unroll 1
        for (int u = 0; u < NSUB_G; ++u) {
          const int s = kGroups * u + s0;
          const int gs = gs0 + u, slot = gs & 1;
          const uint32_t mbits = mbits_next;  // prefetched one sub-tile ahead
          if (E_MBITS && u + 1 < NSUB_G) mbits_next = load_mbits(u + 1);
          // accumulate-scatter: the rows' current values, loaded before the
          // math so their latency overlaps it
          uint4 oldv[4];
          if (E_ACC) {
            const int ccol = n * BN + s * EC + 8 * (gt & 3);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              oldv[k] = (srow[k] >= 0 && ccol < p.n_total)
                            ? *reinterpret_cast<const uint4*>(p.out + srow[k] * p.ldo + ccol)
                            : make_uint4(0, 0, 0, 0);
          }
          uint32_t raw0[16], raw1[16];
          tc::tmem_ld_32x32b_x16(taddr + s * EC, raw0);
          tc::tmem_ld_32x32b_x16(taddr + s * EC + 16, raw1);
          tc::tmem_ld_wait();
          if (u == NSUB_G - 1) release_acc(acc);  // this group's part read
          const int col0 = n * BN + s * EC;
          float v[32];
  #pragma unroll
          for (int i = 0; i < 16; ++i) {
            v[i] = __uint_as_float(raw0[i]);
            v[16 + i] = __uint_as_float(raw1[i]);
          }
          if (has_bias) {
  #pragma unroll
            for (int j = 0; j < 8; ++j) {
              const float4 bb = reinterpret_cast<const float4*>(bias_s + col0)[j];
              v[4 * j + 0] += bb.x;
              v[4 * j + 1] += bb.y;
              v[4 * j + 2] += bb.z;
              v[4 * j + 3] += bb.w;
            }
          }
          if (p.relu && !E_RES) {
  #pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
          }
          if (loads) tc::mbar_wait(&resbar[slot], (gs >> 1) & 1);
          if (E_RES) {
            const uint8_t* rb = res_buf + slot * kSubBytes;
  #pragma unroll
            for (int c = 0; c < 4; ++c) {
              const uint4 rr = *reinterpret_cast<const uint4*>(rb + sw64_off(lrow, c));
              const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&rr);
  #pragma unroll
              for (int i = 0; i < 8; ++i) v[8 * c + i] += __bfloat162float(e[i]);
            }
            if (p.relu) {
  #pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = fmaxf(v[i], 0.f);
            }
          }
          if (E_MASK) {
            const uint8_t* mb = mask_buf + slot * kSubBytes;
  #pragma unroll
            for (int c = 0; c < 4; ++c) {
              const uint4 mm = *reinterpret_cast<const uint4*>(mb + sw64_off(lrow, c));
              const __nv_bfloat16* e = reinterpret_cast<const __nv_bfloat16*>(&mm);
  #pragma unroll
              for (int i = 0; i < 8; ++i) v[8 * c + i] = __bfloat162float(e[i]) > 0.f ? v[8 * c + i] : 0.f;
            }
          }
          uint32_t o[16];
  #pragma unroll
          for (int j = 0; j < 16; ++j) o[j] = tc::pack_bf16(v[2 * j], v[2 * j + 1]);
          if (E_MBITS) {  // relu_backward from the bitmask, on the packed values
  #pragma unroll
            for (int j = 0; j < 16; ++j) o[j] &= tc::bits_keep(mbits, j);
          }
          if (E_BOUT) {  // forward: record bf16(out) > 0 for the backward masks
            const long long row = out_row(u);
            const uint32_t word = tc::relu_bits16(o);
            if (row >= 0 && col0 < p.n_total) p.bits_out[row * p.bits_ld + col0 / 32] = word;
          }
          // staging buffer `slot` was last stored two sub-tiles ago
          if (leader) {
            if (OS == 2) tc::bulk_wait_read<1>();
            else tc::bulk_wait_read<0>();
          }
          tc::named_bar(bar_id, 128);
          if (leader && loads && u + 2 < NSUB_G) issue_loads(s + 2 * kGroups, slot);
          const int rdst = r0 + row_off(col0);
          if (rdst < 0) {
            // Adjoint-shift rows moving above the clip start: TMA stores reject
            // negative coordinates, so this sub-tile is stored per thread and
            // the rows that leave the clip are dropped.
            // (a tile may also run past the clip's last row when the clip is
            // shorter than the tile: those rows belong to the next clip)
            const int myrow = rdst + lrow;
            if (myrow >= 0 && myrow < p.rows_per_clip && r0 + lrow < p.rows_per_clip &&
                col0 < p.n_total) {
              uint4* dst = reinterpret_cast<uint4*>(
                  p.out + ((long long)clip * p.rows_per_clip + myrow) * p.ldo + col0);
  #pragma unroll
              for (int c = 0; c < 4; ++c)
                dst[c] = make_uint4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
            }
            continue;
          }
          uint8_t* ob = out_buf + (OS == 2 ? slot : 0) * kSubBytes;
  #pragma unroll
          for (int c = 0; c < 4; ++c)
            *reinterpret_cast<uint4*>(ob + sw64_off(lrow, c)) =
                make_uint4(o[4 * c], o[4 * c + 1], o[4 * c + 2], o[4 * c + 3]);
          tc::fence_proxy_async();
          tc::named_bar(bar_id, 128);
          if (E_SCAT && p.sc_tma) {  // row-aligned tile: one box of the class map
            if (leader && col0 < p.n_total) {
              tc::tma_store_5d(&map_out, ob, col0, sc_ow, 0, sc_oh, m * p.sc_rows);
              tc::bulk_commit();
            }
            continue;
          }
          if (E_SCAT) {
            if (col0 < p.n_total) {
              const int c = gt & 3;
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                if (srow[k] < 0) continue;
                uint4 vv = *reinterpret_cast<const uint4*>(ob + sw64_off((gt >> 2) + 32 * k, c));
                uint4* dst = reinterpret_cast<uint4*>(p.out + srow[k] * p.ldo + col0 + 8 * c);
                if (E_ACC) {
                  const uint4 old = oldv[k];
                  vv.x = tc::pack_bf16(tc::bf16_lo(old.x) + tc::bf16_lo(vv.x), tc::bf16_hi(old.x) + tc::bf16_hi(vv.x));
                  vv.y = tc::pack_bf16(tc::bf16_lo(old.y) + tc::bf16_lo(vv.y), tc::bf16_hi(old.y) + tc::bf16_hi(vv.y));
                  vv.z = tc::pack_bf16(tc::bf16_lo(old.z) + tc::bf16_lo(vv.z), tc::bf16_hi(old.z) + tc::bf16_hi(vv.z));
                  vv.w = tc::pack_bf16(tc::bf16_lo(old.w) + tc::bf16_lo(vv.w), tc::bf16_hi(old.w) + tc::bf16_hi(vv.w));
                }
                *dst = vv;
              }
            }
            continue;
          }
          if (leader && col0 < p.n_total) {
            const int r = r0 + row_off(col0);
            if (m_rem) tc::tma_store_3d(&map_mask, ob, col0, r0, clip);
            else if (p.map_mode == MAP_CLIP) tc::tma_store_3d(&map_out, ob, col0, r, clip);
            else tc::tma_store_2d(&map_out, ob, col0, r);
            tc::bulk_commit();
          }
        }
      }
      if (leader) tc::bulk_wait<0>();
    };
    const int ef = (has_res ? 1 : 0) | (has_mask ? 2 : 0) | (p.mask_bits ? 4 : 0) |
                   (p.bits_out ? 8 : 0) | (p.shift_out ? 16 : 0) | (p.scatter ? 32 : 0) |
                   (p.acc_out ? 64 : 0);
    switch (ef) {
      case 0: tma_epilogue(std::integral_constant<int, 0>{}); break;    // plain (proj)
      case 8: tma_epilogue(std::integral_constant<int, 8>{}); break;    // fwd + bits
      case 9: tma_epilogue(std::integral_constant<int, 9>{}); break;    // fwd + res + bits
      case 4: tma_epilogue(std::integral_constant<int, 4>{}); break;    // dgrad + mask bits
      case 21: tma_epilogue(std::integral_constant<int, 21>{}); break;  // dgrad c1 (shift)
      case 17: tma_epilogue(std::integral_constant<int, 17>{}); break;  // dgrad c1, no mask
      case 20: tma_epilogue(std::integral_constant<int, 20>{}); break;  // dgrad c1, proj added after
      case 36: tma_epilogue(std::integral_constant<int, 36>{}); break;  // sub-pixel dgrad + bits
      case 32: tma_epilogue(std::integral_constant<int, 32>{}); break;  // strided 1x1 dgrad
      case 100: tma_epilogue(std::integral_constant<int, 100>{}); break;  // += proj dgrad, bits
      default: tma_epilogue(std::integral_constant<int, -1>{}); break;
    }
  } else {
    // ===================== epilogue (warps 2..9), direct path =====================
    // group g handles the 16-column chunks c0 = 16 ((g - it) mod kGroups) + 16 kGroups i
    // (rotated over tiles like the TMA path)
    const int grp = (int)(warp - 2) >> 2;
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int lrow = q * 32 + tc::lane_id();
    int it = 0;
    TileWalk tw(tile0, tstep, nt_walk, m_units);
    for (int tile = tile0; tile < total_tiles; tile += tstep, ++it, tw.next()) {
      int m, n, split, kb0, kb1;
      decode(tw, m, n, split);
      k_range(split, kb0, kb1);
      const int acc = it & 1;
      tc::mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc::tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      const bool has_k = kb1 > kb0;

      if (p.epi == EPI_BF16) {
        // output row of this thread
        long long row;
        bool valid;
        int t_frame = 0;
        if (p.map_mode == MAP_CLIP) {
          const int clip = m / p.tiles_per_clip;
          const int r = (m - clip * p.tiles_per_clip) * BM + lrow;
          valid = r < p.rows_per_clip;
          row = (long long)clip * p.rows_per_clip + r;
        } else {
          const long long r = (long long)m * BM + lrow;
          valid = r < p.m_total;
          row = r;
        }
        // (32-bit: rows < 2^31)
        if (p.shift_out) t_frame = (int)(((uint32_t)row / (uint32_t)p.hw) % (uint32_t)p.frames);
        if (p.scatter) {
          const uint32_t ru = (uint32_t)row, g = (uint32_t)(p.sc_wo * p.sc_ho);
          const uint32_t f = ru / g, rem = ru - f * g;
          const uint32_t ho = rem / (uint32_t)p.sc_wo, wo = rem - ho * (uint32_t)p.sc_wo;
          row = (long long)f * p.sc_hi * p.sc_wi +
                (long long)((ho * p.sc_stride + (p.cls_n ? p.cls_oh[split] : p.sc_oh)) * p.sc_wi +
                            wo * p.sc_stride + (p.cls_n ? p.cls_ow[split] : p.sc_ow));
        }
#pragma unroll 1
        for (int c0 = 16 * ((grp - it % kGroups + kGroups) % kGroups); c0 < BN; c0 += 16 * kGroups) {
          uint32_t raw[16];
          tc::tmem_ld_32x32b_x16(taddr + c0, raw);
          tc::tmem_ld_wait();
          const int col0 = n * BN + c0;
          if (!valid || col0 >= p.n_total) continue;
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = has_k ? __uint_as_float(raw[i]) : 0.f;
          if (p.bias) {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] += __ldg(p.bias + col0 + i);
          }
          if (p.relu && !p.residual) {
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = fmaxf(v[i], 0.f);
          }
          // two 8-column (16 B) pieces, each may land on its own row
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int cc = col0 + 8 * h;
            long long drow = row;
            bool zero_src = false;
            if (p.shift_out) {
              if (cc < p.sg0) {  // adjoint: value of frame t belongs to frame t-1
                if (t_frame >= 1) drow = row - p.hw;
                else { drow = row + (long long)(p.frames - 1) * p.hw; zero_src = true; }
              } else if (cc < p.sg1) {  // value of frame t belongs to frame t+1
                if (t_frame + 1 < p.frames) drow = row + p.hw;
                else { drow = row - (long long)(p.frames - 1) * p.hw; zero_src = true; }
              }
            }
            float w8[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) w8[i] = zero_src ? 0.f : v[8 * h + i];
            const long long off = drow * p.ldo + cc;
            if (p.residual) {
              const uint4 rr = *reinterpret_cast<const uint4*>(p.residual + off);
              const __nv_bfloat16* rb = reinterpret_cast<const __nv_bfloat16*>(&rr);
#pragma unroll
              for (int i = 0; i < 8; ++i) w8[i] += __bfloat162float(rb[i]);
              if (p.relu) {
#pragma unroll
                for (int i = 0; i < 8; ++i) w8[i] = fmaxf(w8[i], 0.f);
              }
            }
            if (p.mask_bits) {
              const uint32_t mw = __ldg(p.mask_bits + drow * p.bits_ld + cc / 32);
#pragma unroll
              for (int i = 0; i < 8; ++i) w8[i] = tc::bit_of(mw, cc % 32 + i) ? w8[i] : 0.f;
            }
            if (p.mask) {
              const uint4 mm = *reinterpret_cast<const uint4*>(p.mask + off);
              const __nv_bfloat16* mb = reinterpret_cast<const __nv_bfloat16*>(&mm);
#pragma unroll
              for (int i = 0; i < 8; ++i)
                w8[i] = __bfloat162float(mb[i]) > 0.f ? w8[i] : 0.f;
            }
            uint4 o;
            o.x = tc::pack_bf16(w8[0], w8[1]);
            o.y = tc::pack_bf16(w8[2], w8[3]);
            o.z = tc::pack_bf16(w8[4], w8[5]);
            o.w = tc::pack_bf16(w8[6], w8[7]);
            *reinterpret_cast<uint4*>(p.out + off) = o;
          }
        }
      } else {
        // EPI_F32: partial tile of the split-K wgrad, rows = M (c_out side)
        const int mrow = m * BM + lrow;
        float* base = p.out_f32 + (long long)split * p.m_total * p.n_total;
#pragma unroll 1
        for (int c0 = 16 * ((grp - it % kGroups + kGroups) % kGroups); c0 < BN; c0 += 16 * kGroups) {
          uint32_t raw[16];
          tc::tmem_ld_32x32b_x16(taddr + c0, raw);
          tc::tmem_ld_wait();
          const int col0 = n * BN + c0;
          if (mrow >= p.m_total || col0 >= p.n_total) continue;
          if (col0 + 16 > p.n_total) {
            // ragged last chunk (e.g. a 392-column weight gradient)
            for (int i = 0; i < 16 && col0 + i < p.n_total; ++i) {
              const float v = has_k ? __uint_as_float(raw[i]) : 0.f;
              if (!p.transpose_f32) base[(long long)mrow * p.n_total + col0 + i] = v;
              else base[(long long)(col0 + i) * p.m_total + mrow] = v;
            }
            continue;
          }
          if (!p.transpose_f32) {
            float4* dst = reinterpret_cast<float4*>(base + (long long)mrow * p.n_total + col0);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              dst[i] = has_k ? make_float4(__uint_as_float(raw[4 * i]),
                                           __uint_as_float(raw[4 * i + 1]),
                                           __uint_as_float(raw[4 * i + 2]),
                                           __uint_as_float(raw[4 * i + 3]))
                             : make_float4(0.f, 0.f, 0.f, 0.f);
          } else {
#pragma unroll
            for (int i = 0; i < 16; ++i)
              base[(long long)(col0 + i) * p.m_total + mrow] =
                  has_k ? __uint_as_float(raw[i]) : 0.f;
          }
        }
      }
      release_acc(acc);
    }
  }

  if constexpr (PAIR) {
    tc::tc_fence_before();
    tc::cluster_sync();  // both CTAs are done with the pair's TMEM and smem
    tc::tc_fence_after();
    if (warp == 1) tc::tmem_dealloc_cg2<C::TMEM_COLS>(tmem_base);
  } else {
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
}

}  // namespace gemm
}  // namespace tsm
