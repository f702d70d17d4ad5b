// tcgen05 GEMM instantiations (see gemm_launch.cuh): single-CTA weight
// gradients staging 128 pixel rows per box and stage (BKT = 128) — the
// swapped c_out = 64 GEMMs and the non-pair N tiles.
#include "gemm_launch.cuh"

namespace tsm {
namespace gemm_host {

tsm_status dispatch_wgrad_bk128(int bn, int kcb, const Maps& m, const Params& p, cudaStream_t s) {
  if (kcb == 64) {
    if (bn == 64) return launch_gemm<64, 64, 64, true, true, 1, 128>(m, p, s);
    if (bn == 128) return launch_gemm<128, 64, 64, true, true, 1, 128>(m, p, s);
    if (bn == 256) return launch_gemm<256, 64, 64, true, true, 1, 128>(m, p, s);
  }
  if (kcb == 32 && bn == 256) return launch_gemm<256, 64, 32, true, true, 1, 128>(m, p, s);
  return fail(TSM_ERR_UNSUPPORTED, "no 128-row wgrad GEMM for BN=" + std::to_string(bn) +
                                       " KC=" + std::to_string(kcb));
}

tsm_status dispatch_wgrad_swapped_bk128(int kca, const Maps& m, const Params& p, cudaStream_t s) {
  if (kca == 64) return dispatch_wgrad_bk128(64, 64, m, p, s);  // the same instantiation
  if (kca == 32) return launch_gemm<64, 32, 64, true, true, 1, 128>(m, p, s);
  return fail(TSM_ERR_UNSUPPORTED, "no 128-row swapped wgrad GEMM for KC=" + std::to_string(kca));
}

bool wgrad_bk128_ok(bool swap, int bn, int kcx) {
  if (swap) return kcx == 64 || kcx == 32;
  return (kcx == 64 && (bn == 64 || bn == 128 || bn == 256)) || (kcx == 32 && bn == 256);
}

}  // namespace gemm_host
}  // namespace tsm
