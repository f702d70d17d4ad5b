// tcgen05 GEMM instantiations (see gemm_launch.cuh), one group per file so
// the kernel templates compile in parallel.
#include "gemm_launch.cuh"

namespace tsm {
namespace gemm_host {

tsm_status dispatch_fwd_kc64(int bn, const Maps& m, const Params& p, cudaStream_t s) {
  if (bn == 64) return launch_gemm<64, 64, 64, false, false>(m, p, s);
  if (bn == 128) return launch_gemm<128, 64, 64, false, false>(m, p, s);
  if (bn == 256) return launch_gemm<256, 64, 64, false, false>(m, p, s);
  return fail(TSM_ERR_UNSUPPORTED, "no tcgen05 GEMM instance for BN=" + std::to_string(bn));
}

// CTA pair (cta_group::2), 256 x BN tiles
tsm_status dispatch_fwd_pair(int bn, const Maps& m, const Params& p, cudaStream_t s) {
  if (bn == 128) return launch_gemm<128, 64, 64, false, false, 2>(m, p, s);
  return launch_gemm<256, 64, 64, false, false, 2>(m, p, s);
}

}  // namespace gemm_host
}  // namespace tsm
