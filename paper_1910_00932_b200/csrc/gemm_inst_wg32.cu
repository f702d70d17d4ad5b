// tcgen05 GEMM instantiations (see gemm_launch.cuh), one group per file so
// the kernel templates compile in parallel.
#include "gemm_launch.cuh"

namespace tsm {
namespace gemm_host {

tsm_status dispatch_wgrad_kc32(int bn, const Maps& m, const Params& p, cudaStream_t s) {
  if (bn == 64) return launch_gemm<64, 64, 32, true, true>(m, p, s);
  if (bn == 128) return launch_gemm<128, 64, 32, true, true>(m, p, s);
  if (bn == 256) return launch_gemm<256, 64, 32, true, true>(m, p, s);
  return fail(TSM_ERR_UNSUPPORTED, "no tcgen05 GEMM instance for BN=" + std::to_string(bn));
}

// swapped weight gradient (c_out < 128): M = the X side
tsm_status dispatch_wgrad_swapped(int kca, const Maps& m, const Params& p, cudaStream_t s) {
  if (kca == 64) return dispatch_wgrad_kc64(64, m, p, s);  // the same instantiation
  if (kca == 32) return launch_gemm<64, 32, 64, true, true>(m, p, s);
  if (kca == 8) return launch_gemm<64, 8, 64, true, true>(m, p, s);
  if (kca == 16) return launch_gemm<64, 16, 64, true, true>(m, p, s);
  return fail(TSM_ERR_UNSUPPORTED, "no swapped wgrad GEMM for KC=" + std::to_string(kca));
}

}  // namespace gemm_host
}  // namespace tsm
