// Drop-in replacement for the temporal-shift section of the reference
// library (vidperf, kernels.cpp:79-157) on top of the tsm_b200 C ABI.
//
// Compiled against the reference's OWN headers (include/vidperf/*.hpp) so the
// three functions below have exactly the reference signatures and types:
//
//   void     vidperf::validate_shift(const ShiftConfig&, int64_t)    kernels.hpp:22
//   Tensor5D vidperf::temporal_shift(const Tensor5D&, const ShiftConfig&)          :24
//   Tensor5D vidperf::temporal_shift_adjoint(const Tensor5D&, const ShiftConfig&)  :26
//
// A maintainer either links this object instead of kernels.cpp's shift
// section, or loads libvidperf_gpu_shim.so ahead of the reference library
// (LD_PRELOAD / RTLD_GLOBAL) so that every caller — Network::run_unit
// (net.cpp:97-99), loss_gradients (net.cpp:217-219), the CLI shift-demo
// (vidperf.cpp:316-318) — resolves to the GPU path.  Value semantics, error
// behaviour and results are the reference's: a new Tensor5D is returned
// (kernels.cpp:102, 134), bad splits throw vidperf::ValidationError with the
// reference's message shape, CUDA failures throw std::runtime_error (the CLI
// maps those to exit 2, tools/vidperf.cpp:475-485), and the output is bitwise
// identical (fp64 moved as bytes; the boundary is +0.0).
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "tsm_b200.h"
#include "vidperf/errors.hpp"
#include "vidperf/kernels.hpp"
#include "vidperf/rational.hpp"
#include "vidperf/tensor.hpp"

namespace vidperf {

namespace {

void split_or_throw(const ShiftConfig& cfg, std::int64_t channels, std::int64_t* f,
                    std::int64_t* b) {
  const tsm_status st =
      tsm_validate_shift(cfg.fraction_fwd.num, cfg.fraction_fwd.den, cfg.fraction_bwd.num,
                         cfg.fraction_bwd.den, channels, f, b);
  if (st == TSM_ERR_INVALID) throw ValidationError(tsm_last_error());
  if (st != TSM_OK) throw std::runtime_error(tsm_last_error());
}

Tensor5D shift_on_gpu(const Tensor5D& x, const ShiftConfig& cfg, int adjoint) {
  const Shape5D& s = x.shape();
  std::int64_t f = 0, b = 0;
  split_or_throw(cfg, s.c, &f, &b);
  Tensor5D out(s);  // same construction (and shape checks) as the reference
  const tsm_status st = tsm_shift_host(x.data().data(), out.data().data(), s.n, s.t, s.c, s.h,
                                       s.w, f, b, TSM_F64, adjoint);
  if (st == TSM_ERR_INVALID) throw ValidationError(tsm_last_error());
  if (st != TSM_OK) throw std::runtime_error(std::string("tsm_b200: ") + tsm_last_error());
  return out;
}

}  // namespace

void validate_shift(const ShiftConfig& cfg, std::int64_t channels) {
  std::int64_t f = 0, b = 0;
  split_or_throw(cfg, channels, &f, &b);
}

Tensor5D temporal_shift(const Tensor5D& x, const ShiftConfig& cfg) {
  return shift_on_gpu(x, cfg, 0);
}

Tensor5D temporal_shift_adjoint(const Tensor5D& y, const ShiftConfig& cfg) {
  return shift_on_gpu(y, cfg, 1);
}

}  // namespace vidperf
