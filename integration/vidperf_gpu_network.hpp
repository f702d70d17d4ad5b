// vidperf::gpu::Network — the reference's Network executor (net.hpp:15-54)
// with every layer on the B200 (libtsm_b200, C ABI tsm_net_*).
//
// Same public surface, argument meaning and error behaviour as
// vidperf::Network, compiled against the reference's own headers:
//
//   Network(ArchSpec, seed)        net.hpp:17  (parameters initialised by the
//                                  reference's own constructor, net.cpp:39-76,
//                                  so param_vector() is identical)
//   arch / param_count / get_param / set_param / param_vector   net.hpp:19-24
//   forward(const Tensor5D&)       net.hpp:26  -> (N, 1, classes, 1, 1)
//   loss(const Tensor5D&)          net.hpp:30  (Sigma y^2)
//   loss_gradients(const Tensor5D&) net.hpp:37 -> Gradients{loss, params in
//                                  declaration order and reference layout,
//                                  dL/dx}
//
// Architectures: the TSM-ResNet-50 family (build_tsm8f with any shift
// fraction, frame count, spatial extent and class count) and build_micro_tsm
// — the residual-shift bottleneck path this library implements.  Any other
// ArchSpec throws ValidationError.  Arithmetic is bf16 with fp32
// accumulation (activations and weights rounded to bf16 on the device), so
// results match the fp64 reference within the tolerances of
// tests/test_network_gpu.py, not bitwise.  Errors: invalid input shapes /
// architectures -> ValidationError (errors.hpp:11-13); CUDA or NCCL failures
// -> std::runtime_error (the CLI maps them to exit 1 / 2, vidperf.cpp:475-485).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <vector>

#include "vidperf/arch.hpp"
#include "vidperf/net.hpp"
#include "vidperf/tensor.hpp"

struct tsm_net;

namespace vidperf {
namespace gpu {

class Network {
 public:
  using Gradients = vidperf::Network::Gradients;

  Network(ArchSpec arch, std::uint64_t seed);
  // The same executor over given parameters (param_vector() order/layout of
  // a reference Network of this architecture).
  Network(ArchSpec arch, std::vector<double> params);
  ~Network();
  Network(const Network&) = delete;
  Network& operator=(const Network&) = delete;

  const ArchSpec& arch() const { return arch_; }
  std::int64_t param_count() const { return static_cast<std::int64_t>(flat_.size()); }
  double get_param(std::int64_t i) const { return flat_[i]; }
  void set_param(std::int64_t i, double v) {
    flat_[i] = v;
    ++version_;
  }
  std::vector<double> param_vector() const { return flat_; }
  // Replace every parameter at once (same order as param_vector()).
  void set_params(const std::vector<double>& v);

  Tensor5D forward(const Tensor5D& x) const;
  double loss(const Tensor5D& x) const;
  Gradients loss_gradients(const Tensor5D& x) const;

  // True when `arch` is one this executor runs (TSM-R50 family, micro-tsm).
  static bool supports(const ArchSpec& arch);

 private:
  struct Bound {  // one device network per batch size
    tsm_net* net = nullptr;
    std::uint64_t uploaded = ~0ull;  // parameter version on the device
  };
  tsm_net* bind(std::int64_t batch) const;
  void check_input(const Tensor5D& x) const;

  ArchSpec arch_;
  std::vector<double> flat_;
  std::uint64_t version_ = 0;
  mutable std::map<std::int64_t, Bound> nets_;
};

}  // namespace gpu
}  // namespace vidperf
