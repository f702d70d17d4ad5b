// vidperf::gpu::Network over the tsm_b200 C ABI (see vidperf_gpu_network.hpp).
#include "vidperf_gpu_network.hpp"

#include <stdexcept>
#include <string>

#include "tsm_b200.h"
#include "vidperf/errors.hpp"

namespace vidperf {
namespace gpu {

namespace {

void check(tsm_status st, const char* what) {
  if (st == TSM_OK) return;
  const std::string msg = std::string(what) + ": " + tsm_last_error();
  if (st == TSM_ERR_INVALID) throw ValidationError(msg);
  throw std::runtime_error("tsm_b200: " + msg);
}

// The residual units' shift fraction (every unit of these presets shares it).
Rational unit_shift(const ArchSpec& a) {
  for (const StageSpec& st : a.stages)
    for (const LayerSpec& l : st.layers)
      if (l.kind == LayerKind::ResBlockBottleneck) return l.shift_fraction;
  return Rational{0, 1};
}

// `preset` re-targeted to a's input shape and class count; equal to `a` iff
// `a` is that preset up to those free parameters.
ArchSpec retarget(ArchSpec preset, const ArchSpec& a) {
  preset.name = a.name;
  preset.input_shape = a.input_shape;
  preset.num_classes = a.num_classes;
  if (!preset.stages.empty()) {
    StageSpec& last = preset.stages.back();
    if (last.layers.size() == 1 && last.layers[0].kind == LayerKind::FullyConnected)
      last.layers[0].channels_out = a.num_classes;
  }
  return preset;
}

// ArchSpec -> tsm_net_desc (arch.cpp:140-161 build_tsm8f, 220-233
// build_micro_tsm); false for anything else.
bool map_arch(const ArchSpec& a, std::int64_t batch, tsm_net_desc* d) {
  const Rational fr = unit_shift(a);
  *d = tsm_net_desc{};
  d->batch = batch;
  d->frames = a.input_shape.t;
  d->height = a.input_shape.h;
  d->width = a.input_shape.w;
  d->classes = a.num_classes;
  d->shift_num = fr.num;
  d->shift_den = fr.num == 0 ? 1 : fr.den;
  try {
    if (a.input_shape.c == 3 && retarget(build_tsm8f(fr), a) == a) {
      d->arch = TSM_ARCH_TSM8F;
      return true;
    }
    if (a.input_shape.c == 8 && retarget(build_micro_tsm(fr), a) == a) {
      d->arch = TSM_ARCH_MICRO_TSM;
      return true;
    }
  } catch (const ValidationError&) {
  }
  return false;
}

}  // namespace

bool Network::supports(const ArchSpec& arch) {
  tsm_net_desc d;
  return map_arch(arch, 1, &d);
}

Network::Network(ArchSpec arch, std::uint64_t seed) : arch_(std::move(arch)) {
  tsm_net_desc d;
  if (!map_arch(arch_, 1, &d))
    throw ValidationError("architecture '" + arch_.name +
                          "' is not a TSM-ResNet-50 / micro-tsm network (the B200 executor "
                          "runs the residual-shift bottleneck path only)");
  // The reference's own constructor draws the parameters (validation, init
  // order and distributions of net.cpp:39-76 and 14-31), so param_vector()
  // is the reference's bit for bit.
  flat_ = vidperf::Network(arch_, seed).param_vector();
}

Network::Network(ArchSpec arch, std::vector<double> params) : arch_(std::move(arch)) {
  tsm_net_desc d;
  if (!map_arch(arch_, 1, &d))
    throw ValidationError("architecture '" + arch_.name +
                          "' is not a TSM-ResNet-50 / micro-tsm network");
  flat_ = std::move(params);
}

Network::~Network() {
  for (auto& kv : nets_) tsm_net_destroy(kv.second.net);
}

void Network::set_params(const std::vector<double>& v) {
  if (static_cast<std::int64_t>(v.size()) != param_count())
    throw ValidationError("expected " + std::to_string(param_count()) + " parameters, got " +
                          std::to_string(v.size()));
  flat_ = v;
  ++version_;
}

void Network::check_input(const Tensor5D& x) const {
  // net.cpp:128-135: the batch is free, the rest must match the architecture
  const Shape5D& want = arch_.input_shape;
  const Shape5D& got = x.shape();
  if (got.t != want.t || got.c != want.c || got.h != want.h || got.w != want.w)
    throw ValidationError("input t=" + std::to_string(got.t) + " c=" + std::to_string(got.c) +
                          " h=" + std::to_string(got.h) + " w=" + std::to_string(got.w) +
                          " does not match the architecture");
}

tsm_net* Network::bind(std::int64_t batch) const {
  Bound& b = nets_[batch];
  if (!b.net) {
    tsm_net_desc d;
    map_arch(arch_, batch, &d);
    check(tsm_net_create(&d, &b.net), "tsm_net_create");
  }
  if (b.uploaded != version_) {
    check(tsm_net_set_params_reference(b.net, flat_.data(), param_count()),
          "tsm_net_set_params_reference");
    b.uploaded = version_;
  }
  return b.net;
}

Tensor5D Network::forward(const Tensor5D& x) const {
  check_input(x);
  const Shape5D& s = x.shape();
  tsm_net* net = bind(s.n);
  Tensor5D y(Shape5D{s.n, 1, arch_.num_classes, 1, 1});
  check(tsm_net_forward_host(net, x.data().data(), y.data().data()), "tsm_net_forward_host");
  return y;
}

double Network::loss(const Tensor5D& x) const {
  const Tensor5D y = forward(x);
  double acc = 0.0;
  for (double v : y.data()) acc += v * v;  // net.cpp:141-146
  return acc;
}

Network::Gradients Network::loss_gradients(const Tensor5D& x) const {
  check_input(x);
  tsm_net* net = bind(x.shape().n);
  Gradients g;
  g.params.assign(flat_.size(), 0.0);
  g.input = Tensor5D(x.shape());
  check(tsm_net_loss_gradients_host(net, x.data().data(), &g.loss, g.params.data(),
                                    g.input.data().data()),
        "tsm_net_loss_gradients_host");
  return g;
}

}  // namespace gpu
}  // namespace vidperf
