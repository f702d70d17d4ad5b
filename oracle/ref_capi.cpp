// TEST INFRASTRUCTURE ONLY — never linked into the product path.
//
// A thin extern "C" shim over the *unmodified* reference library (vidperf),
// compiled in place from /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libvidperf_ref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load it.
//
// Every function converts plain pointers into vidperf::Tensor5D and calls the
// reference symbol named in its comment.  Exceptions never cross the ABI: a
// vidperf::ValidationError returns 1, anything else returns 2 (the CLI's exit
// code mapping, tools/vidperf.cpp:475-485).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "vidperf/arch.hpp"
#include "vidperf/kernels.hpp"
#include "vidperf/net.hpp"
#include "vidperf/ref_kernels.hpp"
#include "vidperf/sim.hpp"
#include "vidperf/tensor.hpp"

using namespace vidperf;

namespace {

thread_local std::string g_last_error;

Shape5D shape_of(const int64_t* s) { return Shape5D{s[0], s[1], s[2], s[3], s[4]}; }

Tensor5D wrap(const double* p, const int64_t* s) {
  Shape5D sh = shape_of(s);
  return Tensor5D::from_data(sh, std::vector<double>(p, p + sh.elems()));
}

void unwrap(const Tensor5D& t, double* out) {
  std::memcpy(out, t.data().data(), sizeof(double) * static_cast<size_t>(t.size()));
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ValidationError& e) {
    g_last_error = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return 2;
  }
}

ShiftConfig cfg_of(int64_t fn, int64_t fd, int64_t bn, int64_t bd) {
  return ShiftConfig{Rational{fn, fd}, Rational{bn, bd}};
}

ConvWeights conv_of(int64_t c_out, int64_t c_in, const int* k, const double* w, const double* b) {
  ConvWeights cw = ConvWeights::zeros(c_out, c_in, {k[0], k[1], k[2]});
  std::memcpy(cw.w.data(), w, sizeof(double) * cw.w.size());
  std::memcpy(cw.bias.data(), b, sizeof(double) * cw.bias.size());
  return cw;
}

ConvGeometry geom_of(const int* k, const int* s, const int* p) {
  return ConvGeometry{{k[0], k[1], k[2]}, {s[0], s[1], s[2]}, {p[0], p[1], p[2]}};
}

}  // namespace

extern "C" {

const char* vref_last_error() { return g_last_error.c_str(); }

// tensor.cpp:41-47
int vref_random_normal(const int64_t* shape, uint64_t seed, double stddev, double* out) {
  return guard([&] { unwrap(random_normal(shape_of(shape), seed, stddev), out); });
}

// tensor.cpp:49-55
int vref_random_uniform(const int64_t* shape, uint64_t seed, double lo, double hi, double* out) {
  return guard([&] { unwrap(random_uniform(shape_of(shape), seed, lo, hi), out); });
}

// kernels.cpp:82-95
int vref_validate_shift(int64_t fn, int64_t fd, int64_t bn, int64_t bd, int64_t channels) {
  return guard([&] { validate_shift(cfg_of(fn, fd, bn, bd), channels); });
}

// kernels.cpp:97-125 (serial=0) or ref_kernels.cpp:142-157 (serial=1)
int vref_temporal_shift(const double* x, const int64_t* shape, int64_t fn, int64_t fd, int64_t bn,
                        int64_t bd, int serial, double* out) {
  return guard([&] {
    Tensor5D t = wrap(x, shape);
    ShiftConfig c = cfg_of(fn, fd, bn, bd);
    unwrap(serial ? ref::temporal_shift(t, c) : temporal_shift(t, c), out);
  });
}

// kernels.cpp:127-157
int vref_temporal_shift_adjoint(const double* y, const int64_t* shape, int64_t fn, int64_t fd,
                                int64_t bn, int64_t bd, double* out) {
  return guard([&] { unwrap(temporal_shift_adjoint(wrap(y, shape), cfg_of(fn, fd, bn, bd)), out); });
}

// Timing helper for the CPU baseline: run the reference shift `iters` times on
// a tensor it owns (no marshalling inside the loop).  Returns seconds per call.
double vref_time_shift(const int64_t* shape, uint64_t seed, int64_t fold_div, int adjoint,
                       int serial, int iters) {
  double secs = -1.0;
  guard([&] {
    Tensor5D x = random_normal(shape_of(shape), seed);
    ShiftConfig c = ShiftConfig::symmetric(Rational{1, fold_div});
    auto run = [&] {
      if (adjoint) return temporal_shift_adjoint(x, c);
      return serial ? ref::temporal_shift(x, c) : temporal_shift(x, c);
    };
    Tensor5D warm = run();
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < iters; ++i) warm = run();
    secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / iters;
  });
  return secs;
}

// kernels.cpp:162-231 (serial=0) or ref_kernels.cpp:26-64 (serial=1)
int vref_conv_forward(const double* x, const int64_t* shape, int64_t c_out, const int* k,
                      const int* s, const int* p, const double* w, const double* b, int serial,
                      double* out, int64_t* out_shape) {
  return guard([&] {
    Tensor5D t = wrap(x, shape);
    ConvWeights cw = conv_of(c_out, shape[2], k, w, b);
    ConvGeometry g = geom_of(k, s, p);
    Tensor5D y = serial ? ref::conv_forward(t, cw, g) : conv_forward(t, cw, g);
    const Shape5D& os = y.shape();
    int64_t o[5] = {os.n, os.t, os.c, os.h, os.w};
    std::memcpy(out_shape, o, sizeof o);
    if (out) unwrap(y, out);
  });
}

// kernels.cpp:233-327
int vref_conv_backward(const double* x, const int64_t* shape, int64_t c_out, const int* k,
                       const int* s, const int* p, const double* w, const double* b,
                       const double* gy, double* gx, double* gw, double* gb) {
  return guard([&] {
    Tensor5D t = wrap(x, shape);
    ConvWeights cw = conv_of(c_out, shape[2], k, w, b);
    ConvGeometry g = geom_of(k, s, p);
    Shape5D os = conv_forward(t, cw, g).shape();
    int64_t o[5] = {os.n, os.t, os.c, os.h, os.w};
    ConvGrads cg = conv_backward(t, cw, g, wrap(gy, o));
    unwrap(cg.grad_x, gx);
    std::memcpy(gw, cg.grad_w.w.data(), sizeof(double) * cg.grad_w.w.size());
    std::memcpy(gb, cg.grad_w.bias.data(), sizeof(double) * cg.grad_w.bias.size());
  });
}

// kernels.cpp:353-390 / 392-455
int vref_max_pool(const double* x, const int64_t* shape, const int* k, const int* s, const int* p,
                  const double* gy, double* out, double* gx, int64_t* out_shape) {
  return guard([&] {
    Tensor5D t = wrap(x, shape);
    ConvGeometry g = geom_of(k, s, p);
    Tensor5D y = max_pool_forward(t, g);
    const Shape5D& os = y.shape();
    int64_t o[5] = {os.n, os.t, os.c, os.h, os.w};
    std::memcpy(out_shape, o, sizeof o);
    if (out) unwrap(y, out);
    if (gy && gx) unwrap(max_pool_backward(t, g, wrap(gy, o)), gx);
  });
}

// ---------------------------------------------------------------------------
// One residual-shift bottleneck unit, forward and backward, composed from the
// reference kernels in exactly the order Network::run_unit (net.cpp:85-126)
// and Network::loss_gradients (net.cpp:184-248) apply them to a unit produced
// by expand_layer (arch.cpp:278-323).  The reference has no standalone block
// function; this is that unit with the upstream gradient `gy`
// supplied by the caller instead of 2*y.
//
// w = {w1,b1,w2,b2,w3,b3,wp,bp}; wp/bp are null when there is no projection.
// Gradients come back in the same slots.  gy == null -> forward only.
int vref_block(const double* x, const int64_t* shape, int64_t c_out, int stride,
               int64_t shift_num, int64_t shift_den, const double* const* w, double* y,
               int64_t* y_shape, const double* gy, double* gx, double* const* gw) {
  return guard([&] {
    LayerSpec spec;
    spec.kind = LayerKind::ResBlockBottleneck;
    spec.kernel = {1, 3, 3};
    spec.stride = {1, stride, stride};
    spec.padding = {0, 1, 1};
    spec.channels_out = c_out;
    spec.shift_fraction = Rational{shift_num, shift_den};
    ResidualUnit ru = expand_layer(spec, shape[2]);
    Tensor5D in = wrap(x, shape);

    std::vector<ConvWeights> convs;
    std::vector<ConvGeometry> geoms;
    int64_t cin = shape[2];
    int slot = 0;
    for (const PrimOp& op : ru.main) {
      if (op.kind == LayerKind::TemporalShift) continue;
      convs.push_back(conv_of(op.channels_out, cin, op.kernel.data(), w[2 * slot], w[2 * slot + 1]));
      geoms.push_back(ConvGeometry{op.kernel, op.stride, op.padding});
      cin = op.channels_out;
      ++slot;
    }
    bool has_proj = ru.projection.has_value();
    if (has_proj != (w[6] != nullptr)) throw ValidationError("projection weights mismatch");
    std::optional<ConvWeights> proj;
    if (has_proj) proj = conv_of(c_out, shape[2], ru.projection->kernel.data(), w[6], w[7]);

    // Forward with a tape, as run_unit does.
    std::vector<Tensor5D> tape;
    Tensor5D cur = in;
    int ci = 0;
    for (const PrimOp& op : ru.main) {
      tape.push_back(cur);
      Tensor5D next;
      if (op.kind == LayerKind::TemporalShift) {
        next = temporal_shift(cur, ShiftConfig::symmetric(op.shift_fraction));
      } else {
        next = conv_forward(cur, convs[ci], geoms[ci]);
        ++ci;
      }
      if (op.relu_after) {
        tape.push_back(next);
        next = relu_forward(next);
      }
      cur = std::move(next);
    }
    Tensor5D skip = proj ? conv_forward(in, *proj, ConvGeometry{ru.projection->kernel,
                                                                ru.projection->stride,
                                                                ru.projection->padding})
                         : in;
    Tensor5D pre = add(cur, skip);
    Tensor5D out = relu_forward(pre);
    const Shape5D& os = out.shape();
    int64_t o[5] = {os.n, os.t, os.c, os.h, os.w};
    std::memcpy(y_shape, o, sizeof o);
    if (y) unwrap(out, y);
    if (!gy) return;

    // Reverse sweep, as loss_gradients does for one unit.
    Tensor5D g = relu_backward(pre, wrap(gy, o));
    Tensor5D skip_grad = g;
    ci = static_cast<int>(convs.size());
    for (size_t i = ru.main.size(); i-- > 0;) {
      const PrimOp& op = ru.main[i];
      if (op.relu_after) {
        Tensor5D p = std::move(tape.back());
        tape.pop_back();
        g = relu_backward(p, g);
      }
      Tensor5D xin = std::move(tape.back());
      tape.pop_back();
      if (op.kind == LayerKind::TemporalShift) {
        g = temporal_shift_adjoint(g, ShiftConfig::symmetric(op.shift_fraction));
      } else {
        --ci;
        ConvGrads cg = conv_backward(xin, convs[ci], geoms[ci], g);
        std::memcpy(gw[2 * ci], cg.grad_w.w.data(), sizeof(double) * cg.grad_w.w.size());
        std::memcpy(gw[2 * ci + 1], cg.grad_w.bias.data(), sizeof(double) * cg.grad_w.bias.size());
        g = std::move(cg.grad_x);
      }
    }
    if (proj) {
      ConvGrads pg = conv_backward(in, *proj, ConvGeometry{ru.projection->kernel,
                                                           ru.projection->stride,
                                                           ru.projection->padding},
                                   skip_grad);
      std::memcpy(gw[6], pg.grad_w.w.data(), sizeof(double) * pg.grad_w.w.size());
      std::memcpy(gw[7], pg.grad_w.bias.data(), sizeof(double) * pg.grad_w.bias.size());
      g = add(g, pg.grad_x);
    } else {
      g = add(g, skip_grad);
    }
    unwrap(g, gx);
  });
}

// ---------------------------------------------------------------------------
// Network (net.cpp).  Handles are heap Network objects.

void* vref_net_create(const char* preset, int64_t shift_num, int64_t shift_den, uint64_t seed) {
  Network* net = nullptr;
  guard([&] {
    std::string p = preset;
    ArchSpec a;
    if (p == "tsm8f") a = build_tsm8f(Rational{shift_num, shift_den});
    else if (p == "micro-tsm") a = build_micro_tsm(Rational{shift_num, shift_den});
    else a = build_preset(p);
    net = new Network(a, seed);
  });
  return net;
}

// build_tsm8f (arch.cpp:140-161) with the clip's spatial extent changed to
// h x w (a bounded CPU-baseline sample; validate() checks it still
// propagates).  Everything else, including init order, is the reference's.
void* vref_net_create_sized(int64_t h, int64_t w, uint64_t seed) {
  Network* net = nullptr;
  guard([&] {
    ArchSpec a = build_tsm8f();
    a.input_shape.h = h;
    a.input_shape.w = w;
    net = new Network(a, seed);
  });
  return net;
}

// Seconds for one Network::loss_gradients (net.cpp:160-272) on `clips`
// clips of random_normal input (seed 43), averaged over `iters`.
double vref_time_loss_gradients(void* h, int64_t clips, int iters) {
  double secs = -1.0;
  guard([&] {
    Network* net = static_cast<Network*>(h);
    Shape5D s = net->arch().input_shape;
    s.n = clips;
    Tensor5D x = random_normal(s, 43);
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < iters; ++i) (void)net->loss_gradients(x);
    secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / iters;
  });
  return secs;
}

void vref_net_destroy(void* h) { delete static_cast<Network*>(h); }

int64_t vref_net_param_count(void* h) { return static_cast<Network*>(h)->param_count(); }

void vref_net_get_params(void* h, double* out) {
  auto v = static_cast<Network*>(h)->param_vector();
  std::memcpy(out, v.data(), sizeof(double) * v.size());
}

void vref_net_set_params(void* h, const double* in) {
  Network* n = static_cast<Network*>(h);
  for (int64_t i = 0; i < n->param_count(); ++i) n->set_param(i, in[i]);
}

// net.cpp:128-139
int vref_net_forward(void* h, const double* x, const int64_t* shape, double* out,
                     int64_t* out_shape) {
  return guard([&] {
    Tensor5D y = static_cast<Network*>(h)->forward(wrap(x, shape));
    const Shape5D& os = y.shape();
    int64_t o[5] = {os.n, os.t, os.c, os.h, os.w};
    std::memcpy(out_shape, o, sizeof o);
    if (out) unwrap(y, out);
  });
}

// net.cpp:160-272
int vref_net_loss_gradients(void* h, const double* x, const int64_t* shape, double* loss,
                            double* grad_params, double* grad_input) {
  return guard([&] {
    Network::Gradients g = static_cast<Network*>(h)->loss_gradients(wrap(x, shape));
    *loss = g.loss;
    std::memcpy(grad_params, g.params.data(), sizeof(double) * g.params.size());
    if (grad_input) unwrap(g.input, grad_input);
  });
}

// net.cpp:274-325
int vref_gradcheck(const char* preset, int64_t shift_num, int64_t shift_den, const double* x,
                   const int64_t* shape, double eps, uint64_t seed, double* max_rel,
                   int64_t* checked) {
  return guard([&] {
    std::string p = preset;
    ArchSpec a = p == "micro-tsm" ? build_micro_tsm(Rational{shift_num, shift_den})
                                  : build_preset(p);
    GradcheckResult r = gradcheck(a, wrap(x, shape), eps, seed);
    *max_rel = r.max_rel_error;
    *checked = r.checked_scalars;
  });
}

// write_tensor / read_tensor (tensor.cpp:78-110): the fixture format.
int vref_write_tensor(const double* x, const int64_t* shape, const char* path) {
  return guard([&] { write_tensor(wrap(x, shape), path); });
}

// read_tensor: shape_out[5] always; data copied when `out` is non-null.
int vref_read_tensor(const char* path, int64_t* shape_out, double* out) {
  return guard([&] {
    Tensor5D t = read_tensor(path);
    const Shape5D& s = t.shape();
    shape_out[0] = s.n; shape_out[1] = s.t; shape_out[2] = s.c; shape_out[3] = s.h; shape_out[4] = s.w;
    if (out) unwrap(t, out);
  });
}

// step_time (sim.cpp:132-144) on a CostReport carrying only the fields it
// reads.  prof = {nodes, gpus_per_node, peak_flops_per_gpu, utilization,
// disk_bandwidth_per_node, net_latency, net_bandwidth, bytes_per_param};
// out = {t_compute, t_io, t_comm, t_step}.
int vref_step_time(const double* prof, int64_t flops, int64_t params, int64_t input_bytes,
                   int per_gpu_batch, double flop_mult, int ring, double* out) {
  return guard([&] {
    ClusterProfile p;
    p.nodes = static_cast<int64_t>(prof[0]);
    p.gpus_per_node = static_cast<int>(prof[1]);
    p.peak_flops_per_gpu = prof[2];
    p.utilization = prof[3];
    p.disk_bandwidth_per_node = prof[4];
    p.net_latency = prof[5];
    p.net_bandwidth = prof[6];
    p.bytes_per_param = prof[7];
    CostReport c;
    c.total_flops = flops;
    c.total_params = params;
    c.input_bytes = input_bytes;
    TrainConfig cfg;
    cfg.per_gpu_batch = per_gpu_batch;
    cfg.train_flop_multiplier = flop_mult;
    StepTime st = step_time(c, p, cfg, ring ? CommMode::Ring : CommMode::Simple);
    out[0] = st.t_compute;
    out[1] = st.t_io;
    out[2] = st.t_comm;
    out[3] = st.t_step;
  });
}

// observed_scalability (sim.cpp:195-215).
int vref_observed_scalability(const int64_t* nodes, const double* seconds, int n, double* out) {
  return guard([&] {
    std::vector<std::pair<std::int64_t, double>> t;
    for (int i = 0; i < n; ++i) t.emplace_back(nodes[i], seconds[i]);
    auto r = observed_scalability(t);
    for (int i = 0; i < n; ++i) out[i] = r[i].second;
  });
}

}  // extern "C"
