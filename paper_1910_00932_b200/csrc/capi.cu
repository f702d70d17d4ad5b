// extern "C" entry points of libtsm_b200.so (declared in include/tsm_b200.h).
#include <cuda_runtime.h>

#include <atomic>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "aux_kernels.cuh"
#include "head_kernels.cuh"
#include "block.h"
#include "conv_ops.h"
#include "network.h"
#include "src_hash.h"

namespace tsm {

std::string& last_error() {
  thread_local std::string msg;
  return msg;
}

static std::atomic<uint64_t> g_launches{0};

namespace {
struct Trace {
  bool on = false;
  std::string label;
  std::vector<std::string> lines;
};
thread_local Trace g_trace;
}  // namespace

bool trace_on() { return g_trace.on; }

TraceScope::TraceScope(const std::string& label) {
  if (!g_trace.on) return;
  saved = g_trace.label;
  g_trace.label = saved.empty() ? label : saved + " " + label;
}

TraceScope::~TraceScope() {
  if (g_trace.on) g_trace.label = saved;
}

void count_launches(uint64_t n) {
  g_launches.fetch_add(n, std::memory_order_relaxed);
  if (g_trace.on && n < (1u << 20))
    for (uint64_t i = 0; i < n; ++i) g_trace.lines.push_back(g_trace.label);
}

// Event pairs around the fused shift + 1x1 conv launches (bench.py's
// in-step roofline).  Host-thread state: the step is issued from one thread.
namespace {
constexpr int kProbeMax = 256;
struct Conv1Probe {
  bool open = false;
  int n = 0;
  int64_t c_in = 0, c_out = 0, pixels = 0;  // c_in == 0: off
  cudaEvent_t ev[2 * kProbeMax] = {};
};
// Per host thread (the thread that issues the step), not process-global:
// concurrent callers on other threads neither record into nor reset it.
thread_local Conv1Probe g_probe;
}  // namespace

void probe_conv1_begin(cudaStream_t s, int64_t c_in, int64_t c_out, int64_t pixels) {
  if (!g_probe.c_in || c_in != g_probe.c_in || c_out != g_probe.c_out || g_probe.n >= kProbeMax)
    return;
  g_probe.pixels = pixels;
  cudaEventRecord(g_probe.ev[2 * g_probe.n], s);
  g_probe.open = true;
}

bool probe_enabled() { return g_probe.c_in != 0; }

void probe_conv1_end(cudaStream_t s) {
  if (!g_probe.open) return;
  cudaEventRecord(g_probe.ev[2 * g_probe.n + 1], s);
  g_probe.open = false;
  ++g_probe.n;
}

tsm_status require_device() {
  thread_local int checked_dev = -1;
  int dev = -1;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "no CUDA device (tsm_b200 has no CPU fallback)");
  if (dev == checked_dev) return TSM_OK;
  int major = 0;
  TSM_CUDA_TRY(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major != 10)
    return fail(TSM_ERR_CUDA, "tsm_b200 is built for sm_100a only (device major != 10)");
  checked_dev = dev;
  return TSM_OK;
}

tsm_status shift_launch(const void* x, void* y, int64_t n, int64_t t, int64_t c, int64_t h,
                        int64_t w, int64_t fold_fwd, int64_t fold_bwd, tsm_dtype dtype,
                        int adjoint, cudaStream_t stream);

}  // namespace tsm

using namespace tsm;

namespace {

int64_t gcd64(int64_t a, int64_t b) {
  if (a < 0) a = -a;
  while (b) {
    int64_t r = a % b;
    a = b;
    b = r;
  }
  return a;
}

// Rational{num, den} normalisation (rational.cpp:10-23).
tsm_status normalise(int64_t& num, int64_t& den) {
  if (den == 0) return fail(TSM_ERR_INVALID, "rational with zero denominator");
  if (den < 0) {
    num = -num;
    den = -den;
  }
  if (num == 0) {
    den = 1;
    return TSM_OK;
  }
  int64_t g = gcd64(num, den);
  num /= g;
  den /= g;
  return TSM_OK;
}

std::string frac(int64_t n, int64_t d) { return std::to_string(n) + "/" + std::to_string(d); }

// Per-thread growable device staging for the host-buffer entry point.
struct HostStage {
  void* dx = nullptr;
  void* dy = nullptr;
  size_t cap = 0;
  cudaStream_t stream = nullptr;
  ~HostStage() {
    if (dx) cudaFree(dx);
    if (dy) cudaFree(dy);
    if (stream) cudaStreamDestroy(stream);
  }
};

}  // namespace

extern "C" {

const char* tsm_last_error(void) { return last_error().c_str(); }

int tsm_abi_version(void) { return 3; }

const char* tsm_source_hash(void) { return TSM_SRC_HASH; }

uint64_t tsm_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

tsm_status tsm_trace_enable(int on) {
  g_trace.on = on != 0;
  g_trace.lines.clear();
  g_trace.label.clear();
  return TSM_OK;
}

tsm_status tsm_trace_dump(const char* path) {
  if (!path) return fail(TSM_ERR_INVALID, "tsm_trace_dump: null path");
  FILE* f = std::fopen(path, "w");
  if (!f) return fail(TSM_ERR_INVALID, std::string("tsm_trace_dump: cannot open ") + path);
  for (const auto& l : g_trace.lines) std::fprintf(f, "%s\n", l.empty() ? "-" : l.c_str());
  std::fclose(f);
  return TSM_OK;
}

tsm_status tsm_probe_shift_conv1(int64_t c_in, int64_t c_out) {
  if (c_in < 0 || c_out < 0) return fail(TSM_ERR_INVALID, "probe: negative channels");
  TSM_TRY(require_device());
  if (c_in) {
    for (auto& e : g_probe.ev)
      if (!e) TSM_CUDA_TRY(cudaEventCreate(&e));
    g_probe.n = 0;
    g_probe.open = false;
    g_probe.pixels = 0;
  }
  g_probe.c_in = c_in;
  g_probe.c_out = c_out;
  return TSM_OK;
}

tsm_status tsm_probe_shift_conv1_read(int* launches, double* mean_us, int64_t* pixels) {
  if (!launches || !mean_us) return fail(TSM_ERR_INVALID, "probe: null output");
  TSM_TRY(require_device());
  double sum = 0.0;
  for (int i = 0; i < g_probe.n; ++i) {
    TSM_CUDA_TRY(cudaEventSynchronize(g_probe.ev[2 * i + 1]));
    float ms = 0.f;
    TSM_CUDA_TRY(cudaEventElapsedTime(&ms, g_probe.ev[2 * i], g_probe.ev[2 * i + 1]));
    sum += ms * 1e3;
  }
  *launches = g_probe.n;
  *mean_us = g_probe.n ? sum / g_probe.n : 0.0;
  if (pixels) *pixels = g_probe.pixels;
  return TSM_OK;
}

// kernels.cpp:82-95 with rational.cpp:50-61.
tsm_status tsm_validate_shift(int64_t fn, int64_t fd, int64_t bn, int64_t bd, int64_t channels,
                              int64_t* fold_fwd, int64_t* fold_bwd) {
  TSM_TRY(normalise(fn, fd));
  TSM_TRY(normalise(bn, bd));
  for (auto [num, den] : {std::pair{fn, fd}, std::pair{bn, bd}}) {
    if (num < 0) return fail(TSM_ERR_INVALID, "shift fraction must be non-negative");
    if ((num * channels) % den != 0)
      return fail(TSM_ERR_INVALID, "shift fraction " + frac(num, den) +
                                       " does not split " + std::to_string(channels) +
                                       " channels evenly");
  }
  const int64_t f = fn * channels / fd, b = bn * channels / bd;
  if (f + b > channels)
    return fail(TSM_ERR_INVALID, "shift splits " + std::to_string(f) + "+" + std::to_string(b) +
                                     " exceed " + std::to_string(channels) + " channels");
  if (fold_fwd) *fold_fwd = f;
  if (fold_bwd) *fold_bwd = b;
  return TSM_OK;
}

tsm_status tsm_shift_fwd(const void* x, void* y, int64_t n, int64_t t, int64_t c, int64_t h,
                         int64_t w, int64_t fold_fwd, int64_t fold_bwd, tsm_dtype dtype,
                         void* stream) {
  return shift_launch(x, y, n, t, c, h, w, fold_fwd, fold_bwd, dtype, 0,
                      static_cast<cudaStream_t>(stream));
}

tsm_status tsm_shift_bwd(const void* dy, void* dx, int64_t n, int64_t t, int64_t c, int64_t h,
                         int64_t w, int64_t fold_fwd, int64_t fold_bwd, tsm_dtype dtype,
                         void* stream) {
  return shift_launch(dy, dx, n, t, c, h, w, fold_fwd, fold_bwd, dtype, 1,
                      static_cast<cudaStream_t>(stream));
}

tsm_status tsm_shift_host(const void* x, void* y, int64_t n, int64_t t, int64_t c, int64_t h,
                          int64_t w, int64_t fold_fwd, int64_t fold_bwd, tsm_dtype dtype,
                          int adjoint) {
  const int64_t elt = elt_size(dtype);
  if (elt == 0) return fail(TSM_ERR_UNSUPPORTED, "tsm_shift_host: unknown dtype");
  if (n <= 0 || t <= 0 || c <= 0 || h <= 0 || w <= 0)
    return fail(TSM_ERR_INVALID, "tsm_shift_host: non-positive tensor shape");
  TSM_TRY(require_device());
  thread_local HostStage st;
  const size_t bytes = static_cast<size_t>(n * t * c * h * w * elt);
  if (!st.stream) TSM_CUDA_TRY(cudaStreamCreateWithFlags(&st.stream, cudaStreamNonBlocking));
  if (bytes > st.cap) {
    if (st.dx) cudaFree(st.dx);
    if (st.dy) cudaFree(st.dy);
    st.dx = st.dy = nullptr;
    st.cap = 0;
    TSM_CUDA_TRY(cudaMalloc(&st.dx, bytes));
    TSM_CUDA_TRY(cudaMalloc(&st.dy, bytes));
    st.cap = bytes;
  }
  TSM_CUDA_TRY(cudaMemcpyAsync(st.dx, x, bytes, cudaMemcpyHostToDevice, st.stream));
  TSM_TRY(shift_launch(st.dx, st.dy, n, t, c, h, w, fold_fwd, fold_bwd, dtype, adjoint,
                       st.stream));
  TSM_CUDA_TRY(cudaMemcpyAsync(y, st.dy, bytes, cudaMemcpyDeviceToHost, st.stream));
  TSM_CUDA_TRY(cudaStreamSynchronize(st.stream));
  return TSM_OK;
}

static tsm_status check_conv_shape(int64_t n, int64_t t, int64_t h, int64_t w_, int64_t c_in,
                                   int64_t c_out, int k, int stride) {
  if (n <= 0 || t <= 0 || h <= 0 || w_ <= 0 || c_in <= 0 || c_out <= 0)
    return fail(TSM_ERR_INVALID, "conv: non-positive shape");
  if (k < 1 || (k % 2) == 0 || stride < 1)
    return fail(TSM_ERR_INVALID, "conv: odd kernel and positive stride required");
  return require_device();
}

static ConvShape conv_shape(int64_t n, int64_t t, int64_t h, int64_t w_, int64_t c_in,
                            int64_t c_out, int k, int stride, int64_t F, int64_t B) {
  return ConvShape{n, t, h, w_, c_in, c_out, k, stride, F, B};
}

tsm_status tsm_conv_fwd(const void* x, const void* w, const float* bias, const void* residual,
                        void* y, int64_t n, int64_t t, int64_t h, int64_t w_, int64_t c_in,
                        int64_t c_out, int k, int stride, int64_t fold_fwd, int64_t fold_bwd,
                        int relu, void* stream) {
  TSM_TRY(check_conv_shape(n, t, h, w_, c_in, c_out, k, stride));
  return conv_fwd(conv_shape(n, t, h, w_, c_in, c_out, k, stride, fold_fwd, fold_bwd), x, w,
                  bias, residual, y, relu, static_cast<cudaStream_t>(stream));
}

tsm_status tsm_conv_dgrad(const void* dy, const void* wt, const void* residual, const void* mask,
                          void* dx, void* scratch, int64_t n, int64_t t, int64_t h, int64_t w_,
                          int64_t c_in, int64_t c_out, int k, int stride, int64_t fold_fwd,
                          int64_t fold_bwd, void* stream) {
  TSM_TRY(check_conv_shape(n, t, h, w_, c_in, c_out, k, stride));
  return conv_dgrad(conv_shape(n, t, h, w_, c_in, c_out, k, stride, fold_fwd, fold_bwd), dy, wt,
                    residual, mask, dx, scratch, static_cast<cudaStream_t>(stream));
}

size_t tsm_conv_wgrad_workspace_bytes(int64_t n, int64_t t, int64_t h, int64_t w_, int64_t c_in,
                                      int64_t c_out, int k, int stride) {
  // The plan (slab width, CTA pair, virtual channels, split count) depends on
  // the shift split, which this query does not take: return the maximum over
  // one split of each slab class, an upper bound for every split.
  size_t b = wgrad_workspace_bytes(conv_shape(n, t, h, w_, c_in, c_out, k, stride, 0, 0));
  if (k == 1 && stride == 1)
    for (int64_t f : {8, 16, 32, 64})
      for (int64_t g : {(int64_t)0, f})
        if (f + g <= c_in)
          b = std::max(b, wgrad_workspace_bytes(conv_shape(n, t, h, w_, c_in, c_out, k, stride,
                                                           f, g)));
  return b;
}

tsm_status tsm_conv_wgrad(const void* x, const void* dy, float* dw, float* db, void* ws,
                          int64_t n, int64_t t, int64_t h, int64_t w_, int64_t c_in,
                          int64_t c_out, int k, int stride, int64_t fold_fwd, int64_t fold_bwd,
                          void* stream) {
  TSM_TRY(check_conv_shape(n, t, h, w_, c_in, c_out, k, stride));
  return conv_wgrad(conv_shape(n, t, h, w_, c_in, c_out, k, stride, fold_fwd, fold_bwd), x, dy,
                    dw, db, static_cast<float*>(ws), static_cast<cudaStream_t>(stream));
}

tsm_status tsm_weights_to_bf16(const float* w, void* w_fwd, void* w_dgrad, int64_t c_out,
                               int64_t c_in, int k, int64_t k_pad, void* stream) {
  TSM_TRY(require_device());
  return weights_to_bf16(w, w_fwd, w_dgrad, c_out, c_in, k, k_pad,
                         static_cast<cudaStream_t>(stream));
}

tsm_status tsm_maxpool_fwd(const void* x, void* y, uint8_t* argmax, int64_t frames, int64_t h,
                           int64_t w, int64_t c, void* stream) {
  TSM_TRY(require_device());
  return maxpool_fwd(x, y, argmax, frames, (int)h, (int)w, (int)c,
                     static_cast<cudaStream_t>(stream));
}

tsm_status tsm_maxpool_bwd(const void* gy, const uint8_t* argmax, void* gx, int64_t frames,
                           int64_t h, int64_t w, int64_t c, void* stream) {
  TSM_TRY(require_device());
  return maxpool_bwd(gy, argmax, gx, frames, (int)h, (int)w, (int)c,
                     static_cast<cudaStream_t>(stream));
}

size_t tsm_bias_grad_workspace_bytes(int64_t rows, int64_t c) {
  return (size_t)colsum_workspace_floats(rows, c) * 4;
}

tsm_status tsm_bias_grad(const void* g, float* db, void* ws, int64_t rows, int64_t c,
                         void* stream) {
  TSM_TRY(require_device());
  return colsum_bf16(g, db, static_cast<float*>(ws), rows, c, static_cast<cudaStream_t>(stream));
}

tsm_status tsm_layout_to_nthwc(const void* x, tsm_dtype dtype, void* y, int64_t frames, int64_t c,
                               int64_t h, int64_t w_, int64_t c_pad, void* stream) {
  TSM_TRY(require_device());
  return ntchw_to_nthwc(x, dtype, y, frames, c, h * w_, c_pad, static_cast<cudaStream_t>(stream));
}

tsm_status tsm_layout_to_ntchw(const void* x, void* y, tsm_dtype dtype, int64_t frames, int64_t c,
                               int64_t h, int64_t w_, void* stream) {
  TSM_TRY(require_device());
  return nthwc_to_ntchw(x, y, dtype, frames, c, h * w_, static_cast<cudaStream_t>(stream));
}

size_t tsm_block_workspace_bytes(const tsm_block_desc* d) { return BlockPlan(*d).bytes; }

tsm_status tsm_block_fwd(const tsm_block_desc* d, const tsm_block_params* p, const void* x,
                         void* y, void* workspace, void* stream) {
  BlockPlan P(*d);
  TSM_TRY(P.validate());
  TSM_TRY(require_device());
  if ((P.has_proj && (!p->wp || !p->bp)) || (!P.has_proj && (p->wp || p->bp)))
    return fail(TSM_ERR_INVALID, "block: projection weights do not match the block geometry");
  auto s = static_cast<cudaStream_t>(stream);
  auto* ws = static_cast<uint8_t*>(workspace);
  TSM_TRY(block_prepare_weights(P, *p, ws, true, s));
  return block_forward(P, *p, x, y, ws, nullptr, s);
}

tsm_status tsm_block_bwd(const tsm_block_desc* d, const tsm_block_params* p, const void* x,
                         const void* y, const void* gy, void* gx, const tsm_block_grads* g,
                         void* workspace, void* stream) {
  BlockPlan P(*d);
  TSM_TRY(P.validate());
  TSM_TRY(require_device());
  return block_backward(P, *p, x, gy, false, y, gx, nullptr, *g,
                        static_cast<uint8_t*>(workspace), static_cast<cudaStream_t>(stream));
}

struct tsm_net {
  std::unique_ptr<Network> impl;
  // host-buffer entry points: a private stream and device staging
  cudaStream_t hs = nullptr;
  void* dx = nullptr;  // input (f64 NTCHW), then reused for the input gradient
  size_t dx_bytes = 0;
  ~tsm_net() {
    if (dx) cudaFree(dx);
    if (hs) cudaStreamDestroy(hs);
  }
  tsm_status host_stage(size_t bytes) {
    if (!hs) TSM_CUDA_TRY(cudaStreamCreateWithFlags(&hs, cudaStreamNonBlocking));
    if (bytes > dx_bytes) {
      if (dx) cudaFree(dx);
      dx = nullptr;
      dx_bytes = 0;
      TSM_CUDA_TRY(cudaMalloc(&dx, bytes));
      dx_bytes = bytes;
    }
    return TSM_OK;
  }
};

tsm_status tsm_net_create(const tsm_net_desc* d, tsm_net** out) {
  if (!d || !out) return fail(TSM_ERR_INVALID, "tsm_net_create: null argument");
  TSM_TRY(require_device());
  std::unique_ptr<Network> n;
  TSM_TRY(Network::create(*d, &n));
  *out = new tsm_net{std::move(n)};
  return TSM_OK;
}

void tsm_net_destroy(tsm_net* net) { delete net; }
int64_t tsm_net_param_count(const tsm_net* net) {
  return net && net->impl ? net->impl->param_count() : -1;
}
int64_t tsm_net_param_tensors(const tsm_net* net) {
  return net && net->impl ? net->impl->param_tensors() : -1;
}

#define TSM_NET_CHECK(net) \
  if (!(net) || !(net)->impl) return fail(TSM_ERR_INVALID, "tsm_net: null network handle")

tsm_status tsm_net_param_info(const tsm_net* net, int64_t i, tsm_net_param* out) {
  TSM_NET_CHECK(net);
  if (!out) return fail(TSM_ERR_INVALID, "tsm_net_param_info: null output");
  if (i < 0 || i >= net->impl->param_tensors()) return fail(TSM_ERR_INVALID, "param index");
  *out = net->impl->param(i);
  return TSM_OK;
}

float* tsm_net_params(tsm_net* net) { return net && net->impl ? net->impl->params() : nullptr; }
float* tsm_net_grads(tsm_net* net) { return net && net->impl ? net->impl->grads() : nullptr; }
float* tsm_net_loss(tsm_net* net) { return net && net->impl ? net->impl->loss() : nullptr; }
float* tsm_net_logits(tsm_net* net) { return net && net->impl ? net->impl->logits() : nullptr; }

tsm_status tsm_net_forward(tsm_net* net, const void* x, tsm_dtype dtype, float* logits,
                           void* stream) {
  TSM_NET_CHECK(net);
  if (!x) return fail(TSM_ERR_INVALID, "tsm_net_forward: null input");
  return net->impl->forward(x, dtype, logits, static_cast<cudaStream_t>(stream));
}

tsm_status tsm_net_train_step(tsm_net* net, const void* x, tsm_dtype dtype, const tsm_sgd* opt,
                              void* stream) {
  TSM_NET_CHECK(net);
  if (!x) return fail(TSM_ERR_INVALID, "tsm_net_train_step: null input");
  tsm_sgd none{};
  return net->impl->train_step(x, dtype, opt ? *opt : none, static_cast<cudaStream_t>(stream));
}

int64_t tsm_net_reference_param_count(const tsm_net* net) {
  return net && net->impl ? net->impl->reference_param_count() : -1;
}

tsm_status tsm_net_set_params_reference(tsm_net* net, const double* flat, int64_t count) {
  TSM_NET_CHECK(net);
  TSM_TRY(net->host_stage(0));
  return net->impl->set_params_reference(flat, count, net->hs);
}

tsm_status tsm_net_get_params_reference(tsm_net* net, double* flat, int64_t count) {
  TSM_NET_CHECK(net);
  TSM_TRY(net->host_stage(0));
  return net->impl->get_reference(false, flat, count, net->hs);
}

tsm_status tsm_net_get_grads_reference(tsm_net* net, double* flat, int64_t count) {
  TSM_NET_CHECK(net);
  TSM_TRY(net->host_stage(0));
  return net->impl->get_reference(true, flat, count, net->hs);
}

tsm_status tsm_net_input_grad(tsm_net* net, void* gx, tsm_dtype dtype, void* stream) {
  TSM_NET_CHECK(net);
  return net->impl->input_grad(gx, dtype, static_cast<cudaStream_t>(stream));
}

tsm_status tsm_net_forward_host(tsm_net* net, const double* x, double* logits) {
  TSM_NET_CHECK(net);
  if (!x || !logits) return fail(TSM_ERR_INVALID, "tsm_net_forward_host: null argument");
  const size_t xb = (size_t)net->impl->input_elems() * sizeof(double);
  TSM_TRY(net->host_stage(xb));
  TSM_CUDA_TRY(cudaMemcpyAsync(net->dx, x, xb, cudaMemcpyHostToDevice, net->hs));
  TSM_TRY(net->impl->forward(net->dx, TSM_F64, nullptr, net->hs));
  const int64_t nl = net->impl->logits_count();
  std::vector<float> l(nl);
  TSM_CUDA_TRY(cudaMemcpyAsync(l.data(), net->impl->logits(), nl * 4, cudaMemcpyDeviceToHost,
                               net->hs));
  TSM_CUDA_TRY(cudaStreamSynchronize(net->hs));
  for (int64_t i = 0; i < nl; ++i) logits[i] = l[i];
  return TSM_OK;
}

tsm_status tsm_net_loss_gradients_host(tsm_net* net, const double* x, double* loss,
                                       double* grad_params, double* grad_input) {
  TSM_NET_CHECK(net);
  if (!x || !loss || !grad_params) return fail(TSM_ERR_INVALID, "tsm_net_loss_gradients_host: null argument");
  const size_t xb = (size_t)net->impl->input_elems() * sizeof(double);
  TSM_TRY(net->host_stage(xb));
  TSM_CUDA_TRY(cudaMemcpyAsync(net->dx, x, xb, cudaMemcpyHostToDevice, net->hs));
  tsm_sgd none{};
  TSM_TRY(net->impl->train_step(net->dx, TSM_F64, none, net->hs));
  // loss = Sigma y^2 over the step's logits in fp64 and flat order, as
  // Network::loss (net.cpp:141-146) computes it from forward()
  const int64_t nl = net->impl->logits_count();
  std::vector<float> lg(nl);
  TSM_CUDA_TRY(cudaMemcpyAsync(lg.data(), net->impl->logits(), nl * 4, cudaMemcpyDeviceToHost,
                               net->hs));
  if (grad_input) {
    TSM_TRY(net->impl->input_grad(net->dx, TSM_F64, net->hs));
    TSM_CUDA_TRY(cudaMemcpyAsync(grad_input, net->dx, xb, cudaMemcpyDeviceToHost, net->hs));
  }
  TSM_TRY(net->impl->get_reference(true, grad_params, net->impl->reference_param_count(),
                                   net->hs));  // synchronises hs
  double acc = 0.0;
  for (int64_t i = 0; i < nl; ++i) acc += (double)lg[i] * (double)lg[i];
  *loss = acc;
  return TSM_OK;
}

tsm_status tsm_net_set_graph(tsm_net* net, int enable) {
  TSM_NET_CHECK(net);
  return net->impl->set_graph(enable != 0);
}

tsm_status tsm_nccl_unique_id(void* out128) {
  if (!out128) return fail(TSM_ERR_INVALID, "tsm_nccl_unique_id: null output");
  return nccl_unique_id(out128);
}

tsm_status tsm_net_dp_init(tsm_net* net, const void* id128, int rank, int world,
                           size_t bucket_bytes) {
  TSM_NET_CHECK(net);
  if (!id128) return fail(TSM_ERR_INVALID, "tsm_net_dp_init: null unique id");
  return net->impl->dp_init(id128, rank, world, bucket_bytes);
}

}  // extern "C"
