// TSM-ResNet-50 8-frame executor and data-parallel training step.
//
// Reference: build_tsm8f (arch.cpp:140-161) expanded by expand (arch.cpp:325)
// and executed by Network (net.cpp): Network::Network (39-76: init and the
// flat parameter order), forward (128-139), loss = sum y^2 (141-146),
// loss_gradients (160-272).  The reference has no device or collective
// layers; the data-parallel step (batch sharded over GPUs, gradient buckets
// allreduced with NCCL over NVLink, overlapped with backward) is the
// B200-native replacement for the analytic model of sim.cpp:104-175.
//
// Layout: activations NTHWC bf16; parameters one flat fp32 buffer in the
// reference's declaration order (net.cpp:63-75), each weight tensor in the
// GEMM layout [c_out][kh][kw][c_in] (stem c_in zero-padded 3 -> 8).  Gradients
// mirror the parameter buffer, so an allreduce bucket is a contiguous range.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <memory>
#include <string>
#include <vector>

#include "aux_kernels.cuh"
#include "block.h"
#include "common.cuh"
#include "head_kernels.cuh"
#include "network.h"

namespace tsm {

// ---------------------------------------------------------------------------
// NCCL, loaded on first use so the library has no hard dependency on it.

namespace {

typedef int nccl_result;
typedef void* nccl_comm;
struct NcclId {
  char internal[128];
};
struct Nccl {
  nccl_result (*get_unique_id)(NcclId*) = nullptr;
  nccl_result (*comm_init_rank)(nccl_comm*, int, NcclId, int) = nullptr;
  nccl_result (*all_reduce)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t) =
      nullptr;
  nccl_result (*comm_destroy)(nccl_comm) = nullptr;
  nccl_result (*comm_abort)(nccl_comm) = nullptr;
  nccl_result (*comm_get_async_error)(nccl_comm, nccl_result*) = nullptr;
  const char* (*error_string)(nccl_result) = nullptr;
  bool ok = false;
  std::string why;
};
constexpr int kNcclFloat32 = 7;  // ncclFloat32
constexpr int kNcclSum = 0;      // ncclSum

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      r.why = std::string("dlopen libnccl.so.2: ") + dlerror();
      return r;
    }
    r.get_unique_id = reinterpret_cast<decltype(r.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    r.comm_init_rank = reinterpret_cast<decltype(r.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    r.all_reduce = reinterpret_cast<decltype(r.all_reduce)>(dlsym(h, "ncclAllReduce"));
    r.comm_destroy = reinterpret_cast<decltype(r.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    r.error_string = reinterpret_cast<decltype(r.error_string)>(dlsym(h, "ncclGetErrorString"));
    r.comm_abort = reinterpret_cast<decltype(r.comm_abort)>(dlsym(h, "ncclCommAbort"));
    r.comm_get_async_error =
        reinterpret_cast<decltype(r.comm_get_async_error)>(dlsym(h, "ncclCommGetAsyncError"));
    r.ok = r.get_unique_id && r.comm_init_rank && r.all_reduce && r.comm_destroy &&
           r.comm_abort && r.comm_get_async_error;
    if (!r.ok) r.why = "libnccl.so.2 lacks required symbols";
    return r;
  }();
  return n;
}

tsm_status nccl_status(nccl_result r, const char* where) {
  if (r == 0) return TSM_OK;
  const Nccl& n = nccl();
  return fail(TSM_ERR_NCCL, std::string(where) + ": " +
                                (n.error_string ? n.error_string(r) : std::to_string(r)));
}

constexpr nccl_result kNcclInProgress = 7;  // ncclInProgress

// Asynchronous NCCL errors (a failed or vanished peer) surface only through
// ncclCommGetAsyncError; without this check a broken communicator makes the
// step hang in its next allreduce.  On error the communicator is aborted (so
// queued collectives return) and TSM_ERR_NCCL is reported.
tsm_status nccl_check_async(nccl_comm& comm) {
  if (!comm) return TSM_OK;
  const Nccl& n = nccl();
  nccl_result async = 0;
  TSM_TRY(nccl_status(n.comm_get_async_error(comm, &async), "ncclCommGetAsyncError"));
  if (async == 0 || async == kNcclInProgress) return TSM_OK;
  const std::string why = std::string("NCCL asynchronous error: ") +
                          (n.error_string ? n.error_string(async) : std::to_string(async));
  n.comm_abort(comm);
  comm = nullptr;
  return fail(TSM_ERR_NCCL, why);
}

}  // namespace

tsm_status nccl_unique_id(void* out128) {
  const Nccl& n = nccl();
  if (!n.ok) return fail(TSM_ERR_NCCL, n.why);
  NcclId id;
  TSM_TRY(nccl_status(n.get_unique_id(&id), "ncclGetUniqueId"));
  memcpy(out128, id.internal, 128);
  return TSM_OK;
}

// ---------------------------------------------------------------------------

struct DevBuf {
  void* p = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  tsm_status alloc(size_t bytes) {
    if (p) cudaFree(p);
    p = nullptr;
    return cuda_status(cudaMalloc(&p, std::max<size_t>(bytes, 256)), "cudaMalloc");
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

struct Network::Impl {
  tsm_net_desc d;
  int64_t N, T, frames;
  int64_t stem_cin = 8;  // 3 input channels zero-padded to 8 (16-byte rows)
  ConvShape stem;       // the 7x7/s2 conv geometry (for extents)
  ConvShape stem_gemm;  // the same conv as a GEMM over the materialised im2col matrix
  bool stem_s2d = false;  // even extents: space-to-depth 4x4/s1 conv instead
  bool micro = false;     // micro-tsm preset: no stem / pool, 8 input channels
  int64_t c_in0 = 3, c_last = 2048;  // network input / last block channels
  DevBuf in_act, gin;     // micro-tsm: NTHWC bf16 input and its (unused) gradient
  int64_t h1, w1, h2, w2;  // after stem, after pool
  std::vector<BlockPlan> blocks;
  std::vector<tsm_net_param> table;
  int64_t n_params = 0;
  // per-unit parameter ranges [first, last) in table / flat offsets
  struct Unit {
    int64_t off0, off1;  // flat range of the unit's parameters
  };
  std::vector<Unit> units;  // stem, blocks..., fc
  // params
  DevBuf params, grads, mom, decay;
  // activations
  DevBuf stem_a, stem_out, pool_out, pool_arg;
  std::vector<std::unique_ptr<DevBuf>> act;  // block outputs
  std::vector<std::unique_ptr<DevBuf>> act_bits;  // their ReLU bitmasks (backward masks)
  std::vector<std::unique_ptr<DevBuf>> bws;  // block workspaces
  DevBuf stem_wf, stem_dw, feat, logits, glogits, gfeat, gmap, gpool, gstem, stem_wg, stem_cs,
      loss;
  DevBuf jobs_fwd, jobs_train;  // batched weight-conversion tables
  int njobs = 0;
  // data parallel
  nccl_comm comm = nullptr;
  int rank = 0, world = 1;
  size_t bucket_bytes = 25u << 20;
  cudaStream_t comm_stream = nullptr;
  std::vector<cudaEvent_t> ev;  // per unit "grads ready"
  cudaEvent_t comm_done = nullptr;
  // weight gradients on a side stream (block_backward's WgradStream)
  cudaStream_t wstream = nullptr;
  cudaEvent_t wfork[3] = {nullptr, nullptr, nullptr}, wjoin = nullptr, wmain = nullptr;
  cudaEvent_t wconv = nullptr;  // block-weight conversion done (side stream)
  bool wconv_pending = false;
  // CUDA-graph mode of train_step (launch-bound small batches): one
  // captured step per (input pointer, dtype, update) key, replayed on gs;
  // the SGD hyperparameters are read from hp_dev so a replay takes new ones
  struct Graph {
    const void* x;
    tsm_dtype dt;
    int update;
    cudaGraphExec_t exec;
    uint64_t launches;  // kernels per replay (for tsm_launch_count)
  };
  bool graph_on = false;
  int64_t eager_steps = 0;
  std::vector<Graph> graphs;
  cudaStream_t gs = nullptr;
  cudaEvent_t g_in = nullptr, g_out = nullptr;
  DevBuf hp_dev;

  ~Impl() {
    for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
    if (g_in) cudaEventDestroy(g_in);
    if (g_out) cudaEventDestroy(g_out);
    if (gs) cudaStreamDestroy(gs);
    if (comm) nccl().comm_destroy(comm);
    for (auto e : ev) cudaEventDestroy(e);
    if (comm_done) cudaEventDestroy(comm_done);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    for (auto e : wfork)
      if (e) cudaEventDestroy(e);
    if (wjoin) cudaEventDestroy(wjoin);
    if (wmain) cudaEventDestroy(wmain);
    if (wconv) cudaEventDestroy(wconv);
    if (wstream) cudaStreamDestroy(wstream);
  }

  int64_t add_param(const char* name, int64_t co, int64_t kh, int64_t kw, int64_t ci,
                    int64_t ci_ref, bool bias) {
    tsm_net_param p{};
    p.offset = n_params;
    p.dims[0] = co;
    p.dims[1] = kh;
    p.dims[2] = kw;
    p.dims[3] = ci;
    p.ci_ref = ci_ref;
    p.is_bias = bias ? 1 : 0;
    p.numel = co * kh * kw * ci;
    snprintf(p.name, sizeof p.name, "%s", name);
    table.push_back(p);
    n_params += p.numel;
    return p.offset;
  }

  float* P(int64_t i) const { return params.as<float>() + table[i].offset; }
  // "res4.2" for the unit whose first parameter is table[i] ("res4.2.w1")
  std::string unit_name(size_t i) const {
    const std::string n = table[i].name;
    return n.substr(0, n.rfind('.'));
  }
  float* G(int64_t i) const { return grads.as<float>() + table[i].offset; }
};

Network::Network() : m(new Impl) {}
Network::~Network() = default;

tsm_status Network::create(const tsm_net_desc& d, std::unique_ptr<Network>* out) {
  if (d.batch <= 0 || d.frames <= 0 || d.height <= 0 || d.width <= 0 || d.classes <= 0)
    return fail(TSM_ERR_INVALID, "net: non-positive shape");
  std::unique_ptr<Network> net(new Network);
  Impl& I = *net->m;
  I.d = d;
  I.N = d.batch;
  I.T = d.frames;
  I.frames = I.N * I.T;
  I.micro = d.arch == TSM_ARCH_MICRO_TSM;
  if (d.arch != TSM_ARCH_TSM8F && !I.micro) return fail(TSM_ERR_INVALID, "net: unknown arch");
  I.stem = ConvShape{I.N, I.T, d.height, d.width, I.stem_cin, 64, 7, 2, 0, 0};
  I.h1 = I.stem.h_out();
  I.w1 = I.stem.w_out();
  I.stem_gemm = ConvShape{I.N, I.T, I.h1, I.w1, kStemK, 64, 1, 1, 0, 0};
  I.h2 = (I.h1 + 2 - 3) / 2 + 1;
  I.w2 = (I.w1 + 2 - 3) / 2 + 1;

  // parameter table in the reference order (net.cpp:63-75)
  int64_t u0 = I.n_params;
  static const int kBlocks[4] = {3, 4, 6, 3};
  static const int64_t kChannels[4] = {256, 512, 1024, 2048};
  static const int kMicroBlocks[4] = {2, 0, 0, 0};  // arch.cpp:225-229
  static const int64_t kMicroChannels[4] = {16, 0, 0, 0};
  const int* nblocks = I.micro ? kMicroBlocks : kBlocks;
  const int64_t* chans = I.micro ? kMicroChannels : kChannels;
  int64_t cin = 64, h = I.h2, w = I.w2;
  if (I.micro) {  // input_shape {1, 4, 8, 5, 5}: blocks straight on the input
    I.c_in0 = 8;
    cin = 8;
    h = d.height;
    w = d.width;
  } else {
    I.add_param("conv1.w", 64, 7, 7, I.stem_cin, 3, false);
    I.add_param("conv1.b", 64, 1, 1, 1, 1, true);
    I.units.push_back({u0, I.n_params});
  }
  for (int s = 0; s < 4; ++s) {
    for (int b = 0; b < nblocks[s]; ++b) {
      tsm_block_desc bd{};
      bd.n = I.N;
      bd.t = I.T;
      bd.h = h;
      bd.w = w;
      bd.c_in = cin;
      bd.c_out = chans[s];
      bd.stride = (s > 0 && b == 0) ? 2 : 1;
      if (d.shift_num != 0) {
        int64_t f = 0, bb = 0;
        TSM_TRY(tsm_validate_shift(d.shift_num, d.shift_den, d.shift_num, d.shift_den, cin, &f,
                                   &bb));
        bd.fold_fwd = f;
        bd.fold_bwd = bb;
      }
      BlockPlan P(bd);
      TSM_TRY(P.validate());
      char nm[48];
      const int64_t wd = P.width;
      u0 = I.n_params;
      snprintf(nm, sizeof nm, "res%d.%d.w1", s + 2, b);
      I.add_param(nm, wd, 1, 1, cin, cin, false);
      snprintf(nm, sizeof nm, "res%d.%d.b1", s + 2, b);
      I.add_param(nm, wd, 1, 1, 1, 1, true);
      snprintf(nm, sizeof nm, "res%d.%d.w2", s + 2, b);
      I.add_param(nm, wd, 3, 3, wd, wd, false);
      snprintf(nm, sizeof nm, "res%d.%d.b2", s + 2, b);
      I.add_param(nm, wd, 1, 1, 1, 1, true);
      snprintf(nm, sizeof nm, "res%d.%d.w3", s + 2, b);
      I.add_param(nm, bd.c_out, 1, 1, wd, wd, false);
      snprintf(nm, sizeof nm, "res%d.%d.b3", s + 2, b);
      I.add_param(nm, bd.c_out, 1, 1, 1, 1, true);
      if (P.has_proj) {
        snprintf(nm, sizeof nm, "res%d.%d.wp", s + 2, b);
        I.add_param(nm, bd.c_out, 1, 1, cin, cin, false);
        snprintf(nm, sizeof nm, "res%d.%d.bp", s + 2, b);
        I.add_param(nm, bd.c_out, 1, 1, 1, 1, true);
      }
      I.units.push_back({u0, I.n_params});
      I.blocks.push_back(P);
      cin = bd.c_out;
      h = P.ho;
      w = P.wo;
    }
  }
  I.c_last = cin;
  u0 = I.n_params;
  I.add_param("fc.w", d.classes, 1, 1, cin, cin, false);
  I.add_param("fc.b", d.classes, 1, 1, 1, 1, true);
  I.units.push_back({u0, I.n_params});

  // allocations
  TSM_TRY(I.params.alloc(I.n_params * 4));
  TSM_TRY(I.grads.alloc(I.n_params * 4));
  TSM_TRY(I.mom.alloc(I.n_params * 4));
  TSM_TRY(I.decay.alloc(I.n_params));
  TSM_CUDA_TRY(cudaMemset(I.mom.p, 0, I.n_params * 4));
  TSM_CUDA_TRY(cudaMemset(I.grads.p, 0, I.n_params * 4));
  TSM_CUDA_TRY(cudaMemset(I.params.p, 0, I.n_params * 4));
  {
    std::vector<uint8_t> dm(I.n_params, 0);
    for (auto& p : I.table)
      if (!p.is_bias) std::fill(dm.begin() + p.offset, dm.begin() + p.offset + p.numel, 1);
    TSM_CUDA_TRY(cudaMemcpy(I.decay.p, dm.data(), dm.size(), cudaMemcpyHostToDevice));
  }
  const int64_t pix1 = I.frames * I.h1 * I.w1, pix2 = I.frames * I.h2 * I.w2;
  // conv1 input: the space-to-depth tensor (16 channels at H/2 x W/2) when
  // the extents are even, else the materialised im2col matrix
  I.stem_s2d = I.d.height % 2 == 0 && I.d.width % 2 == 0 && I.h1 * 2 == I.d.height &&
               I.w1 * 2 == I.d.width;
  if (I.micro) {
    const int64_t pin = I.frames * I.d.height * I.d.width * I.c_in0 * 2;
    TSM_TRY(I.in_act.alloc(pin));
    TSM_TRY(I.gin.alloc(pin));
  } else {
  TSM_TRY(I.stem_a.alloc(I.stem_s2d ? pix1 * 16 * 2 : pix1 * kStemK * 2));
  // (the fused stem + pool kernel never stores the stem output)
  if (!(I.stem_s2d && stem_pool_enabled())) TSM_TRY(I.stem_out.alloc(pix1 * 64 * 2));
  TSM_TRY(I.pool_out.alloc(pix2 * 64 * 2));
  TSM_TRY(I.pool_arg.alloc(pix2 * 64));
  TSM_TRY(I.gpool.alloc(pix2 * 64 * 2));
  TSM_TRY(I.gstem.alloc(pix1 * 64 * 2));
  TSM_TRY(I.stem_wf.alloc(64 * 256 * 2));  // >= 64 x kStemK
  TSM_TRY(I.stem_dw.alloc(64 * 256 * 4));
  TSM_TRY(I.stem_wg.alloc(I.stem_s2d ? stem_s2d_wgrad_workspace_bytes(I.N, I.T, I.h1, I.w1)
                                     : wgrad_workspace_bytes(I.stem_gemm)));
  TSM_TRY(I.stem_cs.alloc(colsum_workspace_floats(pix1, 64) * 4));
  }
  for (auto& P : I.blocks) {
    I.act.emplace_back(new DevBuf);
    TSM_TRY(I.act.back()->alloc(I.frames * P.ho * P.wo * P.d.c_out * 2));
    I.act_bits.emplace_back(new DevBuf);  // ReLU bitmask (tcgen05 blocks with c_out % 32 == 0)
    if (!P.generic && P.d.c_out % 32 == 0)
      TSM_TRY(I.act_bits.back()->alloc(I.frames * P.ho * P.wo * P.d.c_out / 8));
    I.bws.emplace_back(new DevBuf);
    TSM_TRY(I.bws.back()->alloc(P.bytes));
  }
  const BlockPlan& last = I.blocks.back();
  TSM_TRY(I.feat.alloc(I.N * I.c_last * 4));
  TSM_TRY(I.logits.alloc(I.N * d.classes * 4));
  TSM_TRY(I.glogits.alloc(I.N * d.classes * 4));
  TSM_TRY(I.gfeat.alloc(I.N * I.c_last * 4));
  TSM_TRY(I.gmap.alloc(I.frames * last.ho * last.wo * I.c_last * 2));
  TSM_TRY(I.loss.alloc(4));
  I.ev.resize(I.units.size());
  for (auto& e : I.ev) TSM_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  TSM_CUDA_TRY(cudaEventCreateWithFlags(&I.comm_done, cudaEventDisableTiming));
  TSM_CUDA_TRY(cudaStreamCreateWithFlags(&I.wstream, cudaStreamNonBlocking));
  for (auto& e : I.wfork) TSM_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  TSM_CUDA_TRY(cudaEventCreateWithFlags(&I.wjoin, cudaEventDisableTiming));
  TSM_CUDA_TRY(cudaEventCreateWithFlags(&I.wmain, cudaEventDisableTiming));
  TSM_CUDA_TRY(cudaEventCreateWithFlags(&I.wconv, cudaEventDisableTiming));
  *out = std::move(net);
  return TSM_OK;
}

int64_t Network::param_count() const { return m->n_params; }
int64_t Network::param_tensors() const { return (int64_t)m->table.size(); }
const tsm_net_param& Network::param(int64_t i) const { return m->table[i]; }
float* Network::params() const { return m->params.as<float>(); }
float* Network::grads() const { return m->grads.as<float>(); }
float* Network::loss() const { return m->loss.as<float>(); }
float* Network::logits() const { return m->logits.as<float>(); }

int64_t Network::reference_param_count() const {
  int64_t n = 0;
  for (const auto& p : m->table) n += p.is_bias ? p.numel : p.dims[0] * p.dims[1] * p.dims[2] * p.ci_ref;
  return n;
}

int64_t Network::logits_count() const { return m->N * m->d.classes; }

int64_t Network::input_elems() const {
  return m->frames * m->c_in0 * m->d.height * m->d.width;
}

// Reference flat order = the table order; a weight is (c_out, c_in, 1, kh,
// kw) there and [c_out][kh][kw][c_in (padded)] here.
tsm_status Network::set_params_reference(const double* flat, int64_t count, cudaStream_t s) {
  Impl& I = *m;
  if (!flat) return fail(TSM_ERR_INVALID, "set_params_reference: null input");
  if (count != reference_param_count())
    return fail(TSM_ERR_INVALID, "expected " + std::to_string(reference_param_count()) +
                                     " parameters, got " + std::to_string(count));
  std::vector<float> host(I.n_params, 0.f);
  int64_t pos = 0;
  for (const auto& p : I.table) {
    float* dst = host.data() + p.offset;
    if (p.is_bias) {
      for (int64_t i = 0; i < p.numel; ++i) dst[i] = (float)flat[pos + i];
      pos += p.numel;
      continue;
    }
    const int64_t co = p.dims[0], kh = p.dims[1], kw = p.dims[2], ci = p.dims[3], cr = p.ci_ref;
    for (int64_t o = 0; o < co; ++o)
      for (int64_t c = 0; c < cr; ++c)
        for (int64_t y = 0; y < kh; ++y)
          for (int64_t x = 0; x < kw; ++x)
            dst[((o * kh + y) * kw + x) * ci + c] = (float)flat[pos + ((o * cr + c) * kh + y) * kw + x];
    pos += co * cr * kh * kw;
  }
  TSM_CUDA_TRY(cudaMemcpyAsync(I.params.p, host.data(), I.n_params * 4, cudaMemcpyHostToDevice, s));
  return cuda_status(cudaStreamSynchronize(s), "set_params_reference");
}

tsm_status Network::get_reference(bool grads, double* flat, int64_t count, cudaStream_t s) {
  Impl& I = *m;
  if (!flat) return fail(TSM_ERR_INVALID, "get_reference: null output");
  if (count != reference_param_count())
    return fail(TSM_ERR_INVALID, "expected room for " + std::to_string(reference_param_count()) +
                                     " parameters, got " + std::to_string(count));
  std::vector<float> host(I.n_params);
  TSM_CUDA_TRY(cudaMemcpyAsync(host.data(), grads ? I.grads.p : I.params.p, I.n_params * 4,
                               cudaMemcpyDeviceToHost, s));
  TSM_CUDA_TRY(cudaStreamSynchronize(s));
  int64_t pos = 0;
  for (const auto& p : I.table) {
    const float* src = host.data() + p.offset;
    if (p.is_bias) {
      for (int64_t i = 0; i < p.numel; ++i) flat[pos + i] = src[i];
      pos += p.numel;
      continue;
    }
    const int64_t co = p.dims[0], kh = p.dims[1], kw = p.dims[2], ci = p.dims[3], cr = p.ci_ref;
    for (int64_t o = 0; o < co; ++o)
      for (int64_t c = 0; c < cr; ++c)
        for (int64_t y = 0; y < kh; ++y)
          for (int64_t x = 0; x < kw; ++x)
            flat[pos + ((o * cr + c) * kh + y) * kw + x] = src[((o * kh + y) * kw + x) * ci + c];
    pos += co * cr * kh * kw;
  }
  return TSM_OK;
}

tsm_status Network::input_grad(void* gx, tsm_dtype dt, cudaStream_t s) {
  Impl& I = *m;
  if (!gx) return fail(TSM_ERR_INVALID, "input_grad: null output");
  if (dt != TSM_F32 && dt != TSM_F64) return fail(TSM_ERR_UNSUPPORTED, "input_grad: f32 or f64");
  if (I.micro)  // the first unit's input gradient (NTHWC bf16) in the reference layout
    return nthwc_to_ntchw(I.gin.p, gx, dt, I.frames, I.c_in0, I.d.height * I.d.width, s);
  // the stem output gradient: the step's pool backward left it in gstem,
  // unless the pool backward was fused into the stem weight gradient
  if (I.stem_s2d && stem_pool_bwd_enabled())
    TSM_TRY(maxpool_bwd(I.gpool.p, I.pool_arg.as<uint8_t>(), I.gstem.p, I.frames, (int)I.h1,
                        (int)I.w1, 64, s));
  return stem_dgrad(I.gstem.p, I.P(0), gx, dt, I.frames, (int)I.d.height, (int)I.d.width,
                    (int)I.h1, (int)I.w1, s);
}

tsm_status Network::dp_init(const void* id128, int rank, int world, size_t bucket_bytes) {
  const Nccl& n = nccl();
  if (!n.ok) return fail(TSM_ERR_NCCL, n.why);
  if (world < 1 || rank < 0 || rank >= world) return fail(TSM_ERR_INVALID, "dp: bad rank/world");
  NcclId id;
  memcpy(id.internal, id128, 128);
  if (m->comm) {
    n.comm_destroy(m->comm);
    m->comm = nullptr;
  }
  TSM_TRY(nccl_status(n.comm_init_rank(&m->comm, world, id, rank), "ncclCommInitRank"));
  TSM_TRY(nccl_check_async(m->comm));
  m->rank = rank;
  m->world = world;
  if (bucket_bytes) m->bucket_bytes = bucket_bytes;
  if (!m->comm_stream)
    TSM_CUDA_TRY(cudaStreamCreateWithFlags(&m->comm_stream, cudaStreamNonBlocking));
  return TSM_OK;
}

// TSM_SIDE_STREAM=0 serialises the step on the caller's stream (per-layer
// attribution of a profiler launch list; same results).
static bool side_stream_enabled() {
  static const bool on = [] {
    const char* e = getenv("TSM_SIDE_STREAM");
    return !e || atoi(e) != 0;
  }();
  return on;
}

tsm_status Network::prepare_weights(bool dgrad, cudaStream_t s) {
  Impl& I = *m;
  TraceScope trace("weights");
  if (!I.micro)
    TSM_TRY(I.stem_s2d ? stem_weights_s2d(I.P(0), I.stem_wf.p, s)
                       : stem_weights(I.P(0), I.stem_wf.p, s));
  // fp32 masters -> bf16 forward (+ dgrad) operands of every block conv in
  // one launch; the job tables are built once (all pointers are fixed)
  TSM_TRY(build_weight_jobs(dgrad));
  DevBuf& table = dgrad ? I.jobs_train : I.jobs_fwd;
  if (I.njobs == 0) return TSM_OK;
  // on the side stream, after everything before it on s (the previous
  // step's SGD wrote the masters); forward_impl joins before the blocks
  if (!side_stream_enabled()) return weights_to_bf16_batch(table.as<WeightJob>(), I.njobs, s);
  TSM_CUDA_TRY(cudaEventRecord(I.wmain, s));
  TSM_CUDA_TRY(cudaStreamWaitEvent(I.wstream, I.wmain, 0));
  TSM_TRY(weights_to_bf16_batch(table.as<WeightJob>(), I.njobs, I.wstream));
  TSM_CUDA_TRY(cudaEventRecord(I.wconv, I.wstream));
  I.wconv_pending = true;
  return TSM_OK;
}

tsm_status Network::build_weight_jobs(bool dgrad) {
  Impl& I = *m;
  DevBuf& table = dgrad ? I.jobs_train : I.jobs_fwd;
  if (!table.p) {
    std::vector<WeightJob> jobs;
    size_t ti = I.micro ? 0 : 2;
    for (size_t b = 0; b < I.blocks.size(); ++b) {
      const BlockPlan& P = I.blocks[b];
      uint8_t* ws = I.bws[b]->as<uint8_t>();
      auto add = [&](size_t t, size_t of, size_t od, int64_t co, int64_t ci, int kk) {
        jobs.push_back({I.P(t), ws + of, dgrad ? ws + od : nullptr, co, ci, kk, kk * ci});
      };
      if (!P.generic) {  // the direct (generic) convs read the fp32 masters
        add(ti, P.o_w1f, P.o_w1d, P.width, P.d.c_in, 1);
        add(ti + 2, P.o_w2f, P.o_w2d, P.width, P.width, 9);
        add(ti + 4, P.o_w3f, P.o_w3d, P.d.c_out, P.width, 1);
        if (P.has_proj) add(ti + 6, P.o_wpf, P.o_wpd, P.d.c_out, P.d.c_in, 1);
      }
      ti += P.has_proj ? 8 : 6;
    }
    I.njobs = (int)jobs.size();
    if (jobs.empty()) return TSM_OK;
    TSM_TRY(table.alloc(jobs.size() * sizeof(WeightJob)));
    TSM_CUDA_TRY(cudaMemcpy(table.p, jobs.data(), jobs.size() * sizeof(WeightJob),
                            cudaMemcpyHostToDevice));
  }
  return TSM_OK;
}

tsm_status Network::forward_impl(const void* x, tsm_dtype dt, cudaStream_t s) {
  Impl& I = *m;
  // input NTCHW (reference layout) -> NTHWC bf16, channels 3 -> 8 zero-padded
  // conv1's im2col matrix straight from the reference-layout input
  // conv1: 7x7/s2 conv with bias, no ReLU (expand_layer keeps standalone layers
  // linear, arch.cpp:280-283)
  if (I.micro) {
    // micro-tsm: the blocks run on the input itself (NTCHW -> NTHWC bf16)
    TSM_TRY(ntchw_to_nthwc(x, dt, I.in_act.p, I.frames, I.c_in0, I.d.height * I.d.width, I.c_in0,
                           s));
  } else {
  TraceScope trace_stem("fwd stem+pool");
  if (I.stem_s2d && stem_pool_enabled()) {
    // space-to-depth (16 channels at half resolution), then the 4x4/s1 conv
    // and pool1 (1x3x3/s2 max pool, arch.cpp:69-76) in one kernel
    TSM_TRY(stem_s2d(x, dt, I.stem_a.p, I.frames, (int)I.d.height, (int)I.d.width, s));
    TSM_TRY(stem_pool_fwd(I.stem_a.p, I.stem_wf.p, I.P(1), I.pool_out.p,
                          I.pool_arg.as<uint8_t>(), I.frames, I.h1, I.w1, s));
  } else {
    if (I.stem_s2d) {
      TSM_TRY(stem_s2d(x, dt, I.stem_a.p, I.frames, (int)I.d.height, (int)I.d.width, s));
      TSM_TRY(stem_s2d_fwd(I.stem_a.p, I.stem_wf.p, I.P(1), I.stem_out.p, I.frames, I.h1, I.w1,
                           s));
    } else {
      TSM_TRY(stem_im2col(x, dt, I.stem_a.p, I.frames, (int)I.d.height, (int)I.d.width, s));
      TSM_TRY(conv_fwd(I.stem_gemm, I.stem_a.p, I.stem_wf.p, I.P(1), nullptr, I.stem_out.p, 0,
                       s));
    }
    // pool1: 1x3x3/s2 max pool (arch.cpp:69-76)
    TSM_TRY(maxpool_fwd(I.stem_out.p, I.pool_out.p, I.pool_arg.as<uint8_t>(), I.frames,
                        (int)I.h1, (int)I.w1, 64, s));
  }
  }
  const void* cur = I.micro ? I.in_act.p : I.pool_out.p;
  size_t ti = I.micro ? 0 : 2;
  if (I.wconv_pending) {  // block weights converted on the side stream
    TSM_CUDA_TRY(cudaStreamWaitEvent(s, I.wconv, 0));
    I.wconv_pending = false;
  }
  for (size_t b = 0; b < I.blocks.size(); ++b) {
    const BlockPlan& P = I.blocks[b];
    tsm_block_params bp{I.P(ti), I.P(ti + 1), I.P(ti + 2), I.P(ti + 3), I.P(ti + 4), I.P(ti + 5),
                        P.has_proj ? I.P(ti + 6) : nullptr, P.has_proj ? I.P(ti + 7) : nullptr};
    TraceScope trace(I.unit_name(ti) + " fwd");
    TSM_TRY(block_forward(P, bp, cur, I.act[b]->p, I.bws[b]->as<uint8_t>(),
                          I.act_bits[b]->as<uint32_t>(), s));
    cur = I.act[b]->p;
    ti += P.has_proj ? 8 : 6;
  }
  const BlockPlan& L = I.blocks.back();
  TraceScope trace_head("fwd head");  // (to the end of forward_impl)
  TSM_TRY(gap_fwd(cur, I.feat.as<float>(), I.N, I.T * L.ho * L.wo, (int)I.c_last, s));
  const int64_t fc = (int64_t)I.table.size() - 2;
  return fc_fwd(I.feat.as<float>(), I.P(fc), I.P(fc + 1), I.logits.as<float>(), (int)I.N, (int)I.c_last,
                (int)I.d.classes, s);
}

tsm_status Network::forward(const void* x, tsm_dtype dt, float* logits_out, cudaStream_t s) {
  TSM_TRY(prepare_weights(false, s));
  TSM_TRY(forward_impl(x, dt, s));
  if (logits_out && logits_out != m->logits.as<float>())
    TSM_CUDA_TRY(cudaMemcpyAsync(logits_out, m->logits.p, m->N * m->d.classes * 4,
                                 cudaMemcpyDeviceToDevice, s));
  return TSM_OK;
}

tsm_status Network::set_graph(bool on) {
  m->graph_on = on;
  return TSM_OK;
}

tsm_status Network::train_step(const void* x, tsm_dtype dt, const tsm_sgd& opt, cudaStream_t s) {
  Impl& I = *m;
  // errors of the previous step's allreduces (non-blocking poll)
  if (I.comm) TSM_TRY(nccl_check_async(I.comm));
  if (I.world > 1 && !I.comm) return fail(TSM_ERR_NCCL, "dp: communicator was aborted");
  // eager: graphs off, a data-parallel step (NCCL stays outside capture
  // here), or the measurement probe recording (its events are host-side
  // bookkeeping per launch)
  // The first step always runs eagerly: lazy one-time setup (kernel
  // attributes, job tables) then happens outside any capture.
  if (!I.graph_on || I.world > 1 || probe_enabled() || I.eager_steps == 0) {
    ++I.eager_steps;
    return train_step_impl(x, dt, opt, s, nullptr);
  }
  if (!I.gs) {
    TSM_CUDA_TRY(cudaStreamCreateWithFlags(&I.gs, cudaStreamNonBlocking));
    TSM_CUDA_TRY(cudaEventCreateWithFlags(&I.g_in, cudaEventDisableTiming));
    TSM_CUDA_TRY(cudaEventCreateWithFlags(&I.g_out, cudaEventDisableTiming));
    TSM_TRY(I.hp_dev.alloc(4 * sizeof(float)));
  }
  // everything a step allocates lazily (weight-conversion job tables) is
  // allocated before capture: no cudaMalloc inside a capturing stream
  TSM_TRY(build_weight_jobs(true));
  const int update = opt.enabled ? 1 : 0;
  Impl::Graph* g = nullptr;
  for (auto& e : I.graphs)
    if (e.x == x && e.dt == dt && e.update == update) g = &e;
  if (!g) {
    if (I.graphs.size() >= 4) {
      cudaGraphExecDestroy(I.graphs.front().exec);
      I.graphs.erase(I.graphs.begin());
    }
    // capture one step on gs (the side and comm streams join through the
    // step's own event dependencies)
    const uint64_t l0 = tsm_launch_count();
    TSM_CUDA_TRY(cudaStreamBeginCapture(I.gs, cudaStreamCaptureModeThreadLocal));
    const tsm_status st = train_step_impl(x, dt, opt, I.gs, I.hp_dev.as<float>());
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(I.gs, &graph);
    if (st != TSM_OK || ce != cudaSuccess) {
      if (graph) cudaGraphDestroy(graph);
      (void)cudaGetLastError();  // a failed capture must not poison later launch checks
      return st != TSM_OK ? st : cuda_status(ce, "cudaStreamEndCapture");
    }
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    TSM_CUDA_TRY(ie);
    TSM_CUDA_TRY(cudaGraphUpload(exec, I.gs));
    I.graphs.push_back({x, dt, update, exec, tsm_launch_count() - l0});
    g = &I.graphs.back();
    // capture counted the kernels without running them: take them back
    count_launches(0 - g->launches);
  }
  const float hp[4] = {opt.lr, opt.momentum, opt.weight_decay, opt.grad_scale};
  TSM_CUDA_TRY(cudaEventRecord(I.g_in, s));
  TSM_CUDA_TRY(cudaStreamWaitEvent(I.gs, I.g_in, 0));
  // pageable source: staged at the call, safe to reuse on the next step
  TSM_CUDA_TRY(cudaMemcpyAsync(I.hp_dev.p, hp, sizeof hp, cudaMemcpyHostToDevice, I.gs));
  TSM_CUDA_TRY(cudaGraphLaunch(g->exec, I.gs));
  count_launches(g->launches);
  TSM_CUDA_TRY(cudaEventRecord(I.g_out, I.gs));
  return cuda_status(cudaStreamWaitEvent(s, I.g_out, 0), "graph replay join");
}

tsm_status Network::train_step_impl(const void* x, tsm_dtype dt, const tsm_sgd& opt,
                                    cudaStream_t s, const float* hp) {
  Impl& I = *m;
  TSM_TRY(prepare_weights(true, s));
  TSM_TRY(forward_impl(x, dt, s));
  const int64_t fc = (int64_t)I.table.size() - 2;
  const bool dp = I.comm && I.world > 1;
  // loss = sum y^2, g = 2y (net.cpp:178-181)
  {
    TraceScope trace_loss("loss");
    TSM_TRY(sq_loss(I.logits.as<float>(), I.glogits.as<float>(), I.loss.as<float>(),
                    (int)(I.N * I.d.classes), s));
  }
  // bucket bookkeeping: grads become final unit by unit in reverse order
  int64_t pending_end = I.n_params;  // [pending_start, pending_end) not yet launched
  size_t unit = I.units.size() - 1;
  // Launch the allreduce of flat range [off0, off1) once `ready` has fired.
  auto launch_bucket = [&](int64_t off0, int64_t off1, cudaEvent_t ready) -> tsm_status {
    TSM_CUDA_TRY(cudaStreamWaitEvent(I.comm_stream, ready, 0));
    float* gp = I.grads.as<float>() + off0;
    return nccl_status(nccl().all_reduce(gp, gp, (size_t)(off1 - off0), kNcclFloat32, kNcclSum,
                                         I.comm, I.comm_stream),
                       "ncclAllReduce");
  };
  // A unit's gradients are final once both streams passed it: the block
  // wgrads run on I.wstream, fc / stem on s (joined into the side stream).
  cudaStream_t sw = I.wstream;
  auto unit_done = [&](size_t u, bool force) -> tsm_status {
    if (!dp) return TSM_OK;
    TSM_CUDA_TRY(cudaEventRecord(I.wmain, s));
    TSM_CUDA_TRY(cudaStreamWaitEvent(sw, I.wmain, 0));
    TSM_CUDA_TRY(cudaEventRecord(I.ev[u], sw));
    const int64_t start = I.units[u].off0;
    if (force || (size_t)(pending_end - start) * 4 >= I.bucket_bytes) {
      if (pending_end > start) TSM_TRY(launch_bucket(start, pending_end, I.ev[u]));
      pending_end = start;
    }
    return TSM_OK;
  };
  // fc backward (kernels.cpp:542-576) and GAP backward
  const BlockPlan& L = I.blocks.back();
  {
    TraceScope trace_head("bwd head");
    TSM_TRY(fc_bwd(I.glogits.as<float>(), I.feat.as<float>(), I.P(fc), I.gfeat.as<float>(),
                   I.G(fc), I.G(fc + 1), (int)I.N, (int)I.c_last, (int)I.d.classes, s));
    TSM_TRY(unit_done(unit--, false));
    TSM_TRY(gap_bwd(I.gfeat.as<float>(), I.gmap.p, I.N, I.T * L.ho * L.wo, (int)I.c_last, s));
  }
  // blocks in reverse; each unit's input gradient is pre-masked with the
  // previous unit's ReLU (its output y), fused into the conv1 dgrad epilogue
  const void* g = I.gmap.p;
  bool g_masked = false;
  size_t ti = I.table.size() - 2;
  for (size_t bi = I.blocks.size(); bi-- > 0;) {
    const BlockPlan& P = I.blocks[bi];
    ti -= P.has_proj ? 8 : 6;
    tsm_block_params bp{I.P(ti), I.P(ti + 1), I.P(ti + 2), I.P(ti + 3), I.P(ti + 4), I.P(ti + 5),
                        P.has_proj ? I.P(ti + 6) : nullptr, P.has_proj ? I.P(ti + 7) : nullptr};
    tsm_block_grads bg{I.G(ti), I.G(ti + 1), I.G(ti + 2), I.G(ti + 3), I.G(ti + 4), I.G(ti + 5),
                       P.has_proj ? I.G(ti + 6) : nullptr, P.has_proj ? I.G(ti + 7) : nullptr};
    const void* x_in = bi ? I.act[bi - 1]->p : (I.micro ? I.in_act.p : I.pool_out.p);
    void* gx = bi ? I.bws[bi - 1]->as<uint8_t>() + I.blocks[bi - 1].o_g
                  : (I.micro ? I.gin.p : I.gpool.p);
    // producer ReLU mask of gx: the previous unit's output bits (or the bf16
    // output itself where no bitmask exists)
    const uint32_t* gx_bits = bi ? I.act_bits[bi - 1]->as<uint32_t>() : nullptr;
    const void* gx_mask = (bi && !gx_bits) ? I.act[bi - 1]->p : nullptr;
    WgradStream side;
    side.sw = side_stream_enabled() ? sw : nullptr;
    for (int k = 0; k < 3; ++k) side.fork[k] = I.wfork[k];
    TraceScope trace(I.unit_name(ti) + " bwd");
    TSM_TRY(block_backward(P, bp, x_in, g, g_masked, I.act[bi]->p, gx, gx_mask, bg,
                           I.bws[bi]->as<uint8_t>(), s, I.act_bits[bi]->as<uint32_t>(), gx_bits,
                           side));
    if (bi == 0 && I.micro) TSM_TRY(unit_done(unit, true));  // no stem unit: flush
    else TSM_TRY(unit_done(unit--, false));
    g = gx;
    g_masked = true;
  }
  // pool1 backward, then conv1 (stem) weight and bias gradients
  if (!I.micro) {
  TraceScope trace_stem("bwd pool+stem");
  if (I.stem_s2d && stem_pool_bwd_enabled()) {
    // pool backward gathered straight into the stem weight gradient's operand
    // (Network::input_grad recomputes the stem gradient when it is asked for)
    TSM_TRY(stem_s2d_wgrad_pool(I.stem_a.p, I.gpool.p, I.pool_arg.as<uint8_t>(),
                                I.stem_dw.as<float>(), I.G(1), I.stem_wg.as<float>(), I.N, I.T,
                                I.h1, I.w1, s));
    TSM_TRY(stem_wgrad_scatter_s2d(I.stem_dw.as<float>(), I.G(0), s));
    TSM_TRY(unit_done(unit, true));
  } else {
  TSM_TRY(maxpool_bwd(I.gpool.p, I.pool_arg.as<uint8_t>(), I.gstem.p, I.frames, (int)I.h1,
                      (int)I.w1, 64, s));
  if (I.stem_s2d) {
    TSM_TRY(stem_s2d_wgrad(I.stem_a.p, I.gstem.p, I.stem_dw.as<float>(), I.G(1),
                           I.stem_wg.as<float>(), I.N, I.T, I.h1, I.w1, s));
    TSM_TRY(stem_wgrad_scatter_s2d(I.stem_dw.as<float>(), I.G(0), s));
  } else {
    TSM_TRY(conv_wgrad(I.stem_gemm, I.stem_a.p, I.gstem.p, I.stem_dw.as<float>(), I.G(1),
                       I.stem_wg.as<float>(), s));
    TSM_TRY(stem_wgrad_scatter(I.stem_dw.as<float>(), I.G(0), s));
  }
  TSM_TRY(unit_done(unit, true));
  }
  }
  // join the weight-gradient stream (all gradients final; the next step's
  // forward overwrites the activations it reads)
  // (TSM_SIDE_STREAM=0 without DP: nothing ran on it, and under graph
  // capture a join with an uncaptured stream would be an error)
  if (side_stream_enabled() || dp) {
    TSM_CUDA_TRY(cudaEventRecord(I.wjoin, sw));
    TSM_CUDA_TRY(cudaStreamWaitEvent(s, I.wjoin, 0));
  }
  if (dp) {
    TSM_CUDA_TRY(cudaEventRecord(I.comm_done, I.comm_stream));
    TSM_CUDA_TRY(cudaStreamWaitEvent(s, I.comm_done, 0));
    TSM_TRY(nccl_check_async(I.comm));
  }
  TraceScope trace_sgd("sgd");
  if (opt.enabled)
    TSM_TRY(sgd_update(I.params.as<float>(), I.grads.as<float>(), I.mom.as<float>(),
                       I.decay.as<uint8_t>(), I.n_params, opt.lr, opt.momentum, opt.weight_decay,
                       opt.grad_scale, s, hp));
  return TSM_OK;
}

}  // namespace tsm
