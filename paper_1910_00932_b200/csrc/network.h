// TSM-ResNet-50 executor + data-parallel step (see network.cu).
#pragma once
#include <cuda_runtime.h>

#include <memory>

#include "tsm_b200.h"

namespace tsm {

tsm_status nccl_unique_id(void* out128);

class Network {
 public:
  struct Impl;
  static tsm_status create(const tsm_net_desc& d, std::unique_ptr<Network>* out);
  ~Network();
  int64_t param_count() const;
  int64_t param_tensors() const;
  const tsm_net_param& param(int64_t i) const;
  float* params() const;
  float* grads() const;
  float* loss() const;
  float* logits() const;
  tsm_status dp_init(const void* id128, int rank, int world, size_t bucket_bytes);
  tsm_status forward(const void* x, tsm_dtype dt, float* logits_out, cudaStream_t s);
  tsm_status train_step(const void* x, tsm_dtype dt, const tsm_sgd& opt, cudaStream_t s);
  // CUDA-graph replay of train_step (see Impl::Graph)
  tsm_status set_graph(bool on);
  // Reference-layout parameter exchange (net.cpp:63-75 order, ConvWeights
  // (c_out, c_in, kt, kh, kw) / FcWeights (c_out, c_in) layout, fp64, host).
  int64_t reference_param_count() const;
  tsm_status set_params_reference(const double* flat, int64_t count, cudaStream_t s);
  tsm_status get_reference(bool grads, double* flat, int64_t count, cudaStream_t s);
  // dL/dx of the last train_step, NTCHW in dt (Gradients::input, net.hpp:36-40)
  tsm_status input_grad(void* gx, tsm_dtype dt, cudaStream_t s);
  int64_t input_elems() const;
  int64_t logits_count() const;

 private:
  Network();
  // The block-weight conversion runs on the side stream, overlapping the
  // stem; forward_impl waits for it before the first block.
  tsm_status prepare_weights(bool dgrad, cudaStream_t s);
  tsm_status build_weight_jobs(bool dgrad);  // host-side tables (allocates once)
  tsm_status forward_impl(const void* x, tsm_dtype dt, cudaStream_t s);
  tsm_status train_step_impl(const void* x, tsm_dtype dt, const tsm_sgd& opt, cudaStream_t s,
                             const float* hp);
  std::unique_ptr<Impl> m;
};

}  // namespace tsm
