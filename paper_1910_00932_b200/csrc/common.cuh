// Shared plumbing for the tsm_b200 C ABI: per-thread error text, status
// helpers, launch counting.  No exception ever leaves an extern "C" function.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <cstdio>
#include <string>

#include "tsm_b200.h"

namespace tsm {

std::string& last_error();
// Counts this library's kernel launches (tsm_launch_count) and, while the
// launch trace is on (tsm_trace_enable), appends the current trace label
// once per launch: an issue-ordered list of which layer each kernel belongs
// to, joined 1:1 with a profiler's launch list.
void count_launches(uint64_t n = 1);
bool trace_on();
// RAII: label the launches issued inside the scope ("res4.2 dgrad c3").
struct TraceScope {
  std::string saved;
  explicit TraceScope(const std::string& label);
  ~TraceScope();
};
// Measurement probe around the fused shift + 1x1 conv forward launches
// (tsm_probe_shift_conv1): begin/end record CUDA events on `s` when enabled.
void probe_conv1_begin(cudaStream_t s, int64_t c_in, int64_t c_out, int64_t pixels);
void probe_conv1_end(cudaStream_t s);
bool probe_enabled();

inline tsm_status fail(tsm_status s, const std::string& msg) {
  last_error() = msg;
  return s;
}

inline tsm_status cuda_status(cudaError_t e, const char* where) {
  if (e == cudaSuccess) return TSM_OK;
  return fail(TSM_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// Returns TSM_ERR_CUDA unless the current device is an sm_100-class part.
tsm_status require_device();

inline int64_t elt_size(tsm_dtype d) {
  switch (d) {
    case TSM_F32: return 4;
    case TSM_BF16: return 2;
    case TSM_F16: return 2;
    case TSM_F64: return 8;
  }
  return 0;
}

}  // namespace tsm

#define TSM_CUDA_TRY(expr)                                       \
  do {                                                           \
    tsm_status _s = ::tsm::cuda_status((expr), #expr);           \
    if (_s != TSM_OK) return _s;                                 \
  } while (0)

#define TSM_TRY(expr)            \
  do {                           \
    tsm_status _s = (expr);      \
    if (_s != TSM_OK) return _s; \
  } while (0)
