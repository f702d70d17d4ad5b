// A program written against the reference API only (vidperf::Network,
// net.hpp:15-54): builds a preset network (seed 42), draws the
// gradcheck_test.cpp input (seed 43), and writes forward logits, loss,
// parameter gradients and input gradient to a raw fp64 file.  Run as is it
// is the reference CPU executor; run with
//   LD_PRELOAD=integration/_build/libvidperf_gpu_net_shim.so
// every Network call of the same binary executes on the B200
// (tests/test_dropin_gpu.py compares the two files).
//
//   net_shim_demo <micro-tsm|micro-tsm-noshift|micro-linear|tsm8f-64> <clips> <out.bin>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "vidperf/arch.hpp"
#include "vidperf/net.hpp"
#include "vidperf/tensor.hpp"

using namespace vidperf;

int main(int argc, char** argv) {
  if (argc != 4) {
    std::fprintf(stderr, "usage: %s <preset> <clips> <out.bin>\n", argv[0]);
    return 2;
  }
  const std::string p = argv[1];
  ArchSpec a;
  if (p == "micro-tsm") a = build_micro_tsm();
  else if (p == "micro-tsm-noshift") a = build_micro_tsm(Rational{0, 1});
  else if (p == "micro-linear") a = build_micro_linear();
  else if (p == "tsm8f-64") {
    a = build_tsm8f();
    a.input_shape.h = a.input_shape.w = 64;
  } else {
    std::fprintf(stderr, "unknown preset %s\n", p.c_str());
    return 2;
  }
  Network net(a, 42);
  Shape5D s = a.input_shape;
  s.n = std::atoll(argv[2]);
  const Tensor5D x = random_normal(s, 43);
  const Tensor5D y = net.forward(x);
  const double l = net.loss(x);
  const Network::Gradients g = net.loss_gradients(x);
  std::FILE* f = std::fopen(argv[3], "wb");
  if (!f) return 2;
  const double counts[4] = {(double)y.size(), 1.0, (double)g.params.size(), (double)g.input.size()};
  std::fwrite(counts, sizeof(double), 4, f);
  std::fwrite(y.data().data(), sizeof(double), y.size(), f);
  std::fwrite(&l, sizeof(double), 1, f);
  std::fwrite(&g.loss, sizeof(double), 1, f);
  std::fwrite(g.params.data(), sizeof(double), g.params.size(), f);
  std::fwrite(g.input.data().data(), sizeof(double), g.input.size(), f);
  std::fclose(f);
  std::printf("%s: %lld parameters, loss %.9e, gradient loss %.9e\n", p.c_str(),
              (long long)net.param_count(), l, g.loss);
  return 0;
}
