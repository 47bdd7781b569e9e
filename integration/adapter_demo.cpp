// adapter_demo.cpp — compiled by tests/test_integration.py against the
// UNMODIFIED reference headers and libablmc_b200.so: runs the reference's own
// decay-style loop with accumulate_samples routed through the adapter, and
// prints the per-level sums next to the reference's CPU accumulate_samples.
// Without a GPU the adapter must throw std::runtime_error (no fallback).
#include <cstdio>
#include <exception>

#include "ablmc/estimators.hpp"
#include "ablmc_b200_adapter.hpp"

int main(int argc, char** argv) {
  const int n = argc > 1 ? std::atoi(argv[1]) : 20000;
  // optional: shard over this many GPUs of this process (ablmc_init_devices)
  const int gpus = argc > 2 ? std::atoi(argv[2]) : 0;
  if (gpus > 0) {
    try {
      ablmc_b200::init_devices(gpus);
    } catch (const std::exception& e) {
      std::printf("device error: %s\n", e.what());
      return 3;
    }
  }
  const ablmc::Problem pr = ablmc::Problem::make(ablmc::ModelParams{}, ablmc::Integrator::gl,
                                                 ablmc::QoISpec{}, 0.05, 0.1, 1.0, 40, 77);
  for (int l = 0; l <= 3; ++l) {
    ablmc::LevelStats gpu, cpu;
    gpu.init(l, pr.h_level(l), pr.dim());
    cpu.init(l, pr.h_level(l), pr.dim());
    try {
      ablmc_b200::accumulate_samples(gpu, 0, n, pr, l);
    } catch (const std::runtime_error& e) {
      std::printf("device error: %s\n", e.what());
      return 3;
    }
    ablmc::accumulate_samples(cpu, 0, n, 4, pr.level_sampler(l));
    std::printf("level %d gpu %.17g %.17g %lld %lld cpu %.17g %.17g %lld %lld\n", l, gpu.sum_y[0],
                gpu.sum_y2[0], (long long)gpu.n, (long long)gpu.cost_steps, cpu.sum_y[0],
                cpu.sum_y2[0], (long long)cpu.n, (long long)cpu.cost_steps);
  }
  return 0;
}
