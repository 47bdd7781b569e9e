// adapter_demo.cpp — compiled by tests/test_integration.py against the
// UNMODIFIED reference headers and libablmc_b200.so: runs the reference's own
// decay-style loop with accumulate_samples routed through the adapter, and
// prints the per-level sums next to the reference's CPU accumulate_samples.
// Without a GPU the adapter must throw std::runtime_error (no fallback).
#include <cstdio>
#include <exception>

#include "ablmc/estimators.hpp"
#include "ablmc_b200_adapter.hpp"

#include <cstring>

// "drivers" mode: the reference's run_mlmc / run_stmc / decay_sweep on its CPU
// sampler next to the adapter's (every level sampled on the device), same
// seed: the same levels and N_l, estimates equal up to summation rounding.
static void print_run(const char* tag, const ablmc::RunResult& r) {
  std::printf("%s levels_used %d estimate %.17g stat_error %.17g bias %.17g alpha %.17g c1 %.17g "
              "cost %lld pilot %lld failed %lld warnings %zu N_l",
              tag, r.levels_used, r.estimate[0], r.stat_error[0], r.bias_estimate, r.alpha, r.c1,
              (long long)r.total_cost_steps, (long long)r.pilot_cost_steps,
              (long long)r.failed_samples, r.warnings.size());
  for (const ablmc::LevelStats& st : r.level_stats) std::printf(" %lld", (long long)st.n);
  std::printf("\n");
}

static int drivers_demo() {
  const ablmc::Problem pr = ablmc::Problem::make(ablmc::ModelParams{}, ablmc::Integrator::gl,
                                                 ablmc::QoISpec{}, 0.05, 0.1, 1.0, 40, 77);
  try {
    ablmc::MlmcOptions o;
    o.workers = 4;
    print_run("mlmc gpu", ablmc_b200::run_mlmc(pr, 4e-4, o));
    print_run("mlmc cpu", ablmc::run_mlmc(pr, 4e-4, o));
    print_run("stmc gpu", ablmc_b200::run_stmc(pr, 160, 1e-3));
    print_run("stmc cpu", ablmc::run_stmc(pr, 160, 1e-3, 0, 4));
    const auto g = ablmc_b200::decay_sweep(pr, 1, 3, 5000);
    const auto c = ablmc::decay_sweep(pr, 1, 3, 5000, 4);
    for (std::size_t i = 0; i < g.size(); ++i)
      std::printf("decay %d gpu %.17g %.17g %lld %lld cpu %.17g %.17g %lld %lld\n", g[i].level,
                  g[i].var_y, g[i].mean_y, (long long)g[i].n, (long long)g[i].cost_steps,
                  c[i].var_y, c[i].mean_y, (long long)c[i].n, (long long)c[i].cost_steps);
    std::printf("decay empty %zu\n", ablmc_b200::decay_sweep(pr, 3, 2, 10).size());
  } catch (const std::runtime_error& e) {
    std::printf("device error: %s\n", e.what());
    return 3;
  }
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::strcmp(argv[1], "drivers") == 0) return drivers_demo();
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
