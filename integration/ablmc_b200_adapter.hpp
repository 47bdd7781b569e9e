// ablmc_b200_adapter.hpp — the binding a maintainer adds to the reference
// (header-only C++ `ablmc`) to route its level sampling through the B200
// library.  Include it after the reference headers; link libablmc_b200.so.
//
// It converts the reference's own types (ablmc::Problem, estimators.hpp:26-94;
// ablmc::LevelStats, stats.hpp:26-88) to the C ABI of include/ablmc_b200.h and
// maps error codes back to the reference's exception types, so a call site
//
//     accumulate_samples(st, first, count, workers, pr.level_sampler(l));   // stats.hpp:96
//
// becomes
//
//     ablmc_b200::accumulate_samples(st, first, count, pr, l);
//
// with identical semantics (index range, failed-sample exclusion, cost
// accounting, add-merge into st).  See INTEGRATION.md.
#pragma once

#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "ablmc/estimators.hpp"
#include "ablmc/stats.hpp"
#include "ablmc_b200.h"

namespace ablmc_b200 {

struct Descriptor {  // keeps bin_edges alive for the duration of a call
  ablmc_problem c{};
  std::vector<double> edges;
};

inline Descriptor describe(const ablmc::Problem& pr) {
  Descriptor d;
  ablmc_problem_defaults(&d.c);
  const ablmc::ModelParams& p = pr.params;
  d.c.params = {p.kappa_sigma, p.kappa_tau, p.u_star, p.H, p.eps_reg, p.x_ref, p.noise_scale};
  d.c.integrator = static_cast<int32_t>(pr.integrator);  // se, gl, baoab: same order
  d.c.signs_on = pr.opt.signs_on ? 1 : 0;
  d.c.adaptive = pr.opt.adaptive ? 1 : 0;
  d.c.x_adapt = pr.opt.x_adapt;
  d.c.qoi.kind = static_cast<int32_t>(pr.qoi.kind);      // QoIKind: same order
  d.c.qoi.a = pr.qoi.a;
  d.c.qoi.b = pr.qoi.b;
  d.c.qoi.r = pr.qoi.r;
  d.c.qoi.delta = pr.qoi.delta;
  d.edges = pr.qoi.bin_edges;
  d.c.qoi.n_edges = static_cast<int32_t>(d.edges.size());
  d.c.qoi.bin_edges = d.edges.empty() ? nullptr : d.edges.data();
  d.c.x0 = pr.x0;
  d.c.u0 = pr.u0;
  d.c.T = pr.T;
  d.c.m0 = pr.m0;
  d.c.seed = pr.seed;
  return d;
}

inline void check(int rc) {
  if (rc == ABLMC_OK) return;
  const std::string msg = ablmc_last_error();
  switch (rc) {
    case ABLMC_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case ABLMC_ERR_SAMPLE_FAILURE: throw ablmc::SampleFailureError(msg);
    default: throw std::runtime_error(msg);
  }
}

inline ablmc_level_stats view(ablmc::LevelStats& st) {
  ablmc_level_stats v{};
  v.level = st.level;
  v.h = st.h;
  v.dim = static_cast<int64_t>(st.dim);
  v.sum_y = st.sum_y.data();
  v.sum_y2 = st.sum_y2.data();
  v.n = st.n;
  v.failed = st.failed;
  v.cost_steps = st.cost_steps;
  return v;
}

// The reference fans accumulate_samples out over `workers` threads in one
// process (stats.hpp:120-135); the device analogue is one process driving n
// GPUs: after init_devices(n) every accumulate call below -- and so every
// iteration of a driver loop built on it -- shards its super-blocks over the
// n GPUs and exchanges the partials in ONE NCCL all-gather, with the same
// bits as one GPU.  Without it the library uses one device.
inline void init_devices(int n, const int* devices = nullptr) {
  check(ablmc_init_devices(n, devices));
}

// accumulate_samples(acc, first, count, workers, pr.level_sampler(level))
inline void accumulate_samples(ablmc::LevelStats& acc, std::int64_t first, std::int64_t count,
                               const ablmc::Problem& pr, int level) {
  Descriptor d = describe(pr);
  ablmc_level_stats v = view(acc);
  check(ablmc_accumulate_samples(&d.c, level, first, count, &v));
  acc.n = v.n;
  acc.failed = v.failed;
  acc.cost_steps = v.cost_steps;
}

// accumulate_samples(acc, first, count, workers, pr.path_sampler(M, stream_level))
inline void accumulate_paths(ablmc::LevelStats& acc, std::int64_t first, std::int64_t count,
                             const ablmc::Problem& pr, std::int64_t M,
                             std::uint32_t stream_level = 0) {
  Descriptor d = describe(pr);
  ablmc_level_stats v = view(acc);
  check(ablmc_accumulate_paths(&d.c, M, stream_level, first, count, &v));
  acc.n = v.n;
  acc.failed = v.failed;
  acc.cost_steps = v.cost_steps;
}

}  // namespace ablmc_b200
