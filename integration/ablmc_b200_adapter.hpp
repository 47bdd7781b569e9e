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

// ---------------------------------------------------------------- drivers
// The reference's drivers (estimators.hpp:230-485) with every level sampled
// on the device: the library's host drivers make the reference's decisions
// (pilot fit, level choice, N_l allocation rounds: the same floating-point
// operations in the same order), so these return what the reference's own
// run_mlmc / run_stmc / decay_sweep / cost_sweep return on the same seed, up
// to the rounding of the level sums (a different fixed summation tree).
// `workers` has no device meaning and is ignored.
inline ablmc::RunResult to_run_result(const ablmc_run_result& r, std::size_t dim,
                                      const std::vector<double>& est,
                                      const std::vector<double>& err,
                                      const std::vector<double>& sy,
                                      const std::vector<double>& sy2) {
  ablmc::RunResult out;
  out.estimate = est;
  out.stat_error = err;
  out.bias_estimate = r.bias_estimate;
  out.alpha = r.alpha;
  out.c1 = r.c1;
  out.levels_used = r.levels_used;
  for (int l = 0; l < r.n_levels; ++l) {
    ablmc::LevelStats st;
    st.init(l, r.level_h[l], dim);
    for (std::size_t i = 0; i < dim; ++i) {
      st.sum_y[i] = sy[std::size_t(l) * dim + i];
      st.sum_y2[i] = sy2[std::size_t(l) * dim + i];
    }
    st.n = r.level_n[l];
    st.failed = r.level_failed[l];
    st.cost_steps = r.level_cost[l];
    out.level_stats.push_back(std::move(st));
  }
  out.total_cost_steps = r.total_cost_steps;
  out.pilot_cost_steps = r.pilot_cost_steps;
  out.failed_samples = r.failed_samples;
  out.wall_seconds = r.wall_seconds;
  // the reference's two warning strings (estimators.hpp:352-373)
  if (r.warnings_mask & 1)
    out.warnings.push_back("Var[Y_1] >= Var[Y_0]/2: coarsest level M_0 is too coarse to pay off");
  if (r.warnings_mask & 2)
    out.warnings.push_back("sample allocation did not converge in 64 rounds");
  return out;
}

struct ResultBuffers {  // caller-owned storage behind ablmc_run_result's optional vectors
  std::vector<double> est, err, sy, sy2;
  ablmc_run_result r{};
  explicit ResultBuffers(std::size_t dim)
      : est(dim), err(dim), sy(ABLMC_MAX_LEVELS * dim), sy2(ABLMC_MAX_LEVELS * dim) {
    r.est_vec = est.data();
    r.err_vec = err.data();
    r.level_sum_y_vec = sy.data();
    r.level_sum_y2_vec = sy2.data();
  }
};

// run_mlmc(pr, eps, o)  (estimators.hpp:284-397)
inline ablmc::RunResult run_mlmc(const ablmc::Problem& pr, double eps,
                                 const ablmc::MlmcOptions& o = {}) {
  Descriptor d = describe(pr);
  ablmc_mlmc_options oc;
  ablmc_mlmc_options_defaults(&oc);
  oc.pilot_n = o.pilot_n;
  oc.pilot_levels_max = o.pilot_levels_max;
  oc.init_n = o.init_n;
  oc.l_max = o.l_max;
  if (o.bias_fit != nullptr) {
    oc.use_bias_fit = 1;
    oc.alpha = o.bias_fit->alpha;
    oc.c1 = o.bias_fit->c1;
  }
  ResultBuffers b(pr.dim());
  check(ablmc_run_mlmc(&d.c, eps, &oc, &b.r));
  return to_run_result(b.r, pr.dim(), b.est, b.err, b.sy, b.sy2);
}

// run_stmc(pr, M_L, eps, fixed_n)  (estimators.hpp:230-269)
inline ablmc::RunResult run_stmc(const ablmc::Problem& pr, std::int64_t M_L, double eps,
                                 std::int64_t fixed_n = 0) {
  Descriptor d = describe(pr);
  ResultBuffers b(pr.dim());
  check(ablmc_run_stmc(&d.c, M_L, eps, fixed_n, &b.r));
  return to_run_result(b.r, pr.dim(), b.est, b.err, b.sy, b.sy2);
}

// decay_sweep(pr, l_min, l_max, n_per_level)  (estimators.hpp:415-432)
inline std::vector<ablmc::DecayRow> decay_sweep(const ablmc::Problem& pr, int l_min, int l_max,
                                                std::int64_t n_per_level) {
  pr.check_se_stability(pr.T / double(pr.m0));
  if (l_max < l_min) return {};  // the reference's loop does not run
  Descriptor d = describe(pr);
  std::vector<ablmc_decay_row> rows(std::size_t(l_max - l_min + 1));
  check(ablmc_decay_sweep(&d.c, l_min, l_max, n_per_level, rows.data()));
  std::vector<ablmc::DecayRow> out;
  for (const ablmc_decay_row& r : rows)
    out.push_back({r.level, r.h, r.var_y, r.mean_y, r.se_mean, r.n, r.cost_steps});
  return out;
}

// cost_sweep(pr, method, eps_values, fit)  (estimators.hpp:456-485)
inline std::vector<ablmc::CostRow> cost_sweep(const ablmc::Problem& pr, ablmc::Method method,
                                              std::span<const double> eps_values,
                                              const ablmc::BiasFit& fit) {
  Descriptor d = describe(pr);
  std::vector<ablmc_cost_row> rows(eps_values.size());
  check(ablmc_cost_sweep(&d.c, method == ablmc::Method::stmc ? 0 : 1, eps_values.data(),
                         int(eps_values.size()), fit.alpha, fit.c1, rows.data()));
  std::vector<ablmc::CostRow> out;
  for (const ablmc_cost_row& r : rows) {
    ablmc::CostRow c;
    c.eps = r.eps;
    c.method = method;
    c.integrator = pr.integrator;
    c.cost_steps = r.cost_steps;
    c.wall_seconds = r.wall_seconds;
    c.estimate = r.estimate;
    c.stat_error = r.stat_error;
    out.push_back(c);
  }
  return out;
}

}  // namespace ablmc_b200
