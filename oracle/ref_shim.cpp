// ref_shim.cpp — extern "C" wrapper around the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile from
// /root/reference/proj/include (read-only, never copied) into
// oracle/_ref/libablmc_ref.so.  It is used (a) to pin the C restatement in
// oracle/ablmc_oracle.c bit-for-bit, (b) to generate golden fixtures, and (c)
// as bench.py's CPU baseline / --impl reference arm (the reference's own
// accumulate_samples with its std::thread pool, stats.hpp:96-136).
// Flags follow the reference's CMake Release build: -std=gnu++20 -O3 -DNDEBUG
// -pthread, no -march (so no FMA contraction on x86-64).
#include <chrono>
#include <cstring>
#include <exception>
#include <span>
#include <stdexcept>
#include <string>

#include "ablmc/coupling.hpp"
#include "ablmc/estimators.hpp"
#include "ablmc/integrators.hpp"
#include "ablmc/model.hpp"
#include "ablmc/noise.hpp"
#include "ablmc/particle.hpp"
#include "ablmc/qoi.hpp"
#include "ablmc/stats.hpp"

#include "../include/ablmc_b200.h"

using namespace ablmc;

namespace {

thread_local std::string g_err;

ModelParams to_params(const ablmc_model_params& m) {
  ModelParams p;
  p.kappa_sigma = m.kappa_sigma;
  p.kappa_tau = m.kappa_tau;
  p.u_star = m.u_star;
  p.H = m.H;
  p.eps_reg = m.eps_reg;
  p.x_ref = m.x_ref;
  p.noise_scale = m.noise_scale;
  return p;
}

Integrator to_ig(int ig) {
  return ig == ABLMC_SE ? Integrator::se : ig == ABLMC_GL ? Integrator::gl : Integrator::baoab;
}

QoISpec to_qoi(const ablmc_qoi_spec& q) {
  QoISpec s;
  s.kind = static_cast<QoIKind>(q.kind);
  s.a = q.a;
  s.b = q.b;
  s.r = q.r;
  s.delta = q.delta;
  if (q.kind == ABLMC_QOI_BINNED_FIELD && q.bin_edges)
    s.bin_edges.assign(q.bin_edges, q.bin_edges + q.n_edges);
  return s;
}

Problem to_problem(const ablmc_problem& pr) {
  SampleOptions opt;
  opt.signs_on = pr.signs_on != 0;
  opt.adaptive = pr.adaptive != 0;
  opt.x_adapt = pr.x_adapt;
  return Problem::make(to_params(pr.params), to_ig(pr.integrator), to_qoi(pr.qoi), pr.x0, pr.u0,
                       pr.T, pr.m0, pr.seed, opt);
}

void to_stats(const LevelStats& st, ablmc_level_stats* acc) {
  for (std::size_t i = 0; i < st.dim; ++i) {
    acc->sum_y[i] += st.sum_y[i];
    acc->sum_y2[i] += st.sum_y2[i];
  }
  acc->n += st.n;
  acc->failed += st.failed;
  acc->cost_steps += st.cost_steps;
}

void put_state(const ParticleState& s, ablmc_path_state* o, int ok) {
  o->x = s.x;
  o->u = s.u;
  o->parity = s.parity;
  o->n_refl = s.n_refl;
  o->ok = ok;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const SampleFailureError& e) {
    g_err = e.what();
    return ABLMC_ERR_SAMPLE_FAILURE;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return ABLMC_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return ABLMC_ERR_RUNTIME;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_philox4x32(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  const auto w = detail::philox4x32({ctr[0], ctr[1], ctr[2], ctr[3]}, {key[0], key[1]});
  for (int i = 0; i < 4; ++i) out[i] = w[i];
}

uint64_t ref_splitmix64(uint64_t x) { return detail::splitmix64(x); }

void ref_normals(uint64_t seed, uint32_t level, uint64_t idx, uint64_t k0, int64_t n,
                 double* out) {
  NoiseStream ns(seed, level, idx);
  for (int64_t j = 0; j < n; ++j) out[j] = ns.normal_at(k0 + uint64_t(j));
}

void ref_sde_coeffs(double x, const ablmc_model_params* m, double out[4]) {
  const SdeCoeffs c = sde_coeffs(x, to_params(*m));
  out[0] = c.sigma_u2;
  out[1] = c.lambda;
  out[2] = c.sigma;
  out[3] = c.dsigma_u2;
}

int ref_model_values(double x, double u, const ablmc_model_params* m, double out[5]) {
  return guarded([&] {
    const ModelParams p = to_params(*m);
    out[0] = sigma_u(x, p);
    out[1] = tau(x, p);
    out[2] = lambda(x, p);
    out[3] = diffusion_sigma(x, p);
    out[4] = dV_dX(x, u, p);
  });
}

double ref_se_stability_limit(const ablmc_model_params* m) {
  return se_stability_limit(to_params(*m));
}

double ref_coarse_noise_se(double xi0, double xi1, int s0, int s1, int sc) {
  return coarse_noise_se(xi0, xi1, s0, s1, sc);
}

double ref_coarse_noise_gl(double xi0, double xi1, double lam, double h, int s0, int s1,
                           int sc) {
  return coarse_noise_gl(xi0, xi1, lam, h, s0, s1, sc);
}

// reflect (particle.hpp:36-49): returns -1 on UnstableStepError.
int ref_reflect(double x, double u, double H, int parity, int64_t n_refl, double out_xu[2],
                int out_pc[2], int64_t* out_nrefl) {
  try {
    const ReflectOutcome r = reflect(x, u, H, parity, n_refl);
    out_xu[0] = r.x;
    out_xu[1] = r.u;
    out_pc[0] = r.parity;
    out_pc[1] = r.count;
    *out_nrefl = r.n_refl;
    return 0;
  } catch (const UnstableStepError&) {
    return -1;
  }
}

// One integrator step (integrators.hpp:50-117); state in/out; returns -1 on
// UnstableStepError.  parity_at_noise from StepRecord.
int ref_step(int ig, ablmc_path_state* s, double h, double xi, const ablmc_model_params* m,
             int scale_noise_by_parity, int* parity_at_noise) {
  const ModelParams p = to_params(*m);
  ParticleState st{s->x, s->u, 0.0, s->parity, s->n_refl};
  try {
    const StepRecord r = (to_ig(ig) == Integrator::baoab)
                             ? detail::baoab_step_impl(st, h, xi, p, scale_noise_by_parity != 0)
                             : step(to_ig(ig), st, h, xi, p);
    put_state(r.state, s, 1);
    if (parity_at_noise) *parity_at_noise = r.parity_at_noise;
    return 0;
  } catch (const UnstableStepError&) {
    s->ok = 0;
    return -1;
  }
}

// simulate_pair on NoiseStream(seed, level, idx) for idx in [first, first+count).
void ref_pair_states(const ablmc_problem* pr, int level, int64_t first, int64_t count,
                     ablmc_pair_state* out) {
  const ModelParams p = to_params(pr->params);
  const std::int64_t M = pr->m0 << level;
  for (int64_t i = 0; i < count; ++i) {
    NoiseStream ns(pr->seed, uint32_t(level), uint64_t(first + i));
    try {
      const PairResult r =
          simulate_pair(to_ig(pr->integrator), p, pr->x0, pr->u0, pr->T, M, ns, pr->signs_on != 0);
      put_state(r.fine, &out[i].fine, 1);
      put_state(r.coarse, &out[i].coarse, 1);
    } catch (const UnstableStepError&) {
      out[i].fine.ok = out[i].coarse.ok = 0;
    }
  }
}

void ref_path_states(const ablmc_problem* pr, int64_t M, uint32_t stream_level, int64_t first,
                     int64_t count, ablmc_path_state* out) {
  const ModelParams p = to_params(pr->params);
  for (int64_t i = 0; i < count; ++i) {
    NoiseStream ns(pr->seed, stream_level, uint64_t(first + i));
    try {
      const PathResult r = simulate_path(to_ig(pr->integrator), p, pr->x0, pr->u0, pr->T, M, ns);
      put_state(r.state, &out[i], 1);
    } catch (const UnstableStepError&) {
      out[i].ok = 0;
    }
  }
}

int ref_build_smoothing_polynomial(int r, double* coeffs) {
  return guarded([&] {
    const SmoothingPolynomial sp = build_smoothing_polynomial(r);
    for (std::size_t i = 0; i < sp.coeffs.size(); ++i) coeffs[i] = sp.coeffs[i];
  });
}

void ref_evaluate(const ablmc_qoi_spec* q, double x, double* out) {
  const QoISpec s = to_qoi(*q);
  const SmoothingPolynomial sp = build_smoothing_polynomial(s.r);
  ParticleState st{x, 0.0, 0.0, 1, 0};
  evaluate(s, sp, st, std::span<double>(out, s.size()));
}

// accumulate_samples(acc, first, count, workers, pr.level_sampler(level));
// *seconds = wall time of that call alone.
int ref_accumulate_samples(const ablmc_problem* prc, int level, int64_t first, int64_t count,
                           int workers, ablmc_level_stats* acc, double* seconds) {
  return guarded([&] {
    const Problem pr = to_problem(*prc);
    LevelStats st;
    st.init(level, pr.h_level(level), pr.dim());
    const SampleFn fn = pr.level_sampler(level);
    const auto t0 = std::chrono::steady_clock::now();
    accumulate_samples(st, first, count, workers, fn);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    to_stats(st, acc);
  });
}

int ref_accumulate_paths(const ablmc_problem* prc, int64_t M, uint32_t stream_level,
                         int64_t first, int64_t count, int workers, ablmc_level_stats* acc,
                         double* seconds) {
  return guarded([&] {
    const Problem pr = to_problem(*prc);
    LevelStats st;
    st.init(0, pr.T / double(M), pr.dim());
    const SampleFn fn = pr.path_sampler(M, stream_level);
    const auto t0 = std::chrono::steady_clock::now();
    accumulate_samples(st, first, count, workers, fn);
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    to_stats(st, acc);
  });
}

int ref_decay_sweep(const ablmc_problem* prc, int l_min, int l_max, int64_t n, int workers,
                    ablmc_decay_row* rows) {
  return guarded([&] {
    const Problem pr = to_problem(*prc);
    const auto rr = decay_sweep(pr, l_min, l_max, n, workers);
    for (std::size_t i = 0; i < rr.size(); ++i) {
      rows[i].level = rr[i].level;
      rows[i].h = rr[i].h;
      rows[i].var_y = rr[i].var_y;
      rows[i].mean_y = rr[i].mean_y;
      rows[i].se_mean = rr[i].se_mean;
      rows[i].n = rr[i].n;
      rows[i].cost_steps = rr[i].cost_steps;
    }
  });
}

static void fill_result(const RunResult& r, ablmc_run_result* out) {
  std::memset(out, 0, sizeof(*out) - 2 * sizeof(double*));
  out->levels_used = r.levels_used;
  out->n_levels = int(r.level_stats.size());
  out->estimate = r.estimate.empty() ? 0.0 : r.estimate[0];
  out->stat_error = r.stat_error.empty() ? 0.0 : r.stat_error[0];
  out->bias_estimate = r.bias_estimate;
  out->alpha = r.alpha;
  out->c1 = r.c1;
  out->total_cost_steps = r.total_cost_steps;
  out->pilot_cost_steps = r.pilot_cost_steps;
  out->failed_samples = r.failed_samples;
  out->wall_seconds = r.wall_seconds;
  out->n_warnings = int(r.warnings.size());
  for (std::size_t l = 0; l < r.level_stats.size() && l < ABLMC_MAX_LEVELS; ++l) {
    const LevelStats& st = r.level_stats[l];
    out->level_n[l] = st.n;
    out->level_failed[l] = st.failed;
    out->level_cost[l] = st.cost_steps;
    out->level_h[l] = st.h;
    out->level_sum_y[l] = st.sum_y[0];
    out->level_sum_y2[l] = st.sum_y2[0];
  }
  for (std::size_t i = 0; i < r.estimate.size(); ++i) {
    if (out->est_vec) out->est_vec[i] = r.estimate[i];
    if (out->err_vec) out->err_vec[i] = r.stat_error[i];
  }
}

int ref_run_mlmc(const ablmc_problem* prc, double eps, const ablmc_mlmc_options* o,
                 int workers, ablmc_run_result* out) {
  return guarded([&] {
    const Problem pr = to_problem(*prc);
    MlmcOptions mo;
    mo.pilot_n = o->pilot_n;
    mo.pilot_levels_max = o->pilot_levels_max;
    mo.init_n = o->init_n;
    mo.l_max = o->l_max;
    mo.workers = workers;
    BiasFit fit;
    if (o->use_bias_fit) {
      fit.alpha = o->alpha;
      fit.c1 = o->c1;
      mo.bias_fit = &fit;
    }
    fill_result(run_mlmc(pr, eps, mo), out);
  });
}

int ref_run_stmc(const ablmc_problem* prc, int64_t M_L, double eps, int64_t fixed_n,
                 int workers, ablmc_run_result* out) {
  return guarded([&] {
    const Problem pr = to_problem(*prc);
    fill_result(run_stmc(pr, M_L, eps, fixed_n, workers), out);
  });
}

}  // extern "C"
