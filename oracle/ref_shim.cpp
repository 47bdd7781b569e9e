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

#include "ablmc/config.hpp"
#include "ablmc/coupling.hpp"
#include "ablmc/estimators.hpp"
#include "ablmc/output.hpp"
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

// Extended-SDE oracle (integrators.hpp:119-189, acceptance criterion 7): n
// steps of extended_step_oracle from (x0, u0) with draws xi[0..n), folded back
// to the physical state (X, U) = S (eta(x~), u~) with S = fold_sign.
void ref_extended_path(int ig, const ablmc_model_params* m, double x0, double u0, double h,
                       int64_t n, const double* xi, double out_xu[2], int* out_sign) {
  const ModelParams p = to_params(*m);
  ExtendedState e{x0, u0, 0.0};
  for (int64_t k = 0; k < n; ++k) e = extended_step_oracle(e, h, xi[k], p, to_ig(ig));
  const double eta = fold_height(e.x, p.H);
  const int sign = eta >= 0.0 ? +1 : -1;
  out_xu[0] = sign * eta;
  out_xu[1] = sign * e.u;
  *out_sign = sign;
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
          pr->adaptive
              ? simulate_pair_adaptive(to_ig(pr->integrator), p, pr->x0, pr->u0, pr->T,
                                       pr->T / double(M), pr->x_adapt, ns, pr->signs_on != 0)
              : simulate_pair(to_ig(pr->integrator), p, pr->x0, pr->u0, pr->T, M, ns,
                              pr->signs_on != 0);
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
      const PathResult r =
          pr->adaptive ? simulate_path_adaptive(to_ig(pr->integrator), p, pr->x0, pr->u0, pr->T,
                                                pr->T / double(M), pr->x_adapt, ns)
                       : simulate_path(to_ig(pr->integrator), p, pr->x0, pr->u0, pr->T, M, ns);
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
  double* keep[4] = {out->est_vec, out->err_vec, out->level_sum_y_vec, out->level_sum_y2_vec};
  std::memset(out, 0, sizeof(*out));
  out->est_vec = keep[0];
  out->err_vec = keep[1];
  out->level_sum_y_vec = keep[2];
  out->level_sum_y2_vec = keep[3];
  for (const auto& w : r.warnings) {
    if (w.rfind("Var[Y_1]", 0) == 0) out->warnings_mask |= 1;
    if (w.rfind("sample allocation", 0) == 0) out->warnings_mask |= 2;
  }
  for (std::size_t l = 0; l < r.level_stats.size() && l < ABLMC_MAX_LEVELS; ++l) {
    const LevelStats& st = r.level_stats[l];
    for (std::size_t i = 0; i < st.dim; ++i) {
      if (out->level_sum_y_vec) out->level_sum_y_vec[l * st.dim + i] = st.sum_y[i];
      if (out->level_sum_y2_vec) out->level_sum_y2_vec[l * st.dim + i] = st.sum_y2[i];
    }
  }
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

// ---------------------------------------------------------- output.hpp
static RunConfig to_cfg(const ablmc_run_config& c) {
  RunConfig k;
  k.model = to_params(c.model);
  k.method = c.method == 0 ? Method::stmc : Method::mlmc;
  k.integrator = to_ig(c.integrator);
  k.qoi_kind = static_cast<QoIKind>(c.qoi_kind);
  k.qoi_a = c.qoi_a;
  k.qoi_b = c.qoi_b;
  k.qoi_r = c.qoi_r;
  k.qoi_delta = c.qoi_delta;
  k.qoi_bins = c.qoi_bins;
  k.T = c.T;
  k.m0 = c.m0;
  k.eps = c.eps;
  k.fixed_n = c.fixed_n;
  k.seed = c.seed;
  k.x0 = c.x0;
  k.u0 = c.u0;
  k.adaptive = c.adaptive != 0;
  k.x_adapt = c.x_adapt;
  k.coupling_signs = c.coupling_signs != 0;
  k.workers = c.workers;
  k.timings = c.timings != 0;
  k.output_dir = c.output_dir ? c.output_dir : ".";
  return k;
}

static RunResult to_res(const ablmc_run_result& r, int64_t dim) {
  RunResult o;
  for (int64_t i = 0; i < dim; ++i) {
    o.estimate.push_back(r.est_vec ? r.est_vec[i] : r.estimate);
    o.stat_error.push_back(r.err_vec ? r.err_vec[i] : r.stat_error);
  }
  o.bias_estimate = r.bias_estimate;
  o.alpha = r.alpha;
  o.c1 = r.c1;
  o.levels_used = r.levels_used;
  o.total_cost_steps = r.total_cost_steps;
  o.pilot_cost_steps = r.pilot_cost_steps;
  o.failed_samples = r.failed_samples;
  o.wall_seconds = r.wall_seconds;
  if (r.warnings_mask & 1)
    o.warnings.push_back("Var[Y_1] >= Var[Y_0]/2: coarsest level M_0 is too coarse to pay off");
  if (r.warnings_mask & 2) o.warnings.push_back("sample allocation did not converge in 64 rounds");
  for (int l = 0; l < r.n_levels; ++l) {
    LevelStats st;
    st.init(l, r.level_h[l], std::size_t(dim));
    for (int64_t i = 0; i < dim; ++i) {
      st.sum_y[i] = r.level_sum_y_vec ? r.level_sum_y_vec[l * dim + i] : r.level_sum_y[l];
      st.sum_y2[i] = r.level_sum_y2_vec ? r.level_sum_y2_vec[l * dim + i] : r.level_sum_y2[l];
    }
    st.n = r.level_n[l];
    st.failed = r.level_failed[l];
    st.cost_steps = r.level_cost[l];
    o.level_stats.push_back(std::move(st));
  }
  return o;
}

static int64_t emit(const std::string& s, char* buf, int64_t cap) {
  if (buf && cap > 0) {
    const std::size_t n = std::min<std::size_t>(s.size(), std::size_t(cap - 1));
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
  return int64_t(s.size());
}

// exactly what write_result_json (output.hpp:213-219) writes
int64_t ref_result_json(const ablmc_run_config* c, const ablmc_run_result* r, int64_t dim,
                        char* buf, int64_t cap) {
  OutputRecord rec;
  rec.config = to_cfg(*c);
  rec.result = to_res(*r, dim);
  return emit(to_json(rec).dump(2) + "\n", buf, cap);
}

// output_record_from_json (output.hpp:125-159) then to_json again: the
// reference's own read-back of a result.json; -1 on a reader exception.
int64_t ref_result_json_roundtrip(const char* text, char* buf, int64_t cap) {
  try {
    const OutputRecord rec = output_record_from_json(nlohmann::ordered_json::parse(text));
    return emit(to_json(rec).dump(2) + "\n", buf, cap);
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int64_t ref_variance_decay_csv(const ablmc_decay_row* rows, int n, char* buf, int64_t cap) {
  std::vector<DecayRow> v;
  for (int i = 0; i < n; ++i)
    v.push_back({rows[i].level, rows[i].h, rows[i].var_y, rows[i].mean_y, rows[i].se_mean,
                 rows[i].n, rows[i].cost_steps});
  return emit(variance_decay_csv(v), buf, cap);
}

int64_t ref_cost_sweep_csv(const ablmc_cost_row* rows, int n, int timings, char* buf,
                           int64_t cap) {
  std::vector<CostRow> v;
  for (int i = 0; i < n; ++i) {
    CostRow r;
    r.eps = rows[i].eps;
    r.method = rows[i].method == 0 ? Method::stmc : Method::mlmc;
    r.integrator = to_ig(rows[i].integrator);
    r.cost_steps = rows[i].cost_steps;
    r.wall_seconds = rows[i].wall_seconds;
    r.estimate = rows[i].estimate;
    r.stat_error = rows[i].stat_error;
    v.push_back(r);
  }
  return emit(cost_sweep_csv(v, timings != 0), buf, cap);
}

int64_t ref_pdf_csv(const double* edges, int n_edges, const double* conc, const double* se,
                    char* buf, int64_t cap) {
  return emit(pdf_csv(std::span<const double>(edges, std::size_t(n_edges)),
                      std::span<const double>(conc, std::size_t(n_edges - 1)),
                      std::span<const double>(se, std::size_t(n_edges - 1))),
              buf, cap);
}

int ref_cost_sweep(const ablmc_problem* prc, int method, const double* eps, int n_eps,
                   double alpha, double c1, int workers, ablmc_cost_row* rows) {
  return guarded([&] {
    const Problem pr = to_problem(*prc);
    BiasFit fit;
    fit.alpha = alpha;
    fit.c1 = c1;
    const auto rr = cost_sweep(pr, method == 0 ? Method::stmc : Method::mlmc,
                               std::span<const double>(eps, std::size_t(n_eps)), fit, workers);
    for (std::size_t i = 0; i < rr.size(); ++i) {
      rows[i].eps = rr[i].eps;
      rows[i].method = rr[i].method == Method::stmc ? 0 : 1;
      rows[i].integrator = static_cast<int32_t>(rr[i].integrator);
      rows[i].cost_steps = rr[i].cost_steps;
      rows[i].wall_seconds = rr[i].wall_seconds;
      rows[i].estimate = rr[i].estimate;
      rows[i].stat_error = rr[i].stat_error;
    }
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
