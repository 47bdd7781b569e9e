// drivers.cu — host MLMC/StMC drivers over the device level sampler.
//
// Same control flow and arithmetic as the reference drivers
// (estimators.hpp:100-431): fit_power_law, estimate_bias_constants,
// choose_levels, allocate_samples, run_stmc, run_mlmc, decay_sweep.  Every
// accumulate_samples call goes through ablmc_accumulate_samples /
// ablmc_accumulate_paths (the device path); the drivers stay on the host,
// as the north star asks.  Exceptions map to return codes (see ablmc_b200.h).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/ablmc_b200.h"
#include "capi_internal.h"

namespace {

using ablmc_host::set_error;

struct Stats {  // LevelStats (stats.hpp:26-88)
  int level = 0;
  double h = 0.0;
  int64_t dim = 1;
  std::vector<double> sum_y, sum_y2;
  int64_t n = 0, failed = 0, cost_steps = 0;

  void init(int l, double hh, int64_t d) {
    level = l;
    h = hh;
    dim = d;
    sum_y.assign(size_t(d), 0.0);
    sum_y2.assign(size_t(d), 0.0);
    n = failed = cost_steps = 0;
  }
  int64_t attempts() const { return n + failed; }
  double mean(size_t i = 0) const { return sum_y[i] / double(n); }
  double variance(size_t i = 0) const {
    if (n < 2) return 0.0;
    const double m = sum_y[i] / double(n);
    return std::max(0.0, (sum_y2[i] - double(n) * m * m) / double(n - 1));
  }
  double max_variance() const {
    double v = 0.0;
    for (size_t i = 0; i < size_t(dim); ++i) v = std::max(v, variance(i));
    return v;
  }
  double max_abs_mean() const {
    double m = 0.0;
    for (size_t i = 0; i < size_t(dim); ++i) m = std::max(m, std::abs(mean(i)));
    return m;
  }
  double std_error(size_t i = 0) const { return n > 0 ? std::sqrt(variance(i) / double(n)) : 0.0; }

  ablmc_level_stats view() {
    ablmc_level_stats v;
    std::memset(&v, 0, sizeof v);
    v.level = level;
    v.h = h;
    v.dim = dim;
    v.sum_y = sum_y.data();
    v.sum_y2 = sum_y2.data();
    v.n = n;
    v.failed = failed;
    v.cost_steps = cost_steps;
    return v;
  }
  void take(const ablmc_level_stats& v) {
    n = v.n;
    failed = v.failed;
    cost_steps = v.cost_steps;
  }
};

// accumulate_samples(st, first, count, *, sampler) + check_failure_budget.
int accumulate_level(const ablmc_problem* pr, Stats& st, int level, int64_t first, int64_t count) {
  ablmc_level_stats v = st.view();
  if (int rc = ablmc_accumulate_samples(pr, level, first, count, &v)) return rc;
  st.take(v);
  return ablmc_check_failure_budget(&v);
}

// Several levels at once: `ensure_level(l, n_target)` for each (level,
// target) in order, as one device batch (ablmc_accumulate_levels: one
// synchronisation, same bits as the sequential calls); failure budgets are
// checked afterwards in the same order.
int accumulate_levels(const ablmc_problem* pr, std::vector<Stats>& levels,
                      const std::vector<std::pair<int, int64_t>>& want) {
  std::vector<int> ls;
  std::vector<int64_t> firsts, counts;
  std::vector<ablmc_level_stats> views;
  std::vector<size_t> idx;
  views.reserve(want.size());
  for (const auto& w : want) {
    Stats& st = levels[size_t(w.first)];
    if (st.n >= w.second) continue;
    ls.push_back(w.first);
    firsts.push_back(st.attempts());
    counts.push_back(w.second - st.n);
    views.push_back(st.view());
    idx.push_back(size_t(w.first));
  }
  if (ls.empty()) return 0;
  std::vector<ablmc_level_stats*> ptrs;
  for (auto& v : views) ptrs.push_back(&v);
  if (int rc = ablmc_accumulate_levels(pr, int(ls.size()), ls.data(), firsts.data(),
                                       counts.data(), ptrs.data()))
    return rc;
  for (size_t q = 0; q < ls.size(); ++q) {
    levels[idx[q]].take(views[q]);
    if (int rc = ablmc_check_failure_budget(&views[q])) return rc;
  }
  return 0;
}

int accumulate_path(const ablmc_problem* pr, Stats& st, int64_t M, int64_t first, int64_t count) {
  ablmc_level_stats v = st.view();
  if (int rc = ablmc_accumulate_paths(pr, M, 0, first, count, &v)) return rc;
  st.take(v);
  return ablmc_check_failure_budget(&v);
}

struct PowerFit {
  double exponent = 0.0, log_prefactor = 0.0;
};

// estimators.hpp:107-123
int fit_power_law(const std::vector<double>& h, const std::vector<double>& v, PowerFit& out) {
  if (h.size() != v.size() || h.size() < 2) {
    set_error("fit_power_law: need at least two points");
    return ABLMC_ERR_INVALID_ARGUMENT;
  }
  double sx = 0, sy = 0, sxx = 0, sxy = 0;
  const double n = double(h.size());
  for (size_t i = 0; i < h.size(); ++i) {
    if (!(v[i] > 0.0)) {
      set_error("fit_power_law: values must be positive");
      return ABLMC_ERR_INVALID_ARGUMENT;
    }
    const double x = std::log(h[i]);
    const double y = std::log(v[i]);
    sx += x;
    sy += y;
    sxx += x * x;
    sxy += x * y;
  }
  const double slope = (n * sxy - sx * sy) / (n * sxx - sx * sx);
  out = {slope, (sy - slope * sx) / n};
  return 0;
}

struct BiasPoint {
  double h, mean_abs, std_err;
};
struct BiasFit {
  double alpha = 1.0, c1 = 0.0, c_y = 0.0;
};

// estimators.hpp:142-161; ABLMC_ERR_RUNTIME = the reference's runtime_error.
int estimate_bias_constants(const std::vector<BiasPoint>& pts, BiasFit& out) {
  if (pts.size() < 3) {
    set_error("estimate_bias_constants: need at least 3 levels");
    return ABLMC_ERR_INVALID_ARGUMENT;
  }
  std::vector<double> h, v;
  for (const auto& pt : pts) {
    if (!(pt.mean_abs > 3.0 * pt.std_err)) {
      set_error("estimate_bias_constants: E[Y_l] statistically indistinguishable from 0 at h = " +
                std::to_string(pt.h) + "; refine the pilot sample size");
      return ABLMC_ERR_RUNTIME;
    }
    h.push_back(pt.h);
    v.push_back(pt.mean_abs);
  }
  PowerFit f;
  if (int rc = fit_power_law(h, v, f)) return rc;
  out.alpha = f.exponent;
  out.c_y = std::exp(f.log_prefactor);
  out.c1 = out.c_y / (std::pow(2.0, out.alpha) - 1.0);
  return 0;
}

// estimators.hpp:164-175
int choose_levels(double alpha, double c1, double eps, int64_t m0, double T, int l_max, int& L) {
  if (!(alpha > 0.0) || !(c1 > 0.0) || !(eps > 0.0)) {
    set_error("choose_levels: alpha, c1, eps must be positive");
    return ABLMC_ERR_INVALID_ARGUMENT;
  }
  const double target = eps / 1.4142135623730951;
  for (int l = 0; l <= l_max; ++l) {
    const double h = T / double(m0 << l);
    if (c1 * std::pow(h, alpha) <= target) {
      L = l;
      return 0;
    }
  }
  set_error("choose_levels: bias target needs more than " + std::to_string(l_max) + " levels");
  return ABLMC_ERR_RUNTIME;
}

// estimators.hpp:180-191
std::vector<int64_t> allocate_samples(const std::vector<double>& var, const std::vector<double>& h,
                                      double eps) {
  double s = 0.0;
  for (size_t l = 0; l < h.size(); ++l) s += std::sqrt(var[l] / h[l]);
  std::vector<int64_t> n(var.size());
  for (size_t l = 0; l < h.size(); ++l)
    n[l] = int64_t(std::ceil(2.0 / (eps * eps) * std::sqrt(var[l] * h[l]) * s));
  return n;
}

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void fill_levels(const std::vector<Stats>& levels, ablmc_run_result* out) {
  out->n_levels = int(std::min<size_t>(levels.size(), ABLMC_MAX_LEVELS));
  for (size_t l = 0; l < levels.size() && l < ABLMC_MAX_LEVELS; ++l) {
    out->level_n[l] = levels[l].n;
    out->level_failed[l] = levels[l].failed;
    out->level_cost[l] = levels[l].cost_steps;
    out->level_h[l] = levels[l].h;
    out->level_sum_y[l] = levels[l].sum_y[0];
    out->level_sum_y2[l] = levels[l].sum_y2[0];
    const size_t d = size_t(levels[l].dim);
    for (size_t i = 0; i < d; ++i) {
      if (out->level_sum_y_vec) out->level_sum_y_vec[l * d + i] = levels[l].sum_y[i];
      if (out->level_sum_y2_vec) out->level_sum_y2_vec[l * d + i] = levels[l].sum_y2[i];
    }
  }
}

void clear_result(ablmc_run_result* out) {
  double* ev = out->est_vec;
  double* er = out->err_vec;
  double* sy = out->level_sum_y_vec;
  double* sy2 = out->level_sum_y2_vec;
  std::memset(out, 0, sizeof(*out));
  out->est_vec = ev;
  out->err_vec = er;
  out->level_sum_y_vec = sy;
  out->level_sum_y2_vec = sy2;
}

}  // namespace

extern "C" {

void ablmc_mlmc_options_defaults(ablmc_mlmc_options* o) {  // estimators.hpp:271-278
  std::memset(o, 0, sizeof(*o));
  o->pilot_n = 10000;
  o->pilot_levels_max = 4;
  o->init_n = 1000;
  o->l_max = 16;
}

// estimators.hpp:230-269
int ablmc_run_stmc(const ablmc_problem* pr, int64_t M_L, double eps, int64_t fixed_n,
                   ablmc_run_result* out) {
  if (int rc = ablmc_host::validate(pr)) return rc;
  if (M_L < 1) {
    set_error("run_stmc: M_L must be >= 1");
    return ABLMC_ERR_INVALID_ARGUMENT;
  }
  if (fixed_n <= 0 && !(eps > 0.0)) {
    set_error("run_stmc: need a tolerance or a fixed sample count");
    return ABLMC_ERR_INVALID_ARGUMENT;
  }
  if (int rc = ablmc_check_se_stability(pr, pr->T / double(M_L))) return rc;
  const double t0 = now_s();
  clear_result(out);
  Stats acc;
  const int64_t dim = ablmc_host::dim_of(pr);
  acc.init(0, pr->T / double(M_L), dim);
  if (fixed_n > 0) {
    if (int rc = accumulate_path(pr, acc, M_L, 0, fixed_n)) return rc;
  } else {
    if (int rc = accumulate_path(pr, acc, M_L, 0, 1000)) return rc;
    for (int round = 0; round < 64; ++round) {
      const double v = acc.max_variance();
      const int64_t needed = int64_t(std::ceil(2.0 * v / (eps * eps)));
      if (acc.n >= needed) break;
      if (int rc = accumulate_path(pr, acc, M_L, acc.attempts(), needed - acc.n)) return rc;
    }
  }
  out->levels_used = 0;
  out->estimate = acc.mean(0);
  out->stat_error = acc.std_error(0);
  for (int64_t i = 0; i < dim; ++i) {
    if (out->est_vec) out->est_vec[i] = acc.mean(size_t(i));
    if (out->err_vec) out->err_vec[i] = acc.std_error(size_t(i));
  }
  fill_levels({acc}, out);
  out->total_cost_steps = acc.cost_steps;
  out->failed_samples = acc.failed;
  out->wall_seconds = now_s() - t0;
  return 0;
}

// estimators.hpp:284-397
int ablmc_run_mlmc(const ablmc_problem* pr, double eps, const ablmc_mlmc_options* o_in,
                   ablmc_run_result* out) {
  if (int rc = ablmc_host::validate(pr)) return rc;
  if (!(eps > 0.0)) {
    set_error("run_mlmc: eps must be positive");
    return ABLMC_ERR_INVALID_ARGUMENT;
  }
  ablmc_mlmc_options o;
  if (o_in) o = *o_in;
  else ablmc_mlmc_options_defaults(&o);
  // ablmc_run_result holds ABLMC_MAX_LEVELS per-level rows (the reference's
  // vector is unbounded; its default l_max is 16): refuse what cannot be
  // reported instead of truncating
  if (o.l_max < 0 || o.l_max >= ABLMC_MAX_LEVELS || o.pilot_levels_max < 0 ||
      o.pilot_levels_max >= ABLMC_MAX_LEVELS) {
    set_error("run_mlmc: l_max and pilot_levels_max must be in [0, " +
              std::to_string(ABLMC_MAX_LEVELS - 1) + "]");
    return ABLMC_ERR_INVALID_ARGUMENT;
  }
  if (int rc = ablmc_check_se_stability(pr, pr->T / double(pr->m0))) return rc;
  const double t0 = now_s();
  clear_result(out);
  const int64_t dim = ablmc_host::dim_of(pr);
  std::vector<Stats> levels;

  auto ensure_level = [&](int l, int64_t n_target) -> int {
    while (int(levels.size()) <= l) {
      Stats st;
      const int nl = int(levels.size());
      st.init(nl, pr->T / double(pr->m0 << nl), dim);
      levels.push_back(std::move(st));
    }
    Stats& st = levels[size_t(l)];
    if (st.n < n_target) return accumulate_level(pr, st, l, st.attempts(), n_target - st.n);
    return 0;
  };

  auto bias_points = [&](int up_to) {
    std::vector<BiasPoint> pts;
    for (int l = 1; l <= up_to && l < int(levels.size()); ++l) {
      const Stats& st = levels[size_t(l)];
      size_t imax = 0;
      for (size_t i = 1; i < size_t(st.dim); ++i)
        if (std::abs(st.mean(i)) > std::abs(st.mean(imax))) imax = i;
      pts.push_back({st.h, st.max_abs_mean(), st.std_error(imax)});
    }
    return pts;
  };

  // the levels vector grown to hold level `l` (ensure_level's first half)
  auto have_level = [&](int l) {
    while (int(levels.size()) <= l) {
      Stats st;
      const int nl = int(levels.size());
      st.init(nl, pr->T / double(pr->m0 << nl), dim);
      levels.push_back(std::move(st));
    }
  };
  // ensure_level over several levels, as one device batch
  auto ensure_levels = [&](const std::vector<std::pair<int, int64_t>>& want) -> int {
    for (const auto& w : want) have_level(w.first);
    return accumulate_levels(pr, levels, want);
  };

  auto fit_with_refinement = [&](int up_to, BiasFit& fit) -> int {
    int64_t n = o.pilot_n;
    for (int attempt = 0;; ++attempt) {
      std::vector<std::pair<int, int64_t>> want;
      for (int l = 1; l <= up_to; ++l) want.push_back({l, n});
      if (int rc = ensure_levels(want)) return rc;
      const int rc = estimate_bias_constants(bias_points(up_to), fit);
      if (rc == 0) return 0;
      if (rc != ABLMC_ERR_RUNTIME || attempt >= 6) return rc;  // catch (runtime_error)
      n *= 4;
    }
  };

  BiasFit fit;
  int L = 0;
  if (int rc = ensure_level(0, o.pilot_n)) return rc;
  if (o.use_bias_fit) {
    fit.alpha = o.alpha;
    fit.c1 = o.c1;
    if (int rc = choose_levels(fit.alpha, fit.c1, eps, pr->m0, pr->T, o.l_max, L)) return rc;
  } else {
    if (int rc = fit_with_refinement(3, fit)) return rc;
    if (int rc = choose_levels(fit.alpha, fit.c1, eps, pr->m0, pr->T, o.l_max, L)) return rc;
    if (L > 3) {
      if (int rc = fit_with_refinement(std::min(L, int(o.pilot_levels_max)), fit)) return rc;
      if (int rc = choose_levels(fit.alpha, fit.c1, eps, pr->m0, pr->T, o.l_max, L)) return rc;
    }
  }
  {
    std::vector<std::pair<int, int64_t>> want;
    for (int l = 0; l <= L; ++l) want.push_back({l, o.init_n});
    if (int rc = ensure_levels(want)) return rc;
  }
  for (const auto& st : levels) out->pilot_cost_steps += st.cost_steps;

  int n_warn = 0, warn_mask = 0;
  if (L >= 1 && levels.size() > 1 && levels[1].max_variance() >= 0.5 * levels[0].max_variance()) {
    ++n_warn;
    warn_mask |= 1;
  }

  std::vector<double> v(size_t(L) + 1), hs(size_t(L) + 1);
  for (int round = 0; round < 64; ++round) {
    for (int l = 0; l <= L; ++l) {
      v[size_t(l)] = levels[size_t(l)].max_variance();
      hs[size_t(l)] = levels[size_t(l)].h;
    }
    const std::vector<int64_t> target = allocate_samples(v, hs, eps);
    std::vector<std::pair<int, int64_t>> want;
    for (int l = 0; l <= L; ++l)
      if (target[size_t(l)] > levels[size_t(l)].n) want.push_back({l, target[size_t(l)]});
    if (int rc = ensure_levels(want)) return rc;
    double stat2 = 0.0;
    for (int l = 0; l <= L; ++l)
      stat2 += levels[size_t(l)].max_variance() / double(levels[size_t(l)].n);
    if (stat2 <= 0.5 * eps * eps) break;
    if (round == 63) {
      ++n_warn;
      warn_mask |= 2;
    }
  }

  out->levels_used = L;
  out->alpha = fit.alpha;
  out->c1 = fit.c1;
  out->bias_estimate = fit.c1 * std::pow(pr->T / double(pr->m0 << L), fit.alpha);
  std::vector<double> est(size_t(dim), 0.0), err(size_t(dim), 0.0);
  for (int l = 0; l <= L; ++l) {
    const Stats& st = levels[size_t(l)];
    for (size_t i = 0; i < size_t(dim); ++i) {
      est[i] += st.mean(i);
      err[i] += st.variance(i) / double(st.n);
    }
  }
  for (auto& se : err) se = std::sqrt(se);
  out->estimate = est[0];
  out->stat_error = err[0];
  for (int64_t i = 0; i < dim; ++i) {
    if (out->est_vec) out->est_vec[i] = est[size_t(i)];
    if (out->err_vec) out->err_vec[i] = err[size_t(i)];
  }
  for (const auto& st : levels) {
    out->total_cost_steps += st.cost_steps;
    out->failed_samples += st.failed;
  }
  fill_levels(levels, out);
  out->n_warnings = n_warn;
  out->warnings_mask = warn_mask;
  out->wall_seconds = now_s() - t0;
  return 0;
}

// estimators.hpp:456-485: StMC picks M_L = m0 2^L from the bias fit so the
// discretisation error stays below eps/sqrt(2); MLMC reuses the fit.
int ablmc_cost_sweep(const ablmc_problem* pr, int method, const double* eps_values, int n_eps,
                     double alpha, double c1, ablmc_cost_row* rows) {
  if (int rc = ablmc_host::validate(pr)) return rc;
  for (int i = 0; i < n_eps; ++i) {
    const double eps = eps_values[i];
    ablmc_cost_row& row = rows[i];
    std::memset(&row, 0, sizeof row);
    row.eps = eps;
    row.method = method;
    row.integrator = pr->integrator;
    ablmc_run_result r;
    std::memset(&r, 0, sizeof r);
    if (method == 0) {
      int L = 0;
      if (int rc = choose_levels(alpha, c1, eps, pr->m0, pr->T, 16, L)) return rc;
      if (int rc = ablmc_run_stmc(pr, pr->m0 << L, eps, 0, &r)) return rc;
      row.cost_steps = r.total_cost_steps;
    } else {
      ablmc_mlmc_options o;
      ablmc_mlmc_options_defaults(&o);
      o.use_bias_fit = 1;
      o.alpha = alpha;
      o.c1 = c1;
      if (int rc = ablmc_run_mlmc(pr, eps, &o, &r)) return rc;
      row.cost_steps = r.total_cost_steps - r.pilot_cost_steps;
    }
    row.wall_seconds = r.wall_seconds;
    row.estimate = r.estimate;
    row.stat_error = r.stat_error;
  }
  return 0;
}

int ablmc_fit_power_law(const double* h, const double* v, int n, double* exponent,
                        double* log_prefactor) {
  if (!h || !v || !exponent || !log_prefactor || n < 0) {
    set_error("fit_power_law: null argument");
    return ABLMC_ERR_INVALID_ARGUMENT;
  }
  PowerFit f;
  if (int rc = fit_power_law(std::vector<double>(h, h + n), std::vector<double>(v, v + n), f))
    return rc;
  *exponent = f.exponent;
  *log_prefactor = f.log_prefactor;
  return 0;
}

int ablmc_estimate_bias_constants(const double* h, const double* mean_abs, const double* std_err,
                                  int n, double* alpha, double* c1, double* c_y) {
  if (!h || !mean_abs || !std_err || !alpha || !c1 || !c_y || n < 0) {
    set_error("estimate_bias_constants: null argument");
    return ABLMC_ERR_INVALID_ARGUMENT;
  }
  std::vector<BiasPoint> pts;
  for (int i = 0; i < n; ++i) pts.push_back({h[i], mean_abs[i], std_err[i]});
  BiasFit f;
  if (int rc = estimate_bias_constants(pts, f)) return rc;
  *alpha = f.alpha;
  *c1 = f.c1;
  *c_y = f.c_y;
  return 0;
}

int ablmc_choose_levels(double alpha, double c1, double eps, int64_t m0, double T, int l_max,
                        int* L) {
  if (!L) {
    set_error("choose_levels: null argument");
    return ABLMC_ERR_INVALID_ARGUMENT;
  }
  return choose_levels(alpha, c1, eps, m0, T, l_max, *L);
}

int ablmc_allocate_samples(const double* var, const double* h, int n_levels, double eps,
                           int64_t* n_out) {
  if (!var || !h || !n_out || n_levels < 0) {
    set_error("allocate_samples: null argument");
    return ABLMC_ERR_INVALID_ARGUMENT;
  }
  const std::vector<int64_t> n = allocate_samples(std::vector<double>(var, var + n_levels),
                                                  std::vector<double>(h, h + n_levels), eps);
  for (int l = 0; l < n_levels; ++l) n_out[l] = n[size_t(l)];
  return 0;
}

// estimators.hpp:415-431
int ablmc_decay_sweep(const ablmc_problem* pr, int l_min, int l_max, int64_t n_per_level,
                      ablmc_decay_row* rows) {
  if (int rc = ablmc_host::validate(pr)) return rc;
  if (int rc = ablmc_check_se_stability(pr, pr->T / double(pr->m0))) return rc;
  const int64_t dim = ablmc_host::dim_of(pr);
  if (l_min < 0 || l_max < l_min) {
    set_error("decay_sweep: need 0 <= l_min <= l_max");
    return ABLMC_ERR_INVALID_ARGUMENT;
  }
  std::vector<Stats> levels(size_t(l_max) + 1);
  std::vector<std::pair<int, int64_t>> want;
  for (int l = l_min; l <= l_max; ++l) {
    levels[size_t(l)].init(l, pr->T / double(pr->m0 << l), dim);
    want.push_back({l, n_per_level});
  }
  if (int rc = accumulate_levels(pr, levels, want)) return rc;  // one device batch
  for (int l = l_min; l <= l_max; ++l) {
    const Stats& st = levels[size_t(l)];
    size_t imax = 0;
    for (size_t i = 1; i < size_t(dim); ++i)
      if (st.variance(i) > st.variance(imax)) imax = i;
    ablmc_decay_row& r = rows[l - l_min];
    std::memset(&r, 0, sizeof r);
    r.level = l;
    r.h = st.h;
    r.var_y = st.variance(imax);
    r.mean_y = st.mean(imax);
    r.se_mean = st.std_error(imax);
    r.n = st.n;
    r.cost_steps = st.cost_steps;
  }
  return 0;
}

}  // extern "C"
