// output.cpp — driver-facing formats: result.json
// schema v1 and the CSV tables, byte-identical to the reference's
// output.hpp:17-225 (same key order and types through nlohmann::ordered_json,
// dump(2) + "\n"; CSV floats "%.17g").  Host-only C++.
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <json.hpp>

#include "../../include/ablmc_b200.h"

namespace {

using json = nlohmann::ordered_json;

const char* method_name(int m) { return m == 0 ? "stmc" : "mlmc"; }          // estimators.hpp:165
const char* integrator_name(int ig) {                                         // integrators.hpp:14-21
  return ig == ABLMC_SE ? "se" : ig == ABLMC_GL ? "gl" : ig == ABLMC_BAOAB ? "baoab" : "?";
}
const char* qoi_name(int k) {                                                 // qoi.hpp:96-104
  switch (k) {
    case ABLMC_QOI_MEAN_POSITION: return "mean-position";
    case ABLMC_QOI_SMOOTHED_INDICATOR: return "smoothed-indicator";
    case ABLMC_QOI_RAW_INDICATOR: return "raw-indicator";
    case ABLMC_QOI_BINNED_FIELD: return "binned-field";
  }
  return "?";
}

// output.hpp:21-45
json config_json(const ablmc_run_config& c) {
  json j;
  j["model"] = {{"kappa_sigma", c.model.kappa_sigma}, {"kappa_tau", c.model.kappa_tau},
                {"u_star", c.model.u_star},           {"h", c.model.H},
                {"eps_reg", c.model.eps_reg},         {"x_ref", c.model.x_ref},
                {"noise_scale", c.model.noise_scale}};
  j["run"] = {{"method", method_name(c.method)},
              {"integrator", integrator_name(c.integrator)},
              {"t", c.T},
              {"m0", c.m0},
              {"eps", c.eps},
              {"n_samples", c.fixed_n},
              {"seed", c.seed},
              {"x0", c.x0},
              {"u0", c.u0},
              {"adaptive", c.adaptive != 0},
              {"x_adapt", c.x_adapt},
              {"coupling_signs", c.coupling_signs != 0},
              {"workers", int(c.workers)},
              {"timings", c.timings != 0}};
  j["qoi"] = {{"kind", qoi_name(c.qoi_kind)}, {"a", c.qoi_a}, {"b", c.qoi_b},
              {"r", int(c.qoi_r)},            {"delta", c.qoi_delta}, {"bins", int(c.qoi_bins)}};
  j["output"] = {{"dir", std::string(c.output_dir ? c.output_dir : ".")}};
  return j;
}

std::vector<double> vec(const double* p, int64_t n) { return std::vector<double>(p, p + n); }

// output.hpp:91-123
json record_json(const ablmc_run_config& c, const ablmc_run_result& r, int64_t dim) {
  json j;
  j["schema_version"] = 1;
  j["config"] = config_json(c);
  json res;
  res["estimate"] = r.est_vec ? vec(r.est_vec, dim) : std::vector<double>{r.estimate};
  res["stat_error"] = r.err_vec ? vec(r.err_vec, dim) : std::vector<double>{r.stat_error};
  res["bias_estimate"] = r.bias_estimate;
  res["alpha"] = r.alpha;
  res["c1"] = r.c1;
  res["levels_used"] = int(r.levels_used);
  res["total_cost_steps"] = r.total_cost_steps;
  res["pilot_cost_steps"] = r.pilot_cost_steps;
  res["failed_samples"] = r.failed_samples;
  std::vector<std::string> warnings;  // estimators.hpp:352-355,372-373, in emission order
  if (r.warnings_mask & 1)
    warnings.push_back("Var[Y_1] >= Var[Y_0]/2: coarsest level M_0 is too coarse to pay off");
  if (r.warnings_mask & 2) warnings.push_back("sample allocation did not converge in 64 rounds");
  res["warnings"] = warnings;
  json levels = json::array();
  for (int l = 0; l < r.n_levels && l < ABLMC_MAX_LEVELS; ++l) {
    json lv;
    lv["level"] = l;
    lv["h"] = r.level_h[l];
    lv["n"] = r.level_n[l];
    lv["failed"] = r.level_failed[l];
    lv["cost_steps"] = r.level_cost[l];
    lv["sum_y"] = r.level_sum_y_vec ? vec(r.level_sum_y_vec + l * dim, dim)
                                    : std::vector<double>{r.level_sum_y[l]};
    lv["sum_y2"] = r.level_sum_y2_vec ? vec(r.level_sum_y2_vec + l * dim, dim)
                                      : std::vector<double>{r.level_sum_y2[l]};
    levels.push_back(std::move(lv));
  }
  res["levels"] = std::move(levels);
  j["result"] = std::move(res);
  j["timings"] = {{"wall_seconds", c.timings ? r.wall_seconds : 0.0}};
  return j;
}

std::string fmt(double v) {  // output.hpp:169-173
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

int64_t emit(const std::string& s, char* buf, int64_t cap) {
  if (buf && cap > 0) {
    const size_t n = std::min<size_t>(s.size(), size_t(cap - 1));
    std::memcpy(buf, s.data(), n);
    buf[n] = '\0';
  }
  return int64_t(s.size());
}

}  // namespace

extern "C" {

void ablmc_run_config_defaults(ablmc_run_config* c) {  // config.hpp:18-40
  std::memset(c, 0, sizeof(*c));
  c->model = {1.3, 0.5, 0.2, 1.0, 0.01, 1.0, 1.0};
  c->method = 1;
  c->integrator = ABLMC_GL;
  c->qoi_kind = ABLMC_QOI_MEAN_POSITION;
  c->qoi_a = 0.1055;
  c->qoi_b = 0.1555;
  c->qoi_r = 4;
  c->qoi_delta = 0.1;
  c->qoi_bins = 20;
  c->T = 1.0;
  c->m0 = 40;
  c->eps = 1e-3;
  c->seed = 12345;
  c->x0 = 0.05;
  c->u0 = 0.1;
  c->x_adapt = 0.05;
  c->coupling_signs = 1;
  c->workers = 1;
  c->timings = 1;
  c->output_dir = ".";
}

int64_t ablmc_result_json(const ablmc_run_config* c, const ablmc_run_result* r, int64_t dim,
                          char* buf, int64_t cap) {
  if (!c || !r || dim < 1) return -1;
  try {
    return emit(record_json(*c, *r, dim).dump(2) + "\n", buf, cap);
  } catch (...) {
    return -1;
  }
}

int64_t ablmc_variance_decay_csv(const ablmc_decay_row* rows, int n, char* buf, int64_t cap) {
  std::string s = "level,h,var_Y,mean_Y,n_samples,cost_steps\n";  // output.hpp:184-191
  for (int i = 0; i < n; ++i) {
    const ablmc_decay_row& r = rows[i];
    s += std::to_string(r.level) + "," + fmt(r.h) + "," + fmt(r.var_y) + "," + fmt(r.mean_y) +
         "," + std::to_string(r.n) + "," + std::to_string(r.cost_steps) + "\n";
  }
  return emit(s, buf, cap);
}

int64_t ablmc_cost_sweep_csv(const ablmc_cost_row* rows, int n, int timings, char* buf,
                             int64_t cap) {
  std::string s = "eps,method,integrator,cost_steps,wall_seconds,estimate,stat_error\n";
  for (int i = 0; i < n; ++i) {  // output.hpp:193-200
    const ablmc_cost_row& r = rows[i];
    s += fmt(r.eps) + "," + method_name(r.method) + "," + integrator_name(r.integrator) + "," +
         std::to_string(r.cost_steps) + "," + fmt(timings ? r.wall_seconds : 0.0) + "," +
         fmt(r.estimate) + "," + fmt(r.stat_error) + "\n";
  }
  return emit(s, buf, cap);
}

int64_t ablmc_pdf_csv(const double* edges, int n_edges, const double* concentration,
                      const double* std_error, char* buf, int64_t cap) {
  std::string s = "bin_lo,bin_hi,concentration,std_error\n";  // output.hpp:202-209
  for (int i = 0; i + 1 < n_edges; ++i)
    s += fmt(edges[i]) + "," + fmt(edges[i + 1]) + "," + fmt(concentration[i]) + "," +
         fmt(std_error[i]) + "\n";
  return emit(s, buf, cap);
}

}  // extern "C"
