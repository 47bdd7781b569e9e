// output.cpp — driver-facing formats: result.json
// schema v1 and the CSV tables, byte-identical to the reference's
// output.hpp:17-225 (same key order and types through nlohmann::ordered_json,
// dump(2) + "\n"; CSV floats "%.17g").  Host-only C++.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <stdexcept>
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

int method_from(const std::string& v) {  // estimators.hpp:165-172
  if (v == "stmc") return 0;
  if (v == "mlmc") return 1;
  throw std::invalid_argument("unknown method '" + v + "'");
}
int integrator_from(const std::string& v) {  // integrators.hpp:14-21
  if (v == "se") return ABLMC_SE;
  if (v == "gl") return ABLMC_GL;
  if (v == "baoab") return ABLMC_BAOAB;
  throw std::invalid_argument("unknown integrator '" + v + "'");
}
int qoi_from(const std::string& v) {  // qoi.hpp:96-104
  for (int k = ABLMC_QOI_MEAN_POSITION; k <= ABLMC_QOI_BINNED_FIELD; ++k)
    if (v == qoi_name(k)) return k;
  throw std::invalid_argument("unknown qoi kind '" + v + "'");
}

thread_local std::string g_read_error;

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

// output.hpp:47-81 (config_from_json) + 125-159 (output_record_from_json)
int ablmc_read_result_json(const char* text, ablmc_run_config* cfg, ablmc_run_result* out,
                           int64_t* dim, char* output_dir, int64_t cap) {
  if (!text) return ABLMC_ERR_INVALID_ARGUMENT;
  try {
    const json j = json::parse(text);
    const int schema = j.at("schema_version");
    if (schema != 1)
      throw std::runtime_error("result file has schema version " + std::to_string(schema) +
                               ", this reader expects 1");
    const auto& res = j.at("result");
    const auto est = res.at("estimate").get<std::vector<double>>();
    const int64_t d = int64_t(est.size());
    if (dim) *dim = d;
    const auto& jc = j.at("config");
    const std::string dir = jc.at("output").at("dir").get<std::string>();
    ablmc_run_config local;
    if (!cfg) cfg = &local;  // parsed (and so validated) either way
    {
      ablmc_run_config_defaults(cfg);
      const auto& m = jc.at("model");
      cfg->model = {m.at("kappa_sigma"), m.at("kappa_tau"), m.at("u_star"), m.at("h"),
                    m.at("eps_reg"),     m.at("x_ref"),     m.at("noise_scale")};
      const auto& r = jc.at("run");
      cfg->method = method_from(r.at("method").get<std::string>());
      cfg->integrator = integrator_from(r.at("integrator").get<std::string>());
      cfg->T = r.at("t");
      cfg->m0 = r.at("m0");
      cfg->eps = r.at("eps");
      cfg->fixed_n = r.at("n_samples");
      cfg->seed = r.at("seed");
      cfg->x0 = r.at("x0");
      cfg->u0 = r.at("u0");
      cfg->adaptive = r.at("adaptive").get<bool>() ? 1 : 0;
      cfg->x_adapt = r.at("x_adapt");
      cfg->coupling_signs = r.at("coupling_signs").get<bool>() ? 1 : 0;
      cfg->workers = r.at("workers");
      cfg->timings = r.at("timings").get<bool>() ? 1 : 0;
      const auto& q = jc.at("qoi");
      cfg->qoi_kind = qoi_from(q.at("kind").get<std::string>());
      cfg->qoi_a = q.at("a");
      cfg->qoi_b = q.at("b");
      cfg->qoi_r = q.at("r");
      cfg->qoi_delta = q.at("delta");
      cfg->qoi_bins = q.at("bins");
      cfg->output_dir = output_dir;
    }
    if (output_dir && cap > 0) emit(dir, output_dir, cap);
    ablmc_run_result local_out;
    if (!out) {
      std::memset(&local_out, 0, sizeof local_out);
      out = &local_out;  // parsed (and so validated) either way
    }
    {
      const auto err = res.at("stat_error").get<std::vector<double>>();
      out->estimate = d > 0 ? est[0] : 0.0;
      out->stat_error = err.empty() ? 0.0 : err[0];
      if (out->est_vec) std::copy(est.begin(), est.end(), out->est_vec);
      if (out->err_vec) std::copy(err.begin(), err.end(), out->err_vec);
      out->bias_estimate = res.at("bias_estimate");
      out->alpha = res.at("alpha");
      out->c1 = res.at("c1");
      out->levels_used = res.at("levels_used");
      out->total_cost_steps = res.at("total_cost_steps");
      out->pilot_cost_steps = res.at("pilot_cost_steps");
      out->failed_samples = res.at("failed_samples");
      out->warnings_mask = 0;
      out->n_warnings = 0;
      for (const auto& w : res.at("warnings")) {
        const std::string ws = w.get<std::string>();
        if (ws.rfind("Var[Y_1] >= Var[Y_0]/2", 0) == 0) out->warnings_mask |= 1;
        else if (ws.rfind("sample allocation did not converge", 0) == 0) out->warnings_mask |= 2;
        else throw std::invalid_argument("unknown warning '" + ws + "'");
        ++out->n_warnings;
      }
      const auto& levels = res.at("levels");
      if (levels.size() > size_t(ABLMC_MAX_LEVELS))
        throw std::invalid_argument("more levels than ABLMC_MAX_LEVELS");
      out->n_levels = int(levels.size());
      int l = 0;
      for (const auto& lv : levels) {
        out->level_h[l] = lv.at("h");
        out->level_n[l] = lv.at("n");
        out->level_failed[l] = lv.at("failed");
        out->level_cost[l] = lv.at("cost_steps");
        const auto sy = lv.at("sum_y").get<std::vector<double>>();
        const auto sy2 = lv.at("sum_y2").get<std::vector<double>>();
        if (int64_t(sy.size()) != d || int64_t(sy2.size()) != d)
          throw std::invalid_argument("level sums do not match the estimate's dimension");
        out->level_sum_y[l] = sy[0];
        out->level_sum_y2[l] = sy2[0];
        if (out->level_sum_y_vec) std::copy(sy.begin(), sy.end(), out->level_sum_y_vec + l * d);
        if (out->level_sum_y2_vec) std::copy(sy2.begin(), sy2.end(), out->level_sum_y2_vec + l * d);
        ++l;
      }
      out->wall_seconds = j.at("timings").at("wall_seconds");
    }
    return 0;
  } catch (const std::runtime_error& e) {
    g_read_error = e.what();
    return ABLMC_ERR_RUNTIME;
  } catch (const std::exception& e) {
    g_read_error = e.what();
    return ABLMC_ERR_INVALID_ARGUMENT;
  }
}

const char* ablmc_read_result_json_error(void) { return g_read_error.c_str(); }

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
