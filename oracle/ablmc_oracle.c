/*
 * ablmc_oracle.c — CPU restatement of the reference's coupled level sampler.
 *
 * TEST INFRASTRUCTURE ONLY (see ablmc_oracle.h): the checker, never the
 * thing measured or shipped.  Every function cites the reference file:line
 * (under /root/reference/proj/include/ablmc/) it restates.  Expression order
 * follows the reference exactly; build with -ffp-contract=off.
 */
#include "ablmc_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ORC_PI 3.141592653589793238462643383279502884
#define ORC_SQRT2 1.414213562373095048801688724209698079

/* noise.hpp:14-27 — Philox4x32-10. */
void orc_philox4x32(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int round = 0; round < 10; ++round) {
    const uint64_t p0 = (uint64_t)M0 * c0;
    const uint64_t p1 = (uint64_t)M1 * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    const uint32_t n1 = (uint32_t)p1;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    const uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += W0;
    k1 += W1;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* noise.hpp:29-34 */
uint64_t orc_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* noise.hpp:51-55 — key = splitmix64(splitmix64(seed) ^ level). */
void orc_stream_key(uint64_t seed, uint32_t level, uint32_t key[2]) {
  const uint64_t k = orc_splitmix64(orc_splitmix64(seed) ^ (uint64_t)level);
  key[0] = (uint32_t)k;
  key[1] = (uint32_t)(k >> 32);
}

/* noise.hpp:37-40 */
double orc_bits_to_unit(uint32_t hi, uint32_t lo) {
  const uint64_t b = ((uint64_t)hi << 32) | lo;
  return ((double)(b >> 11) + 0.5) * 0x1.0p-53;
}


/* ---------------------------------------------------- device-math mode
 * NOT the reference: a restatement of this project's device elementary
 * functions (paper_1612_07717_b200/csrc/ablmc_device.cuh log_unit_tab,
 * sincos_2pi, expm1_exp_core and the expm1(2x) = em1 (em1 + 2) identity),
 * with the same explicit FMAs, so tests can drive the oracle with the
 * device's exact log/sin/cos/exp/expm1 and require bit-identical paths for
 * every integrator.  The reference's own math (glibc) stays the default. */
static __thread int g_devmath = 0;
void orc_set_device_math(int on) { g_devmath = on; }
/* diagnostics: the largest pending-sub-interval count of the last adaptive pair */
static __thread int g_max_pending;
int orc_last_max_pending(void) { return g_max_pending; }

static uint64_t dbits(double v) { uint64_t b; memcpy(&b, &v, 8); return b; }
static double bitsd(uint64_t b) { double v; memcpy(&v, &b, 8); return v; }
static int lo_int(double v) { return (int)(int32_t)(uint32_t)dbits(v); }

static const double kS[6] = {-1.66666666666666324348e-01, 8.33333333332248946124e-03,
                             -1.98412698298579493134e-04, 2.75573137070700676789e-06,
                             -2.50507602534068634195e-08, 1.58969099521155010221e-10};
static const double kC[6] = {4.16666666666666019037e-02, -1.38888888888741095749e-03,
                             2.48015872894767294178e-05, -2.75573143513906633035e-07,
                             2.08757232129817482790e-09, -1.13596475577881948265e-11};
static const double kBm[6] = {6.93147180369123816490e-01, 1.90821492927058770002e-10,
                              6.36619772367581382433e-01, 1.57079632673412561417e+00,
                              6.07710050650619224932e-11, 6755399441055744.0};
static const double kEP[12] = {1.0 / 2, 1.0 / 6, 1.0 / 24, 1.0 / 120, 1.0 / 720, 1.0 / 5040,
                               1.0 / 40320, 1.0 / 362880, 1.0 / 3628800, 1.0 / 39916800,
                               1.0 / 479001600, 1.0 / 6227020800.0};
static const double kER[4] = {1.44269504088896338700e+00, 6.93147180369123816490e-01,
                              1.90821492927058770002e-10, 6755399441055744.0};

/* device log_unit_tab: Tang's table method (see ablmc_device.cuh), the same
 * table built by the same code as the library's upload_log_table */
static double dm_invc[256], dm_thi[256], dm_tlo[256];
static int dm_tab_built = 0;
static void dm_build_log_table(void) {
  for (int j = 0; j < 256; ++j) {
    const int e = j >> 7, b = j & 0x7f;
    const double lo = (e ? 1.0 : 0.5) * (1.0 + b / 128.0);
    const double hi = (e ? 1.0 : 0.5) * (1.0 + (b + 1) / 128.0);
    double c = 0.5 * (lo + hi);
    if (lo == 1.0 || hi == 1.0) c = 1.0;
    const double invc = (c == 1.0) ? 1.0 : 1.0 / c;
    const long double L = -logl((long double)invc);
    const double th = (double)L;
    dm_invc[j] = invc;
    dm_thi[j] = th;
    dm_tlo[j] = (double)(L - (long double)th);
  }
  dm_tab_built = 1;
}
static const double kQ[7] = {-1.0 / 2, 1.0 / 3, -1.0 / 4, 1.0 / 5, -1.0 / 6, 1.0 / 7, -1.0 / 8};

static double dm_log_unit(double u) {
  if (!dm_tab_built) dm_build_log_table();
  const uint64_t b = dbits(u);
  int32_t hx = (int32_t)(b >> 32);
  int k = (hx >> 20) - 1023;
  hx &= 0x000fffff;
  const int i = (hx + 0x95f64) & 0x100000;
  const int32_t mhi = hx | (i ^ 0x3ff00000);
  const double mnt = bitsd(((uint64_t)(uint32_t)mhi << 32) | (uint32_t)b);
  k += i >> 20;
  const int j = ((mhi >> 13) & 0x7f) | ((mhi >> 13) & 0x80);
  const double r = fma(mnt, dm_invc[j], -1.0);
  const double r2 = r * r;
  double q = kQ[6];
  for (int t = 5; t >= 0; --t) q = fma(q, r, kQ[t]);
  const double dk = (double)k;
  const double hi = fma(dk, kBm[0], dm_thi[j]);
  const double lo = fma(dk, kBm[1], dm_tlo[j]);
  return hi + (r + fma(r2, q, lo));
}

static void dm_sincos_2pi(double th, double* sn, double* cs) {
  const double t = fma(th, kBm[2], kBm[5]);
  const int q = lo_int(t);
  const double kd = t - kBm[5];
  double r = fma(-kd, kBm[3], th);
  r = fma(-kd, kBm[4], r);
  const double z = r * r;
  const double v = z * r;
  const double ps = fma(z, fma(z, fma(z, fma(z, kS[5], kS[4]), kS[3]), kS[2]), kS[1]);
  const double s = fma(v, fma(z, ps, kS[0]), r);
  const double pc = z * fma(z, fma(z, fma(z, fma(z, fma(z, kC[5], kC[4]), kC[3]), kC[2]), kC[1]),
                            kC[0]);
  const double hz = 0.5 * z;
  const double w = 1.0 - hz;
  const double c = w + fma(z, pc, (1.0 - w) - hz);
  const int swap = q & 1;
  const double s0 = swap ? c : s, c0 = swap ? s : c;
  *sn = (q & 2) ? -s0 : s0;
  *cs = ((q + 1) & 2) ? -c0 : c0;
}

/* exp(x), expm1(x) for x = -lam h (device ou_exp; libm below -700) */
static void dm_expm1_exp(double x, double* em1, double* ex) {
  if (!(x >= -700.0)) {
    *em1 = expm1(x);
    *ex = exp(x);
    return;
  }
  const double t = fma(x, kER[0], kER[3]);
  const int k = lo_int(t);
  const double kd = t - kER[3];
  double r = fma(-kd, kER[1], x);
  r = fma(-kd, kER[2], r);
  double q = kEP[11];
  for (int i = 10; i >= 0; --i) q = fma(q, r, kEP[i]);
  const double P = fma(r * r, q, r);
  const double s = bitsd((uint64_t)(uint32_t)((k + 1023) << 20) << 32);
  *em1 = fma(s, P, s - 1.0);
  *ex = fma(s, P, s);
}

/* exp(-lam h) (integrators.hpp:31-33), either math */
static double orc_exp_neg(double lam, double h) {
  if (!g_devmath) return exp(-lam * h);
  double em1, ex;
  dm_expm1_exp(-lam * h, &em1, &ex);
  return ex;
}

/* noise.hpp:60-75 — Box-Muller pair of block k>>1; cos for even k, sin for odd. */
double orc_normal_at(uint64_t seed, uint32_t level, uint64_t idx, uint64_t k) {
  uint32_t key[2];
  orc_stream_key(seed, level, key);
  const uint64_t block = k >> 1;
  const uint32_t ctr[4] = {(uint32_t)block, (uint32_t)(block >> 32), (uint32_t)idx,
                           (uint32_t)(idx >> 32)};
  uint32_t w[4];
  orc_philox4x32(ctr, key, w);
  const double u1 = orc_bits_to_unit(w[0], w[1]);
  const double u2 = orc_bits_to_unit(w[2], w[3]);
  const double r = sqrt(-2.0 * (g_devmath ? dm_log_unit(u1) : log(u1)));
  const double th = 2.0 * ORC_PI * u2;
  if (g_devmath) {
    double sn, cs;
    dm_sincos_2pi(th, &sn, &cs);
    return (k & 1) ? r * sn : r * cs;
  }
  return (k & 1) ? r * sin(th) : r * cos(th);
}

/* noise.hpp:91-94 */
double orc_coarse_noise_se(double xi0, double xi1, int s0, int s1, int sc) {
  return sc * (s0 * xi0 + s1 * xi1) / ORC_SQRT2;
}

/* noise.hpp:100-104 */
double orc_coarse_noise_gl(double xi0, double xi1, double lam, double h, int s0, int s1,
                           int sc) {
  const double e = orc_exp_neg(lam, h);
  return sc * (e * (s0 * xi0) + s1 * xi1) / sqrt(e * e + 1.0);
}

/* model.hpp:60-62 (std::clamp semantics: v<lo ? lo : hi<v ? hi : v) */
static double clamp_height(double x, const ablmc_model_params* p) {
  const double lo = p->eps_reg, hi = p->H - p->eps_reg;
  return (x < lo) ? lo : (hi < x) ? hi : x;
}

/* Extension profiles (NOT in the reference; BASELINE.json configs 1-5 as
 * written): restated from this project's definition in
 * paper_1612_07717_b200/csrc/ablmc_device.cuh coeffs<PROF>, so the device
 * extension paths have a checker.  Selected per thread by orc_set_profile
 * (orc_accumulate_* set it from the problem). */
typedef struct {
  int profile; /* ABLMC_PROFILE_* */
  double const_sigma_u, const_tau, sigma_floor, tau_min, tau_max;
} orc_profile;
static __thread orc_profile g_prof = {0, 0, 0, 0, 0, 0};

void orc_set_profile(int profile, double const_sigma_u, double const_tau, double sigma_floor,
                     double tau_min, double tau_max) {
  g_prof.profile = profile;
  g_prof.const_sigma_u = const_sigma_u;
  g_prof.const_tau = const_tau;
  g_prof.sigma_floor = sigma_floor;
  g_prof.tau_min = tau_min;
  g_prof.tau_max = tau_max;
}

static orc_coeffs ext_coeffs(double x, const ablmc_model_params* p) {
  orc_coeffs c;
  if (g_prof.profile == ABLMC_PROFILE_CONSTANT) { /* D1: homogeneous OU */
    const double su2 = g_prof.const_sigma_u * g_prof.const_sigma_u;
    const double lam = 1.0 / g_prof.const_tau;
    c.sigma_u2 = su2;
    c.lambda = lam;
    c.sigma = p->noise_scale * sqrt(2.0 * su2 * lam);
    c.dsigma_u2 = 0.0;
    return c;
  }
  /* D3: sigma_U floored, tau = kappa_tau x / sigma_U clamped to [tau_min, tau_max] */
  const double xc = fmin(fmax(x, 0.0), p->H);
  const double t = 1.0 - xc / p->H;
  const double st = sqrt(t);
  const double su_raw = (p->kappa_sigma * p->u_star) * sqrt(t * st);
  const int floored = !(su_raw > g_prof.sigma_floor);
  const double su = floored ? g_prof.sigma_floor : su_raw;
  double tau = (p->kappa_tau * xc) / su;
  tau = fmin(fmax(tau, g_prof.tau_min), g_prof.tau_max);
  const double a = p->kappa_sigma * p->u_star;
  c.sigma_u2 = su * su;
  c.lambda = 1.0 / tau;
  c.sigma = p->noise_scale * sqrt(2.0 * c.sigma_u2 * c.lambda);
  c.dsigma_u2 = floored ? 0.0 : (-1.5 * a * a * st) / p->H;
  return c;
}

/* model.hpp:73-89 */
orc_coeffs orc_sde_coeffs(double x, const ablmc_model_params* p) {
  if (g_prof.profile != ABLMC_PROFILE_REFERENCE) return ext_coeffs(x, p);
  const double xc = clamp_height(x, p);
  const double a = p->kappa_sigma * p->u_star;
  const double t = 1.0 - xc / p->H;
  const double st = sqrt(t);
  const double sigma_u2 = a * a * t * st;
  const double sigma_u = a * sqrt(t * st);
  const double lambda = sigma_u / (p->kappa_tau * xc);
  orc_coeffs c;
  c.sigma_u2 = sigma_u2;
  c.lambda = lambda;
  c.sigma = p->noise_scale * sqrt(2.0 * sigma_u2 * lambda);
  c.dsigma_u2 = (x < p->eps_reg || x > p->H - p->eps_reg) ? 0.0 : -1.5 * a * a * st / p->H;
  return c;
}

/* model.hpp:116-118 */
double orc_dv_dx(const orc_coeffs* c, double u) {
  return -0.5 * (1.0 + u * u / c->sigma_u2) * c->dsigma_u2;
}

/* particle.hpp:36-49 */
int orc_reflect(double* x, double* u, double H, int* parity, int64_t* n_refl, int* count) {
  double xx = *x, uu = *u;
  if (!isfinite(xx) || !isfinite(uu) || fabs(xx) > 10.0 * H) return -1;
  int c = 0;
  while (xx < 0.0 || xx > H) {
    xx = (xx < 0.0) ? -xx : 2.0 * H - xx;
    uu = -uu;
    *parity = -*parity;
    ++*n_refl;
    ++c;
  }
  *x = xx;
  *u = uu;
  if (count) *count = c;
  return 0;
}

/* integrators.hpp:31-37 */
static double ou_decay(double lam, double h) { return orc_exp_neg(lam, h); }
static double ou_noise_sd(double lam, double h) {
  if (g_devmath) { /* device ou_terms: expm1(2x) = em1 (em1 + 2), x = -lam h */
    double em1, ex;
    dm_expm1_exp(-lam * h, &em1, &ex);
    return sqrt(-(em1 * (em1 + 2.0)) / (2.0 * lam));
  }
  return sqrt(-expm1(-2.0 * lam * h) / (2.0 * lam));
}

/* integrators.hpp:41-43 */
double orc_se_stability_limit(const ablmc_model_params* p) {
  return 2.0 / orc_sde_coeffs(p->eps_reg, p).lambda;
}

/* integrators.hpp:50-58 (se), 63-72 (gl), 82-98 (baoab_step_impl) */
int orc_step(int ig, orc_state* s, double h, double xi, const ablmc_model_params* p,
             int scale_noise_by_parity, int* parity_at_noise) {
  if (ig == ABLMC_SE) {
    const orc_coeffs c = orc_sde_coeffs(s->x, p);
    const double u1 = (1.0 - c.lambda * h) * s->u - orc_dv_dx(&c, s->u) * h + c.sigma * sqrt(h) * xi;
    double x1 = s->x + u1 * h, uu = u1;
    if (parity_at_noise) *parity_at_noise = s->parity;
    if (orc_reflect(&x1, &uu, p->H, &s->parity, &s->n_refl, NULL)) return -1;
    s->x = x1;
    s->u = uu;
    return 0;
  }
  if (ig == ABLMC_GL) {
    const orc_coeffs c = orc_sde_coeffs(s->x, p);
    const double ustar = ou_decay(c.lambda, h) * s->u + c.sigma * ou_noise_sd(c.lambda, h) * xi;
    const double u1 = ustar - orc_dv_dx(&c, ustar) * h;
    double x1 = s->x + u1 * h, uu = u1;
    if (parity_at_noise) *parity_at_noise = s->parity;
    if (orc_reflect(&x1, &uu, p->H, &s->parity, &s->n_refl, NULL)) return -1;
    s->x = x1;
    s->u = uu;
    return 0;
  }
  /* BAOAB */
  const double h2 = 0.5 * h;
  const orc_coeffs c0 = orc_sde_coeffs(s->x, p);
  const double uh = s->u - orc_dv_dx(&c0, s->u) * h2;
  double x1 = s->x + uh * h2, u1 = uh;
  int par = s->parity;
  int64_t nr = s->n_refl;
  if (orc_reflect(&x1, &u1, p->H, &par, &nr, NULL)) return -1;
  const orc_coeffs cm = orc_sde_coeffs(x1, p);
  const double xi_eff = scale_noise_by_parity ? par * xi : xi;
  const double us = ou_decay(cm.lambda, h) * u1 + cm.sigma * ou_noise_sd(cm.lambda, h) * xi_eff;
  if (parity_at_noise) *parity_at_noise = par;
  double x2 = x1 + us * h2, u2 = us;
  if (orc_reflect(&x2, &u2, p->H, &par, &nr, NULL)) return -1;
  const orc_coeffs c1 = orc_sde_coeffs(x2, p);
  const double uend = u2 - orc_dv_dx(&c1, u2) * h2;
  s->x = x2;
  s->u = uend;
  s->parity = par;
  s->n_refl = nr;
  return 0;
}

/* Sequential NoiseStream::next() over draws k = 0, 1, ... (noise.hpp:57). */
typedef struct { uint64_t seed; uint32_t level; uint64_t idx; const double* xi; uint64_t k; } orc_stream;
static double stream_next(orc_stream* ns) {
  const uint64_t k = ns->k++;
  return ns->xi ? ns->xi[k] : orc_normal_at(ns->seed, ns->level, ns->idx, k);
}

/* coupling.hpp:64-105 */
int orc_simulate_pair(int ig, const ablmc_model_params* p, double x0, double u0, double T,
                      int64_t M, uint64_t seed, uint32_t level, uint64_t idx,
                      const double* xi, int signs_on, orc_state* fine, orc_state* coarse) {
  orc_stream ns = {seed, level, idx, xi, 0};
  orc_state f = {x0, u0, +1, 0}, c = {x0, u0, +1, 0};
  const double h = T / (double)M;
  const double h2 = 2.0 * h;
  int rc = 0;
  for (int64_t n = 0; n < M / 2; ++n) {
    const double xi0 = stream_next(&ns);
    const double xi1 = stream_next(&ns);
    const double lam_fine = orc_sde_coeffs(f.x, p).lambda;
    int pn0, pn1;
    if (orc_step(ig, &f, h, xi0, p, 0, &pn0)) { rc = -1; break; }
    if (orc_step(ig, &f, h, xi1, p, 0, &pn1)) { rc = -1; break; }
    const int s0 = signs_on ? pn0 : 1;
    const int s1 = signs_on ? pn1 : 1;
    if (ig == ABLMC_SE) {
      const int sc = signs_on ? c.parity : 1;
      if (orc_step(ig, &c, h2, orc_coarse_noise_se(xi0, xi1, s0, s1, sc), p, 0, NULL)) { rc = -1; break; }
    } else if (ig == ABLMC_GL) {
      const int sc = signs_on ? c.parity : 1;
      if (orc_step(ig, &c, h2, orc_coarse_noise_gl(xi0, xi1, lam_fine, h, s0, s1, sc), p, 0, NULL)) { rc = -1; break; }
    } else {
      const double xi_hat = orc_coarse_noise_gl(xi0, xi1, lam_fine, h, s0, s1, 1);
      if (orc_step(ig, &c, h2, xi_hat, p, signs_on, NULL)) { rc = -1; break; }
    }
  }
  *fine = f;
  *coarse = c;
  return rc;
}

/* coupling.hpp:22-29 */
int orc_simulate_path(int ig, const ablmc_model_params* p, double x0, double u0, double T,
                      int64_t M, uint64_t seed, uint32_t level, uint64_t idx,
                      const double* xi, orc_state* out) {
  orc_stream ns = {seed, level, idx, xi, 0};
  orc_state s = {x0, u0, +1, 0};
  const double h = T / (double)M;
  int rc = 0;
  for (int64_t n = 0; n < M; ++n)
    if (orc_step(ig, &s, h, stream_next(&ns), p, 0, NULL)) { rc = -1; break; }
  *out = s;
  return rc;
}

/* ------------------------------------------------- adaptive (non-nested) */
/* timeline.hpp:18-23 — min{h, lambda(x_adapt)/lambda(x) h} */
static double adaptive_step_size(double x, double h, double x_adapt, const ablmc_model_params* p) {
  const double lam_ref = orc_sde_coeffs(x_adapt, p).lambda;
  const double lam_x = orc_sde_coeffs(x, p).lambda;
  const double v = (lam_ref / lam_x) * h;
  return (v < h) ? v : h; /* std::min(h, v) */
}

/* coupling.hpp:31-51 */
int orc_simulate_path_adaptive(int ig, const ablmc_model_params* p, double x0, double u0,
                               double T, double h_base, double x_adapt, uint64_t seed,
                               uint32_t level, uint64_t idx, const double* xi, orc_state* out,
                               int64_t* steps_out) {
  orc_stream ns = {seed, level, idx, xi, 0};
  orc_state s = {x0, u0, +1, 0};
  int64_t steps = 0;
  const int64_t max_steps = 64 * (int64_t)ceil(T / h_base) + 64;
  double t = 0.0;
  int rc = 0;
  while (t < T) {
    double h = adaptive_step_size(s.x, h_base, x_adapt, p);
    if (t + h >= T) h = T - t;
    if (orc_step(ig, &s, h, stream_next(&ns), p, 0, NULL)) { rc = -1; break; }
    t = (t + h >= T) ? T : t + h;
    if (++steps > max_steps) { rc = -1; break; }
  }
  *out = s;
  *steps_out = steps;
  return rc;
}

/* timeline.hpp:75-105: the adaptive increments over the pending sub-intervals */
static double increment_se(const double* xi, const double* dt, const int* sg, int n, int sc,
                           int is_coarse) {
  double acc = 0.0;
  for (int j = 0; j < n; ++j) {
    const double s = is_coarse ? (double)sg[j] : 1.0;
    acc += s * xi[j] * sqrt(dt[j]);
  }
  return (is_coarse ? sc : 1) * acc;
}
static double increment_gl(const double* xi, const double* dt, const double* lam, const int* sg,
                           int n, int sc, int is_coarse) {
  double acc = 0.0, damp = 1.0;
  for (int r = n; r-- > 0;) {
    const double s = is_coarse ? (double)sg[r] : 1.0;
    acc += s * xi[r] * ou_noise_sd(lam[r], dt[r]) * damp;
    damp *= orc_exp_neg(lam[r], dt[r]);
  }
  return (is_coarse ? sc : 1) * acc;
}

#define ORC_MAX_PENDING 65536
typedef struct {
  orc_state s;
  double t, h_cur, t_next;
  int done;
  int64_t steps;
  int n;
  double xi[ORC_MAX_PENDING], dt[ORC_MAX_PENDING], lam[ORC_MAX_PENDING];
  int sg[ORC_MAX_PENDING];
} orc_leg;

static void leg_schedule(orc_leg* L, double base, double T, double x_adapt,
                         const ablmc_model_params* p) {
  double h = adaptive_step_size(L->s.x, base, x_adapt, p);
  if (L->t + h >= T) {
    h = T - L->t;
    L->t_next = T;
  } else {
    L->t_next = L->t + h;
  }
  L->h_cur = h;
}

static int leg_take(int ig, orc_leg* L, int is_coarse, const ablmc_model_params* p) {
  double xi_eq;
  if (ig == ABLMC_SE) {
    const double dw = increment_se(L->xi, L->dt, L->sg, L->n, is_coarse ? L->s.parity : 1, is_coarse);
    xi_eq = dw / sqrt(L->h_cur);
  } else {
    const double g = increment_gl(L->xi, L->dt, L->lam, L->sg, L->n, is_coarse ? L->s.parity : 1,
                                  is_coarse);
    xi_eq = g / ou_noise_sd(L->lam[0], L->h_cur);
  }
  if (orc_step(ig, &L->s, L->h_cur, xi_eq, p, 0, NULL)) return -1;
  L->t = L->t_next;
  ++L->steps;
  L->n = 0;
  return 0;
}

/* coupling.hpp:137-214 */
int orc_simulate_pair_adaptive(int ig, const ablmc_model_params* p, double x0, double u0,
                               double T, double h_base, double x_adapt, uint64_t seed,
                               uint32_t level, uint64_t idx, const double* xi_in, int signs_on,
                               orc_state* fine, orc_state* coarse, int64_t* steps_out) {
  orc_stream ns = {seed, level, idx, xi_in, 0};
  static __thread orc_leg F, Cc;
  orc_leg* f = &F;
  orc_leg* c = &Cc;
  f->s = (orc_state){x0, u0, +1, 0};
  f->t = 0.0; f->done = 0; f->steps = 0; f->n = 0;
  *c = *f;
  g_max_pending = 0;
  leg_schedule(f, h_base, T, x_adapt, p);
  leg_schedule(c, 2.0 * h_base, T, x_adapt, p);
  const int64_t max_iter = 256 * (int64_t)ceil(T / h_base) + 256;
  int64_t iter = 0;
  double t = 0.0;
  int rc = 0;
  while (!f->done || !c->done) {
    const double a = f->done ? T : f->t_next, b = c->done ? T : c->t_next;
    const double tau_next = (b < a) ? b : a; /* std::min */
    const double dt = tau_next - t;
    if (dt > 0.0) {
      const double xi = stream_next(&ns);
      const int sf = signs_on ? f->s.parity : 1;
      if (!f->done) {
        if (f->n >= ORC_MAX_PENDING) { rc = -2; break; }
        f->xi[f->n] = xi; f->dt[f->n] = dt; f->lam[f->n] = orc_sde_coeffs(f->s.x, p).lambda;
        f->sg[f->n++] = 1;
      }
      if (!c->done) {
        if (c->n >= ORC_MAX_PENDING) { rc = -2; break; }
        c->xi[c->n] = xi; c->dt[c->n] = dt; c->lam[c->n] = orc_sde_coeffs(c->s.x, p).lambda;
        c->sg[c->n++] = sf;
      }
      if (f->n > g_max_pending) g_max_pending = f->n;
      if (c->n > g_max_pending) g_max_pending = c->n;
    }
    if (!f->done && f->t_next == tau_next) {
      if (leg_take(ig, f, 0, p)) { rc = -1; break; }
      if (f->t_next >= T) f->done = 1;
      else leg_schedule(f, h_base, T, x_adapt, p);
    }
    if (!c->done && c->t_next == tau_next) {
      if (leg_take(ig, c, 1, p)) { rc = -1; break; }
      if (c->t_next >= T) c->done = 1;
      else leg_schedule(c, 2.0 * h_base, T, x_adapt, p);
    }
    t = tau_next;
    if (++iter > max_iter) { rc = -1; break; }
  }
  *fine = f->s;
  *coarse = c->s;
  *steps_out = f->steps + c->steps;
  return rc;
}

/* qoi.hpp:31-77 — Gaussian elimination with partial pivoting. */
int orc_build_smoothing_polynomial(int r, double* x) {
  if (r < 0 || r > 12) return -1;
  const int n = r + 2;
  double A[14 * 14], b[14];
  memset(A, 0, sizeof A);
  memset(b, 0, sizeof b);
#define AT(row, col) A[(row) * n + (col)]
  for (int i = 0; i < n; ++i) {
    AT(0, i) = (i % 2 == 0) ? 1.0 : -1.0;
    AT(1, i) = 1.0;
  }
  b[0] = 1.0;
  b[1] = 0.0;
  for (int j = 0; j < r; ++j) {
    for (int i = 0; i < n; ++i) AT(2 + j, i) = ((i + j) % 2 == 1) ? 0.0 : 2.0 / (double)(i + j + 1);
    b[2 + j] = ((j % 2 == 0) ? 1.0 : -1.0) / (double)(j + 1);
  }
  for (int col = 0; col < n; ++col) {
    int piv = col;
    for (int row = col + 1; row < n; ++row)
      if (fabs(AT(row, col)) > fabs(AT(piv, col))) piv = row;
    if (fabs(AT(piv, col)) < 1e-14) return -2;
    if (piv != col) {
      for (int k = 0; k < n; ++k) { double t = AT(piv, k); AT(piv, k) = AT(col, k); AT(col, k) = t; }
      double t = b[piv]; b[piv] = b[col]; b[col] = t;
    }
    for (int row = col + 1; row < n; ++row) {
      const double f = AT(row, col) / AT(col, col);
      for (int k = col; k < n; ++k) AT(row, k) -= f * AT(col, k);
      b[row] -= f * b[col];
    }
  }
  for (int row = n - 1; row >= 0; --row) {
    double acc = b[row];
    for (int k = row + 1; k < n; ++k) acc -= AT(row, k) * x[k];
    x[row] = acc / AT(row, row);
  }
#undef AT
  return 0;
}

/* qoi.hpp:22-26 (Horner), 80-84 (g_r) */
static double poly_eval(const double* c, int r, double s) {
  double acc = 0.0;
  for (int i = r + 2; i-- > 0;) acc = acc * s + c[i];
  return acc;
}
static double g_r(double x, const double* c, int r) {
  if (x < -1.0) return 1.0;
  if (x > 1.0) return 0.0;
  return poly_eval(c, r, x);
}

/* qoi.hpp:171-188 with 89-92 (smoothed_indicator) and 157-167 (binned_field). */
void orc_evaluate(const ablmc_qoi_spec* q, const double* poly, int r, double x, double* out) {
  switch (q->kind) {
    case ABLMC_QOI_MEAN_POSITION: out[0] = x; return;
    case ABLMC_QOI_RAW_INDICATOR: out[0] = (x >= q->a && x <= q->b) ? 1.0 : 0.0; return;
    case ABLMC_QOI_SMOOTHED_INDICATOR:
      out[0] = g_r((x - q->b) / q->delta, poly, r) - g_r((x - q->a) / q->delta, poly, r);
      return;
    case ABLMC_QOI_BINNED_FIELD: {
      const int k = q->n_edges - 1;
      double g_lo = 0.0;
      for (int i = 0; i < k; ++i) {
        const double g_hi = (i + 1 == k) ? 1.0 : g_r((x - q->bin_edges[i + 1]) / q->delta, poly, r);
        out[i] = g_hi - g_lo;
        g_lo = g_hi;
      }
      return;
    }
  }
}

static int64_t qoi_dim(const ablmc_qoi_spec* q) {
  return q->kind == ABLMC_QOI_BINNED_FIELD ? (int64_t)q->n_edges - 1 : 1;
}

/* One sample of level_sampler(level) (estimators.hpp:60-72) or
 * path_sampler(M, stream_level) (estimators.hpp:75-81): returns steps, or -1
 * for a failed sample (coupling.hpp:241-243,266-268). */
static int64_t one_sample(const ablmc_problem* pr, const double* poly, int coupled, int level,
                          int64_t M, uint32_t stream_level, int64_t idx, double* y,
                          double* scratch) {
  const ablmc_model_params* p = &pr->params;
  double u0 = pr->u0;
  if (pr->random_u0) {
    /* Extension D2 (not in the reference): u0 = sigma_U(x0) z with z = draw
     * k = M of the sample's stream, shared by fine and coarse (device
     * run_sample). */
    const double z = orc_normal_at(pr->seed, coupled ? (uint32_t)level : stream_level,
                                   (uint64_t)idx, (uint64_t)M);
    u0 = sqrt(orc_sde_coeffs(pr->x0, p).sigma_u2) * z;
  }
  if (coupled) {
    orc_state f, c;
    int64_t steps = M + M / 2;
    int rc;
    if (pr->adaptive) /* coupling.hpp:262-265 */
      rc = orc_simulate_pair_adaptive(pr->integrator, p, pr->x0, u0, pr->T, pr->T / (double)M,
                                      pr->x_adapt, pr->seed, (uint32_t)level, (uint64_t)idx,
                                      NULL, pr->signs_on, &f, &c, &steps);
    else
      rc = orc_simulate_pair(pr->integrator, p, pr->x0, u0, pr->T, M, pr->seed,
                             (uint32_t)level, (uint64_t)idx, NULL, pr->signs_on, &f, &c);
    if (rc) return -1;
    orc_evaluate(&pr->qoi, poly, pr->qoi.r, f.x, y);
    orc_evaluate(&pr->qoi, poly, pr->qoi.r, c.x, scratch);
    const int64_t d = qoi_dim(&pr->qoi);
    for (int64_t i = 0; i < d; ++i) y[i] -= scratch[i];
    return steps;
  }
  orc_state s;
  int64_t steps = M;
  int rc;
  if (pr->adaptive) /* coupling.hpp:238-240 */
    rc = orc_simulate_path_adaptive(pr->integrator, p, pr->x0, u0, pr->T, pr->T / (double)M,
                                    pr->x_adapt, pr->seed, stream_level, (uint64_t)idx, NULL, &s,
                                    &steps);
  else
    rc = orc_simulate_path(pr->integrator, p, pr->x0, u0, pr->T, M, pr->seed, stream_level,
                           (uint64_t)idx, NULL, &s);
  if (rc) return -1;
  orc_evaluate(&pr->qoi, poly, pr->qoi.r, s.x, y);
  return steps;
}

/* stats.hpp:96-136 (the result is independent of the worker count, so one
 * thread restates it) with LevelStats::add/merge (stats.hpp:46-63). */
static int accumulate(const ablmc_problem* pr, int coupled, int level, int64_t M,
                      uint32_t stream_level, int64_t first, int64_t count,
                      ablmc_level_stats* acc) {
  if (count <= 0) return 0;
  orc_set_profile(pr->profile, pr->const_sigma_u, pr->const_tau, pr->sigma_floor, pr->tau_min,
                  pr->tau_max);
  double poly[14] = {0};
  if (orc_build_smoothing_polynomial(pr->qoi.r, poly)) return -1;
  const int64_t dim = qoi_dim(&pr->qoi);
  double* y = calloc((size_t)dim * 4, sizeof(double));
  double* scratch = y + dim;
  double* ps = y + 2 * dim;
  double* ps2 = y + 3 * dim;
  const int64_t block = 4096;
  const int64_t n_blocks = (count + block - 1) / block;
  for (int64_t b = 0; b < n_blocks; ++b) {
    for (int64_t i = 0; i < dim; ++i) ps[i] = ps2[i] = 0.0;
    int64_t pn = 0, pf = 0, pc = 0;
    const int64_t lo = first + b * block;
    const int64_t hi = (first + count < lo + block) ? first + count : lo + block;
    for (int64_t idx = lo; idx < hi; ++idx) {
      const int64_t steps = one_sample(pr, poly, coupled, level, M, stream_level, idx, y, scratch);
      if (steps >= 0) {
        for (int64_t i = 0; i < dim; ++i) {
          ps[i] += y[i];
          ps2[i] += y[i] * y[i];
        }
        ++pn;
        pc += steps;
      } else {
        ++pf;
      }
    }
    for (int64_t i = 0; i < dim; ++i) {
      acc->sum_y[i] += ps[i];
      acc->sum_y2[i] += ps2[i];
    }
    acc->n += pn;
    acc->failed += pf;
    acc->cost_steps += pc;
  }
  free(y);
  orc_set_profile(ABLMC_PROFILE_REFERENCE, 0, 0, 0, 0, 0);
  return 0;
}

int orc_accumulate_samples(const ablmc_problem* pr, int level, int64_t first, int64_t count,
                           ablmc_level_stats* acc) {
  if (level == 0) return accumulate(pr, 0, 0, pr->m0, 0, first, count, acc);
  return accumulate(pr, 1, level, pr->m0 << level, 0, first, count, acc);
}

int orc_accumulate_paths(const ablmc_problem* pr, int64_t M, uint32_t stream_level,
                         int64_t first, int64_t count, ablmc_level_stats* acc) {
  return accumulate(pr, 0, 0, M, stream_level, first, count, acc);
}
