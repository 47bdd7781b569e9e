"""Randomised campaign of the host drivers against the reference's own
(oracle/_ref: the unmodified run_mlmc / run_stmc, estimators.hpp:230-397, on
the reference's CPU sampler) on the GPU box: random problems on the reference
profile (model parameters, release, M0, integrator, QoI kind, signs), random
tolerances and MlmcOptions; same seed on both sides.  Compared: the return
code (both succeed or both refuse: SE stability, an indistinguishable bias
fit, the failure budget), levels_used, warnings, failed samples; N_l and the
costs (equal, or one allocation ceil apart: the level sums differ at 1e-11
between the two summation trees); estimate, statistical error, bias
estimate, alpha and c1 (relative 1e-6 of the statistical error / value).
usage: python tools/fuzz_drivers.py [first_trial] [n_trials]"""
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle_lib as O  # noqa: E402
from paper_1612_07717_b200 import ablmc, capi  # noqa: E402

first_trial = int(sys.argv[1]) if len(sys.argv) > 1 else 0
n_trials = int(sys.argv[2]) if len(sys.argv) > 2 else 100
R = O.ref()
assert R is not None, "oracle/_ref/libablmc_ref.so missing"
threads = min(16, os.cpu_count() or 1)
ablmc.init(0)
L = ablmc.lib()
bad, runs, refused, exact, t0 = [], 0, 0, 0, time.time()
Ig = ablmc.Integrator
QOIS = (ablmc.QoIKind.mean_position, ablmc.QoIKind.smoothed_indicator)


def near(a, b, tol, scale=None):
    return abs(a - b) <= tol * (abs(b) if scale is None else scale) + 1e-300


for trial in range(first_trial, first_trial + n_trials):
    rng = np.random.default_rng(210_000 + trial)
    ig = Ig(int(rng.integers(0, 3)))
    mp = ablmc.ModelParams(kappa_sigma=float(rng.uniform(1.0, 1.6)),
                           kappa_tau=float(rng.uniform(0.4, 0.7)),
                           u_star=float(rng.choice([0.1, 0.2, 0.3])))
    m0 = int(rng.choice([8, 20, 40])) if ig != Ig.se else int(rng.choice([40, 80, 160]))
    q = ablmc.QoISpec(kind=QOIS[int(rng.random() < 0.25)])
    opt = ablmc.SampleOptions(signs_on=bool(rng.random() < 0.9))
    try:
        pr = ablmc.Problem.make(mp, ig, q, float(rng.uniform(0.03, 0.6)),
                                float(rng.choice([0.0, 0.1, -0.2])), 1.0, m0,
                                int(rng.integers(0, 2**40)), opt)
    except Exception:
        continue
    stmc = rng.random() < 0.3
    eps = float(rng.choice([4e-3, 2e-3, 1e-3]))
    o = capi.MlmcOptionsC()
    L.ablmc_mlmc_options_defaults(C.byref(o))
    o.pilot_n = int(rng.choice([2000, 5000, 10000]))
    o.pilot_levels_max = int(rng.choice([3, 4]))
    o.init_n = int(rng.choice([500, 1000]))
    rd, rr = capi.RunResultC(), capi.RunResultC()
    if stmc:
        M = m0 << int(rng.integers(0, 3))
        rc_d = L.ablmc_run_stmc(C.byref(pr._c), M, eps, 0, C.byref(rd))
        rc_r = R.ref_run_stmc(C.byref(pr._c), M, eps, 0, threads, C.byref(rr))
    else:
        rc_d = L.ablmc_run_mlmc(C.byref(pr._c), eps, C.byref(o), C.byref(rd))
        rc_r = R.ref_run_mlmc(C.byref(pr._c), eps, C.byref(o), threads, C.byref(rr))
    runs += 1
    tag = (trial, "stmc" if stmc else "mlmc", ig.name, m0, eps)
    if (rc_d == 0) != (rc_r == 0):
        bad.append((*tag, "return code", rc_d, rc_r, L.ablmc_last_error().decode()[:80]))
        continue
    if rc_d != 0:
        refused += 1
        continue
    ok = True
    for f in ("levels_used", "n_levels", "failed_samples", "warnings_mask"):
        if getattr(rd, f) != getattr(rr, f):
            bad.append((*tag, f, getattr(rd, f), getattr(rr, f)))
            ok = False
    if not ok:
        continue
    same_n = all(rd.level_n[l] == rr.level_n[l] for l in range(rd.n_levels))
    for l in range(rd.n_levels):  # one allocation ceil apart at most
        if abs(rd.level_n[l] - rr.level_n[l]) > max(1, 1e-6 * rr.level_n[l]):
            bad.append((*tag, "N_l", l, rd.level_n[l], rr.level_n[l]))
            ok = False
    if same_n and (rd.total_cost_steps, rd.pilot_cost_steps) != (rr.total_cost_steps,
                                                                 rr.pilot_cost_steps):
        bad.append((*tag, "cost", rd.total_cost_steps, rr.total_cost_steps))
        ok = False
    se = rr.stat_error
    if not near(rd.estimate, rr.estimate, 1e-6, se) or not near(rd.stat_error, se, 1e-6):
        bad.append((*tag, "estimate", rd.estimate, rr.estimate, rd.stat_error, se))
        ok = False
    if not stmc and not (near(rd.alpha, rr.alpha, 1e-6) and near(rd.c1, rr.c1, 1e-6) and
                         near(rd.bias_estimate, rr.bias_estimate, 1e-6)):
        bad.append((*tag, "bias fit", rd.alpha, rr.alpha, rd.c1, rr.c1))
        ok = False
    exact += ok and same_n
for b in bad[:20]:
    print("MISMATCH", b)
print(f"fuzz_drivers: trials {first_trial}..{first_trial + n_trials - 1}: {runs} driver runs next to "
      f"the reference's own ({threads} host threads), {refused} refused by both alike, {exact} with "
      f"identical levels, N_l, costs and warnings, {len(bad)} mismatches, {time.time() - t0:.0f} s")
sys.exit(1 if bad else 0)
