"""BASELINE.json configs 4 and 5 at their FULL sizes on one B200, and the
reference's own CPU run_mlmc at the tightest config-3 tolerance (VERDICT r1
"Record the full-size configs").

  * config 4: release at z0 = 10 m (x0 = 0.01), 64-bin smoothed
    concentration field (binned_field, r = 4, delta = 0.1), GL, floored
    profile, w0 ~ N(0, sigma_w(z0)^2), levels 0..10, 2e8 coupled paths per
    level: one accumulate_samples call per level into a host LevelStats
    (qoi.hpp:144-167, stats.hpp:96-136);
  * config 5: SE, level 10, reference profile, x0 = 0.5, N = 1e9 and 4e9
    coupled paths in one accumulate_samples call each (the public API, host
    result);
  * config 3 at eps = 3e-3 m: the product's run_mlmc (BAOAB, reference
    profile, x0 = 0.5, M0 = 1) and, with --cpu, the reference's own run_mlmc
    (oracle/_ref, all host threads) on the same problem and seed.

    python tools/full_configs.py [--cpu] > profiles/r2_full_configs.json
"""
import ctypes as C
import json
import os
import sys
import time

sys.path[:0] = [".", "tests"]
from paper_1612_07717_b200 import ablmc, capi  # noqa: E402

Ig = ablmc.Integrator


def timed(fn):
    t0 = time.perf_counter()
    r = fn()
    return r, time.perf_counter() - t0


def main():
    cpu = "--cpu" in sys.argv
    ablmc.init(0)
    mp = ablmc.ModelParams()
    out = {"device": "B200 x1"}

    # ---- config 4
    q = ablmc.QoISpec(kind=ablmc.QoIKind.binned_field, bin_edges=ablmc.equidistant_edges(64, 1.0))
    pr = ablmc.Problem.make(mp, Ig.gl, q, 0.01, 0.0, 1.0, 1, 42, profile=ablmc.Profile.floored,
                            random_u0=True)
    n4 = 200_000_000
    warm = ablmc.LevelStats().init(0, pr.h_level(0), 64)
    ablmc.accumulate_samples(warm, 0, 1 << 22, pr, 0)
    rows, total = [], 0.0
    for level in range(11):
        st = ablmc.LevelStats().init(level, pr.h_level(level), 64)
        _, t = timed(lambda: ablmc.accumulate_samples(st, 0, n4, pr, level))
        total += t
        rows.append({"level": level, "seconds": t, "paths_per_s": n4 / t,
                     "fine_path_steps_per_s": n4 * (1 << level) / t, "n": st.n,
                     "failed": st.failed, "max_abs_mean": float(abs(st.sum_y / st.n).max()),
                     "sum_components_mean": float(st.sum_y.sum() / st.n)})
    out["config4_z0_10m_64bins_gl_2e8_per_level"] = {"levels": rows, "total_seconds": total}

    # ---- config 5
    pr = ablmc.Problem.make(mp, Ig.se, ablmc.QoISpec(), 0.5, 0.1, 1.0, 1, 42)
    c5 = {}
    for n in (10**9, 4 * 10**9):
        st = ablmc.LevelStats().init(10, pr.h_level(10), 1)
        _, t = timed(lambda: ablmc.accumulate_samples(st, 0, n, pr, 10))
        c5[f"{n:.0e}"] = {"seconds": t, "path_steps_per_s": n * 1024 / t, "n": st.n,
                          "failed": st.failed, "mean_y": st.mean(), "std_error": st.std_error()}
    out["config5_se_l10_full"] = c5

    # ---- config 3, tightest tolerance
    pr = ablmc.Problem.make(mp, Ig.baoab, ablmc.QoISpec(), 0.5, 0.1, 1.0, 1, 42)
    eps = 3e-6
    r, t = timed(lambda: ablmc.run_mlmc(pr, eps))
    row = {"eps_m": eps * 1000, "seconds": t, "estimate": r.estimate[0],
           "stat_error": r.stat_error[0], "levels": r.levels_used,
           "N_l": [s.n for s in r.level_stats], "total_cost_steps": r.total_cost_steps}
    if cpu:
        import oracle_lib as O
        R = O.ref()
        threads = len(os.sched_getaffinity(0))
        o = capi.MlmcOptionsC()
        ablmc.lib().ablmc_mlmc_options_defaults(C.byref(o))
        rr = capi.RunResultC()
        t0 = time.perf_counter()
        rc = R.ref_run_mlmc(C.byref(pr._c), eps, C.byref(o), threads, C.byref(rr))
        row["reference_cpu"] = {"rc": rc, "seconds": time.perf_counter() - t0,
                                "estimate": rr.estimate, "threads": threads,
                                "levels": rr.n_levels,
                                "N_l": [rr.level_n[i] for i in range(rr.n_levels)],
                                "total_cost_steps": rr.total_cost_steps}
    out["config3_mlmc_baoab_eps_3e-3m"] = row
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
