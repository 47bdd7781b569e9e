"""The paper's Table 3: runtime to reach an
RMS error of eps = 4e-3 on the 20-bin smoothed concentration field (box size
0.05, r = 4, delta = 0.1), release heights X0 = 0.05 / 0.10 / 0.20, M0 = 80
for SE and GL, 40 for BAOAB; MLMC (SE, GL) and StMC (SE, GL, BAOAB, finest
level from the same bias fit, as cost_sweep does).  The paper ran on one core
of an i5-4460; here the reference's own drivers run on the B200 sampler, and
with --cpu also the reference itself (oracle/_ref, all host threads).

    python tools/paper_table3.py [--cpu] > profiles/r1_paper_table3.json
"""
import ctypes as C
import json
import os
import sys
import time

sys.path[:0] = [".", "tests"]
from paper_1612_07717_b200 import ablmc, capi  # noqa: E402

PAPER = {  # seconds, i5-4460 one core (Table 3)
    0.05: {"stmc_se": 2561.41, "stmc_gl": 321.77, "stmc_baoab": 91.21, "mlmc_se": 218.52,
           "mlmc_gl": 265.84},
    0.10: {"stmc_se": 867.32, "stmc_gl": 277.72, "stmc_baoab": 79.25, "mlmc_se": 120.17,
           "mlmc_gl": 125.92},
    0.20: {"stmc_se": 316.33, "stmc_gl": 280.04, "stmc_baoab": 78.15, "mlmc_se": 64.78,
           "mlmc_gl": 103.69},
}
EPS = 4e-3
Ig = ablmc.Integrator


def problem(ig, x0):
    q = ablmc.QoISpec(kind=ablmc.QoIKind.binned_field, bin_edges=ablmc.equidistant_edges(20, 1.0))
    return ablmc.Problem.make(ablmc.ModelParams(), ig, q, x0, 0.1, 1.0, 40 if ig == Ig.baoab else 80,
                              2017)


def main():
    cpu = "--cpu" in sys.argv
    ablmc.init(0)
    ablmc.run_mlmc(problem(Ig.gl, 0.2), 2e-2)  # warm-up (context, workspaces)
    out = {"eps": EPS, "bins": 20, "rows": {}}
    R = None
    if cpu:
        import oracle_lib as O
        R = O.ref()
    threads = len(os.sched_getaffinity(0))
    for x0 in (0.05, 0.10, 0.20):
        row = {}
        fits = {}
        for ig in (Ig.se, Ig.gl, Ig.baoab):
            pr = problem(ig, x0)
            t = time.perf_counter()
            r = ablmc.run_mlmc(pr, EPS)
            dt = time.perf_counter() - t
            fits[ig] = (r.alpha, r.c1)
            if ig != Ig.baoab:  # the paper reports MLMC for SE and GL only
                row[f"mlmc_{ig.name}"] = {"b200_seconds": dt, "levels": r.levels_used,
                                          "total_cost_steps": r.total_cost_steps,
                                          "paper_seconds": PAPER[x0][f"mlmc_{ig.name}"]}
                if R is not None:
                    o = capi.MlmcOptionsC()
                    ablmc.lib().ablmc_mlmc_options_defaults(C.byref(o))
                    rr = capi.RunResultC()
                    t = time.perf_counter()
                    R.ref_run_mlmc(C.byref(pr._c), EPS, C.byref(o), threads, C.byref(rr))
                    row[f"mlmc_{ig.name}"]["reference_cpu_seconds"] = time.perf_counter() - t
                    row[f"mlmc_{ig.name}"]["reference_cpu_threads"] = threads
        for ig in (Ig.se, Ig.gl, Ig.baoab):
            pr = problem(ig, x0)
            L = ablmc.choose_levels(*fits[ig], EPS, pr.m0, 1.0)
            t = time.perf_counter()
            r = ablmc.run_stmc(pr, pr.m0 << L, EPS)
            dt = time.perf_counter() - t
            row[f"stmc_{ig.name}"] = {"b200_seconds": dt, "M_L": pr.m0 << L,
                                      "total_cost_steps": r.total_cost_steps,
                                      "paper_seconds": PAPER[x0][f"stmc_{ig.name}"]}
        out["rows"][f"x0={x0}"] = row
        print(json.dumps({f"x0={x0}": row}), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
