"""Randomised parity campaign for the binned-field QoI (K1 position store +
K4 banded kernel, qoi.hpp:144-188; BASELINE config 4) on the GPU box: random
problems (the generator of tests/test_gpu_fuzz.py, uniform and adaptive
grids), random fields: 1 .. 700 bins, equidistant or random edges (incl.
near-duplicate edges), delta from 1e-6 H (band disabled) to 0.6 H (every
edge in the band), r in 1..8, levels 0-3 and ragged counts; per-bin sums of
accumulate_samples vs the C oracle on the device's elementary functions
(counts exact; sum_y, sum_y2 per bin within 1e-11 relative / 1e-11 absolute,
the summation trees differ).
usage: python tools/fuzz_binned.py [first_trial] [n_trials]"""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle_lib as O  # noqa: E402
from paper_1612_07717_b200 import ablmc  # noqa: E402
from test_gpu_fuzz import random_problem  # noqa: E402

first_trial = int(sys.argv[1]) if len(sys.argv) > 1 else 0
n_trials = int(sys.argv[2]) if len(sys.argv) > 2 else 300
ablmc.init(0)
bad, calls, bins_total = [], 0, 0
t0 = time.time()
for trial in range(first_trial, first_trial + n_trials):
    rng = np.random.default_rng(170_000 + trial)
    try:
        pr0, level = random_problem(rng)
    except Exception:
        continue
    c0 = pr0._c
    H = c0.params.H
    bins = int(rng.choice([1, 2, 3, 7, 16, 17, 64, 65, 200, 700]))
    if rng.random() < 0.5:
        edges = ablmc.equidistant_edges(bins, H)
    else:
        inner = np.sort(rng.uniform(0.0, H, bins - 1))
        if bins > 3 and rng.random() < 0.3:
            inner[1] = np.nextafter(inner[0], H)  # near-duplicate edges
            inner.sort()
        edges = [0.0] + inner.tolist() + [H]
    if any(b <= a for a, b in zip(edges, edges[1:])):
        continue  # the reference requires strictly increasing edges
    delta = float(rng.choice([1e-6, 1e-3, 0.02, 0.1, 0.6])) * H
    q = ablmc.QoISpec(kind=ablmc.QoIKind.binned_field, bin_edges=edges, delta=delta,
                      r=int(rng.integers(1, 9)))
    mp = ablmc.ModelParams(kappa_sigma=c0.params.kappa_sigma, kappa_tau=c0.params.kappa_tau,
                           u_star=c0.params.u_star, H=H, eps_reg=c0.params.eps_reg,
                           x_ref=c0.params.x_ref, noise_scale=c0.params.noise_scale)
    if c0.adaptive and (c0.m0 << 3) > 512:
        continue
    try:
        pr = ablmc.Problem.make(mp, ablmc.Integrator(c0.integrator), q, c0.x0, c0.u0, c0.T, c0.m0,
                                c0.seed, ablmc.SampleOptions(signs_on=bool(c0.signs_on),
                                                             adaptive=bool(c0.adaptive),
                                                             x_adapt=c0.x_adapt))
    except Exception:
        continue
    c = pr._c
    level = int(rng.integers(0, 4))
    first = int(rng.integers(0, 2**40))
    cnt = int(rng.integers(1, 2500))
    O.orc().orc_set_device_math(1)
    try:
        acc = ablmc.LevelStats().init(level, pr.h_level(level), bins)
        ablmc.accumulate_samples(acc, first, cnt, pr, level)
        st = O.Stats(bins)
        if O.orc().orc_accumulate_samples(C.byref(c), level, first, cnt, C.byref(st.c)) != 0:
            continue
        calls += 1
        bins_total += bins
        if (acc.n, acc.failed, acc.cost_steps) != (st.n, st.failed, st.cost_steps):
            bad.append((trial, "counts", (acc.n, acc.failed, acc.cost_steps),
                        (st.n, st.failed, st.cost_steps)))
            continue
        for name, a, b in (("sum_y", acc.sum_y, st.sum_y), ("sum_y2", acc.sum_y2, st.sum_y2)):
            err = np.abs(np.asarray(a) - np.asarray(b))
            lim = 1e-11 * np.abs(np.asarray(b)) + 1e-11
            if np.any(err > lim):
                k = int(np.argmax(err - lim))
                bad.append((trial, name, bins, level, k, float(a[k]), float(b[k])))
    finally:
        O.orc().orc_set_device_math(0)
for b in bad[:20]:
    print("MISMATCH", b)
print(f"fuzz_binned: trials {first_trial}..{first_trial + n_trials - 1}, {calls} binned accumulate "
      f"calls ({bins_total} bins) compared with the oracle, {len(bad)} mismatches, "
      f"{time.time() - t0:.0f} s")
sys.exit(1 if bad else 0)
