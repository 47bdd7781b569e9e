"""Randomised parity campaign for the single-path samplers (level 0 / StMC:
simulate_path, coupling.hpp:22-51; path_sampler, estimators.hpp:75-81) on the
GPU box: the generator of tests/test_gpu_fuzz.py on fresh seeds, path lengths
M from {1, 2, 3, 4, 5, 8, m0, m0 << level} (the lean one-step kernel, the
4-samples-per-thread short-path kernel, odd lengths, the general loop),
random stream levels, uniform and adaptive grids, QoI kinds:
  states   simulate_paths vs the C oracle on the device's elementary
           functions: bit-identical (x, u, parity, reflections, ok);
  sums     accumulate_paths (the production kernels, incl. the hoisted first
           step) vs the oracle's accumulate: counts exact, sums rel 1e-11;
  level 0  accumulate_samples(level 0) vs the oracle, and the same sums from
           two calls split at a ragged index (continuing sample indices).
usage: python tools/fuzz_paths.py [first_trial] [n_trials]"""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle_lib as O  # noqa: E402
from paper_1612_07717_b200 import ablmc  # noqa: E402
from test_gpu_fuzz import Ig, random_problem  # noqa: E402

first_trial = int(sys.argv[1]) if len(sys.argv) > 1 else 0
n_trials = int(sys.argv[2]) if len(sys.argv) > 2 else 500
ablmc.init(0)
bad, paths, sums_checked, failed_paths, adaptive_n = [], 0, 0, 0, 0
t0 = time.time()
QOIS = (ablmc.QoIKind.mean_position, ablmc.QoIKind.smoothed_indicator, ablmc.QoIKind.raw_indicator)


def close(a, b):
    return abs(a - b) <= 1e-11 * max(1.0, abs(b))


for trial in range(first_trial, first_trial + n_trials):
    rng = np.random.default_rng(130_000 + trial)
    try:
        pr, level = random_problem(rng)
    except Exception:
        continue
    c = pr._c
    c.qoi.kind = int(QOIS[int(rng.integers(0, 3))])
    M = int(rng.choice([1, 2, 3, 4, 5, 8, c.m0, c.m0 << level]))
    if c.adaptive and M > 640:
        continue
    sl = int(rng.choice([0, 0, 1, level, 7]))
    n = 96
    first = int(rng.integers(0, 2**40))
    adaptive_n += bool(c.adaptive)
    O.orc().orc_set_device_math(1)
    O.orc().orc_set_profile(c.profile, c.const_sigma_u, c.const_tau, c.sigma_floor, c.tau_min,
                            c.tau_max)
    try:
        got = ablmc.simulate_paths(pr, M, first, n, sl)
        for i in range(n):
            if c.adaptive:
                rc, s, _ = O.orc_path_adaptive(c.integrator, c.params, c.x0, c.u0, c.T, c.T / M,
                                               c.x_adapt, c.seed, sl, first + i)
            else:
                rc, s = O.orc_path(c.integrator, c.params, c.x0, c.u0, c.T, M, c.seed, sl,
                                   first + i)
            g = got[i]
            paths += 1
            failed_paths += rc != 0
            if (rc == 0) != bool(g["ok"]):
                bad.append((trial, i, "ok flag", rc, int(g["ok"])))
            elif rc == 0 and [g["x"], g["u"], g["parity"], g["n_refl"]] != [s.x, s.u, s.parity,
                                                                             s.n_refl]:
                bad.append((trial, i, "state", [g["x"], g["u"], g["parity"], g["n_refl"]],
                            [s.x, s.u, s.parity, s.n_refl]))
        # the production accumulate kernels on a ragged count
        cnt = int(rng.integers(1, 3000))
        acc = ablmc.LevelStats().init(0, c.T / M, 1)
        ablmc.accumulate_paths(acc, first, cnt, pr, M, sl)
        st = O.Stats(1)
        if O.orc().orc_accumulate_paths(C.byref(c), M, sl, first, cnt, C.byref(st.c)) == 0:
            sums_checked += 1
            if (acc.n, acc.failed, acc.cost_steps) != (st.n, st.failed, st.cost_steps):
                bad.append((trial, -1, "path counts", (acc.n, acc.failed, acc.cost_steps),
                            (st.n, st.failed, st.cost_steps)))
            elif not (close(acc.sum_y[0], st.sum_y[0]) and close(acc.sum_y2[0], st.sum_y2[0])):
                bad.append((trial, -1, "path sums", acc.sum_y[0], st.sum_y[0]))
        # level 0 through the level sampler, one call and two calls split at a ragged index
        a1 = ablmc.LevelStats().init(0, pr.h_level(0), 1)
        ablmc.accumulate_samples(a1, first, cnt, pr, 0)
        cut = int(rng.integers(0, cnt + 1))
        a2 = ablmc.LevelStats().init(0, pr.h_level(0), 1)
        ablmc.accumulate_samples(a2, first, cut, pr, 0)
        ablmc.accumulate_samples(a2, first + cut, cnt - cut, pr, 0)
        s0 = O.Stats(1)
        if O.orc().orc_accumulate_samples(C.byref(c), 0, first, cnt, C.byref(s0.c)) == 0:
            sums_checked += 1
            for a in (a1, a2):
                if (a.n, a.failed, a.cost_steps) != (s0.n, s0.failed, s0.cost_steps):
                    bad.append((trial, -2, "level-0 counts", (a.n, a.failed, a.cost_steps),
                                (s0.n, s0.failed, s0.cost_steps)))
                elif not (close(a.sum_y[0], s0.sum_y[0]) and close(a.sum_y2[0], s0.sum_y2[0])):
                    bad.append((trial, -2, "level-0 sums", a.sum_y[0], s0.sum_y[0]))
    finally:
        O.orc().orc_set_device_math(0)
        O.orc().orc_set_profile(0, 0, 0, 0, 0, 0)
for b in bad[:20]:
    print("MISMATCH", b)
print(f"fuzz_paths: trials {first_trial}..{first_trial + n_trials - 1}, {paths} single paths "
      f"compared bit for bit ({adaptive_n} adaptive problems, {failed_paths} failed paths agreed), "
      f"{sums_checked} accumulate calls checked, {len(bad)} mismatches, {time.time() - t0:.0f} s")
sys.exit(1 if bad else 0)
