"""Long randomised parity campaign on the GPU box: the generator of
tests/test_gpu_fuzz.py on fresh seeds (and with wider ranges: levels 1-5,
releases at the walls, 96 samples per problem), device pair states vs the C
oracle on the device's elementary functions (bit-identical), plus the
accumulate path's counts (exact) and sums (rel 1e-11) on the same problem.
usage: python tools/fuzz_campaign.py [first_trial] [n_trials]   -> one summary line"""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle_lib as O  # noqa: E402
from paper_1612_07717_b200 import ablmc  # noqa: E402
from test_gpu_fuzz import KPEND_DEEP, Ig, random_problem  # noqa: E402

first_trial = int(sys.argv[1]) if len(sys.argv) > 1 else 0
n_trials = int(sys.argv[2]) if len(sys.argv) > 2 else 500
ablmc.init(0)
bad, deep_seen, samples, failed_paths, adaptive_n = [], 0, 0, 0, 0
t0 = time.time()
for trial in range(first_trial, first_trial + n_trials):
    rng = np.random.default_rng(50_000 + trial)
    try:
        pr, level = random_problem(rng)
    except Exception:  # the host validation rejected the draw (e.g. SE stability): next
        continue
    c = pr._c
    if rng.random() < 0.3:
        level = int(rng.integers(1, 6))
    if rng.random() < 0.15:  # releases at / next to the walls
        c.x0 = float(rng.choice([0.0, c.params.H, 1e-9 * c.params.H, (1 - 1e-12) * c.params.H]))
    n = 96
    first = int(rng.integers(0, 2**40))
    M = c.m0 << level
    if c.adaptive and M > 1024:
        continue
    got = ablmc.simulate_pairs(pr, level, first, n)
    O.orc().orc_set_device_math(1)
    O.orc().orc_set_profile(c.profile, c.const_sigma_u, c.const_tau, c.sigma_floor, c.tau_min,
                            c.tau_max)
    adaptive_n += bool(c.adaptive)
    try:
        for i in range(n):
            if c.adaptive:
                rc, f, cc, _ = O.orc_pair_adaptive(c.integrator, c.params, c.x0, c.u0, c.T,
                                                   c.T / M, c.x_adapt, c.seed, level, first + i,
                                                   c.signs_on)
            else:
                rc, f, cc = O.orc_pair(c.integrator, c.params, c.x0, c.u0, c.T, M, c.seed, level,
                                       first + i, signs_on=c.signs_on)
            g = got[i]
            samples += 1
            failed_paths += rc != 0
            if (rc == 0) != bool(g["fok"]):
                bad.append((trial, i, "ok flag", rc, int(g["fok"])))
                continue
            if rc != 0:
                continue
            deep = (c.adaptive and c.integrator != Ig.se
                    and O.orc().orc_last_max_pending() > KPEND_DEEP)
            deep_seen += deep
            have = [g["fx"], g["fu"], g["fpar"], g["fn"], g["cx"], g["cu"], g["cpar"], g["cn"]]
            want = [f.x, f.u, f.parity, f.n_refl, cc.x, cc.u, cc.parity, cc.n_refl]
            if deep:
                okv = all(abs(a - b) <= 1e-12 * max(abs(b), 1e-3) for a, b in zip(have, want))
            else:
                okv = have == want
            if not okv:
                bad.append((trial, i, "state", have, want))
        # the accumulate path on the same samples
        acc = ablmc.LevelStats().init(level, pr.h_level(level), 1)
        ablmc.accumulate_samples(acc, first, n, pr, level)
        st = O.Stats(1)
        if O.orc().orc_accumulate_samples(C.byref(c), level, first, n, C.byref(st.c)) == 0:
            if (acc.n, acc.failed, acc.cost_steps) != (st.n, st.failed, st.cost_steps):
                bad.append((trial, -1, "counts", (acc.n, acc.failed, acc.cost_steps),
                            (st.n, st.failed, st.cost_steps)))
            elif abs(acc.sum_y[0] - st.sum_y[0]) > 1e-11 * max(1.0, abs(st.sum_y[0])):
                bad.append((trial, -1, "sum", acc.sum_y[0], st.sum_y[0]))
    finally:
        O.orc().orc_set_device_math(0)
        O.orc().orc_set_profile(0, 0, 0, 0, 0, 0)
for b in bad[:20]:
    print("MISMATCH", b)
print(f"fuzz_campaign: trials {first_trial}..{first_trial + n_trials - 1}, {samples} pairs compared "
      f"({adaptive_n} adaptive problems, {failed_paths} failed paths agreed, {deep_seen} beyond "
      f"{KPEND_DEEP} pending), {len(bad)} mismatches, {time.time() - t0:.0f} s")
sys.exit(1 if bad else 0)
