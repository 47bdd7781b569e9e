"""Randomised parity campaign against the UNMODIFIED reference (oracle/_ref,
the reference headers behind a C shim) on the GPU box: random uniform-grid
problems on the reference profile (the generator of tests/test_gpu_fuzz.py,
fresh seeds), two legs per problem:
  oracle mode   the device driven by host-supplied normals (the reference
                stream's own draws) vs the reference's simulate_pair: SE must
                be bit-identical, GL/BAOAB within the north-star 1e-12 relative;
  Philox mode   the device's in-register normals vs the same reference states,
                at the test suite's 1e-10.
Parities, reflection counts and failure flags must agree.  Pairs outside the
tolerance are listed, not hidden (a 1-ulp libm difference can tip a
reflection for a path that lands within an ulp of a wall).
With --adaptive: adaptive (non-nested) problems only, Philox mode only (the
adaptive draws are data dependent, so there is no host-normal mode): the
schedule's comparisons see normals that differ from glibc's by an ulp, so a
pair's step sequence can legitimately differ; the share of pairs within
1e-10 is reported, and the run never fails on it (tests/test_gpu_adaptive.py
bounds the share by the reference's own 1-ulp sensitivity).
usage: python tools/fuzz_reference.py [first_trial] [n_trials] [--adaptive]"""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle_lib as O  # noqa: E402
from paper_1612_07717_b200 import ablmc, capi  # noqa: E402
from test_gpu_fuzz import Ig, random_problem  # noqa: E402

ADAPTIVE = "--adaptive" in sys.argv
argv = [a for a in sys.argv[1:] if not a.startswith("--")]
first_trial = int(argv[0]) if len(argv) > 0 else 0
n_trials = int(argv[1]) if len(argv) > 1 else 500
R = O.ref()
assert R is not None, "oracle/_ref/libablmc_ref.so missing (built where /root/reference exists)"
ablmc.init(0)
n = 32
stats = {m: {"pairs": 0, "bit": 0, "max_rel": 0.0, "out": [], "ints": 0, "worst": 0.0,
             "by_ig": {ig: [0, 0, 0] for ig in (0, 1, 2)}}  # pairs, bit-identical, outside
         for m in ("oracle", "philox")}
flags_bad, problems, failed_paths = [], 0, 0
t0 = time.time()


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-3)


for trial in range(first_trial, first_trial + n_trials):
    rng = np.random.default_rng(90_000 + trial)
    try:
        pr, level = random_problem(rng)
    except Exception:
        continue
    c = pr._c
    if bool(c.adaptive) != ADAPTIVE or c.profile != 0:
        continue
    if rng.random() < 0.3:
        level = int(rng.integers(1, 6))
    M = c.m0 << level
    if ADAPTIVE and M > 640:
        continue
    first = int(rng.integers(0, 2**40))
    problems += 1
    want = (capi.PairStateC * n)()
    R.ref_pair_states(C.byref(c), level, first, n, want)
    legs = [("philox", ablmc.simulate_pairs(pr, level, first, n))]
    if not ADAPTIVE:
        xi = np.stack([O.ref_normals(c.seed, level, first + i, 0, M) for i in range(n)])
        legs.insert(0, ("oracle", ablmc.simulate_pairs(pr, level, first, n, xi=xi)))
    for mode, got in legs:
        tol = 1e-12 if mode == "oracle" else 1e-10
        S = stats[mode]
        for i in range(n):
            w, g = want[i], got[i]
            ok_ref = bool(w.fine.ok) and bool(w.coarse.ok)
            if ok_ref != bool(g["fok"]):
                flags_bad.append((trial, i, mode, "ok flag", ok_ref, int(g["fok"])))
                continue
            if not ok_ref:
                failed_paths += mode == "oracle"
                continue
            S["pairs"] += 1
            ints_w = (w.fine.parity, w.fine.n_refl, w.coarse.parity, w.coarse.n_refl)
            ints_g = (int(g["fpar"]), int(g["fn"]), int(g["cpar"]), int(g["cn"]))
            vw = (w.fine.x, w.fine.u, w.coarse.x, w.coarse.u)
            vg = (float(g["fx"]), float(g["fu"]), float(g["cx"]), float(g["cu"]))
            r = max(rel(a, b) for a, b in zip(vg, vw))
            B = S["by_ig"][int(c.integrator)]
            B[0] += 1
            if vg == vw and ints_g == ints_w:
                S["bit"] += 1
                B[1] += 1
            S["ints"] += ints_g != ints_w
            S["worst"] = max(S["worst"], r)
            if ints_g != ints_w or r > tol or (mode == "oracle" and c.integrator == Ig.se and vg != vw):
                S["out"].append((trial, i, int(c.integrator), M, r, ints_g, ints_w))
                B[2] += 1
            else:
                S["max_rel"] = max(S["max_rel"], r)
for b in flags_bad[:10]:
    print("FLAG MISMATCH", b)
for m, S in stats.items():
    for o in S["out"][:10]:
        print("OUTSIDE", m, o)
    print(f"{m}: {S['pairs']} pairs, {S['bit']} bit-identical, max rel diff within tolerance "
          f"{S['max_rel']:.2e}, {len(S['out'])} outside tolerance (worst {S['worst']:.2e}), "
          f"{S['ints']} parity / reflection-count mismatches; per integrator (pairs, bit-identical, "
          f"outside): se {S['by_ig'][0]}, gl {S['by_ig'][1]}, baoab {S['by_ig'][2]}")
print(f"fuzz_reference: trials {first_trial}..{first_trial + n_trials - 1}: {problems} problems vs "
      f"the unmodified reference, {failed_paths} failed paths agreed, {len(flags_bad)} flag "
      f"mismatches, {time.time() - t0:.0f} s")
sys.exit(1 if (flags_bad or stats["oracle"]["out"]) and not ADAPTIVE else 0)
