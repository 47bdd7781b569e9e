"""MLMC wall time vs level-sampler (K1) time: how much of a run_mlmc call is
outside the sampler kernels (host driver, launches, the per-round sync and
result copies).  BASELINE config 3 problem (BAOAB, reference profile,
x0 = 0.5, u0 = 0.1, T = 1, M0 = 1, seed 42).

  python tools/mlmc_profile.py > profiles/r2_mlmc_profile.txt
"""
import ctypes as C
import sys
import time

sys.path.insert(0, '.')
from paper_1612_07717_b200 import ablmc, capi  # noqa: E402

lib = capi.load()
pr = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.baoab, ablmc.QoISpec(), 0.5, 0.1,
                        1.0, 1, 42)
ablmc.run_mlmc(pr, 1e-4)  # warm-up: context, workspaces
for eps in (1e-4, 3e-5, 1e-5):
    best = None
    for _ in range(5):
        lib.ablmc_set_profiling(1)
        t = time.perf_counter()
        r = ablmc.run_mlmc(pr, eps)
        wall = time.perf_counter() - t
        tot, cnt = C.c_double(), C.c_int64()
        lib.ablmc_level_kernel_times(C.byref(tot), C.byref(cnt))
        lib.ablmc_set_profiling(0)
        row = (r.wall_seconds * 1e3, wall * 1e3, tot.value, cnt.value, [s.n for s in r.level_stats])
        if best is None or row[0] < best[0]:
            best = row
    drv, py, k1, n, N = best
    # the same run without the per-launch profiling events
    plain = min(ablmc.run_mlmc(pr, eps).wall_seconds for _ in range(5)) * 1e3
    print(f"eps {eps:g}: driver wall {plain:.3f} ms ({drv:.3f} ms with per-launch events; python "
          f"call {py:.3f} ms), K1 {k1:.3f} ms over {n} launches -> {100 * (1 - k1 / plain):.1f}% "
          f"of the driver wall outside K1; N_l {N}")
