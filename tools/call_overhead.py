"""Per-call latency of a minimal accumulate_samples through the raw C ABI
(no Python wrapper work inside the timed loop)."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1612_07717_b200 import ablmc, capi  # noqa: E402

lib = capi.load()
pr = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.se, ablmc.QoISpec(), 0.5, 0.1, 1.0, 1, 42)
sy, sy2 = np.zeros(1), np.zeros(1)
v = capi.LevelStatsC()
v.dim = 1
v.sum_y = sy.ctypes.data_as(C.POINTER(C.c_double))
v.sum_y2 = sy2.ctypes.data_as(C.POINTER(C.c_double))
pc, pv = C.byref(pr._c), C.byref(v)
for n, level in ((256, 0), (256, 1), (4096, 1), (65536, 1)):
    for _ in range(50):
        lib.ablmc_accumulate_samples(pc, level, 0, n, pv)
    t = time.perf_counter()
    for _ in range(500):
        lib.ablmc_accumulate_samples(pc, level, 0, n, pv)
    print(f"n={n} level={level}: {(time.perf_counter() - t) / 500 * 1e6:.1f} us/call, "
          f"launches {lib.ablmc_last_launch_count()}")
