"""Host cost of one MLMC allocation round: ablmc_accumulate_levels over 4
levels with tiny sample counts (launch + sync + merge dominated), and of a
single tiny accumulate call, through the raw C ABI."""
import ctypes as C
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1612_07717_b200 import ablmc, capi  # noqa: E402

lib = capi.load()
ablmc.init(0)
pr = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.baoab, ablmc.QoISpec(), 0.5, 0.1, 1.0,
                        1, 42)
pc = C.byref(pr._c)
views, keep = [], []
for l in range(4):
    sy, sy2 = np.zeros(1), np.zeros(1)
    v = capi.LevelStatsC()
    v.level, v.dim = l, 1
    v.sum_y = sy.ctypes.data_as(C.POINTER(C.c_double))
    v.sum_y2 = sy2.ctypes.data_as(C.POINTER(C.c_double))
    views.append(v)
    keep += [sy, sy2]
ptrs = (C.POINTER(capi.LevelStatsC) * 4)(*[C.pointer(v) for v in views])
levels = (C.c_int * 4)(0, 1, 2, 3)
firsts = (C.c_int64 * 4)(0, 0, 0, 0)
for n in (256, 10000):
    counts = (C.c_int64 * 4)(n, n, n, n)
    for _ in range(50):
        lib.ablmc_accumulate_levels(pc, 4, levels, firsts, counts, ptrs)
    t = time.perf_counter()
    for _ in range(500):
        lib.ablmc_accumulate_levels(pc, 4, levels, firsts, counts, ptrs)
    print(f"accumulate_levels 4 x {n}: {(time.perf_counter() - t) / 500 * 1e6:.1f} us/call")
for n in (256, 10000):
    for _ in range(50):
        lib.ablmc_accumulate_samples(pc, 1, 0, n, ptrs[0])
    t = time.perf_counter()
    for _ in range(500):
        lib.ablmc_accumulate_samples(pc, 1, 0, n, ptrs[0])
    print(f"accumulate_samples 1 x {n}: {(time.perf_counter() - t) / 500 * 1e6:.1f} us/call")
