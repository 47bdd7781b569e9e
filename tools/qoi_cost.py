"""Throughput of the level sampler per QoI kind at low and high levels
(config 4 shape: GL, x0 = 0.01, 64 bins) — device-resident accumulate calls."""
import ctypes as C
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1612_07717_b200 import ablmc  # noqa: E402

ablmc.init(0)
lib = ablmc.lib()
edges = ablmc.equidistant_edges(64, 1.0)
for name, q in [("mean", ablmc.QoISpec()),
                ("binned64", ablmc.QoISpec(kind=ablmc.QoIKind.binned_field, bin_edges=edges))]:
    pr = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.gl, q, 0.01, 0.1, 1.0, 1, 7)
    for level in (0, 1, 3, 6, 10):
        n = 1 << 24 if level < 6 else 1 << 22
        lib.ablmc_accumulate_device(C.byref(pr._c), level, 0, n)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            lib.ablmc_accumulate_device(C.byref(pr._c), level, 0, n)
        acc = ablmc.LevelStats().init(level, pr.h_level(level), pr.dim())
        v = acc._view()
        lib.ablmc_fetch_device_result(C.byref(pr._c), level, C.byref(v))
        dt = (time.perf_counter() - t0) / 3
        print(f"{name:9s} level {level:2d}: {n / dt:.3e} samples/s, {n * (1 << level) / dt:.3e} path-steps/s")
