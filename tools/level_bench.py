"""One timed device accumulate call of a chosen level sampler (for A/B runs
and ncu captures of a single configuration).
usage: python tools/level_bench.py [--ig se|gl|baoab] [--level L] [--n N] [--fp32]
                                   [--profile reference|constant|floored] [--x0 X] [--m0 M]"""
import argparse
import ctypes as C
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1612_07717_b200 import ablmc, capi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ig", default="se")
ap.add_argument("--level", type=int, default=10)
ap.add_argument("--n", type=int, default=1 << 22)
ap.add_argument("--fp32", action="store_true")
ap.add_argument("--profile", default="reference")
ap.add_argument("--x0", type=float, default=0.5)
ap.add_argument("--m0", type=int, default=1)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--bins", type=int, default=0, help="binned-field QoI with this many equidistant bins")
ap.add_argument("--delta", type=float, default=0.1)
ap.add_argument("--random-u0", action="store_true")
a = ap.parse_args()
lib = capi.load()
stream = torch.cuda.Stream()
lib.ablmc_set_stream(C.c_void_p(stream.cuda_stream))
q = (ablmc.QoISpec(kind=ablmc.QoIKind.binned_field, bin_edges=ablmc.equidistant_edges(a.bins, 1.0),
                   delta=a.delta) if a.bins else ablmc.QoISpec())
pr = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator[a.ig], q, a.x0,
                        0.0 if a.random_u0 else 0.1, 1.0, a.m0, 42, profile=ablmc.Profile[a.profile],
                        fp32=a.fp32, random_u0=a.random_u0)
pc = C.byref(pr._c)
lib.ablmc_accumulate_device(pc, a.level, 0, a.n)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(stream)
for _ in range(a.reps):
    lib.ablmc_accumulate_device(pc, a.level, 0, a.n)
e.record(stream)
torch.cuda.synchronize()
ms = s.elapsed_time(e) / a.reps
mf = a.m0 << a.level
print(json.dumps({"ig": a.ig, "level": a.level, "n": a.n, "fp32": a.fp32, "profile": a.profile,
                  "bins": a.bins, "x0": a.x0,
                  "ms": ms, "fine_path_steps_per_s": a.n * mf / (ms * 1e-3)}))
