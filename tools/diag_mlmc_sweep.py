"""Diagnostic: bench.py's MLMC time-to-eps sweep alone, with the library
bound to a torch stream, optionally after bench.py's per-integrator and
adaptive runs, to locate a first-call cost."""
import ctypes as C
import sys
import time
import types

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1612_07717_b200 import ablmc  # noqa: E402

steps = sys.argv[1:] or ["mlmc"]
ablmc.init(0)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ablmc.set_stream(s.cuda_stream)
lib = ablmc.lib()
a = types.SimpleNamespace(mlmc_eps="1e-4,3e-5,1e-5,3e-6", level=10)
pr = bench.problem_c(2)


def probe(tag):
    for eps in (3e-5, 3e-6):
        t = time.perf_counter()
        ablmc.run_mlmc(pr, eps)
        print(tag, eps, round((time.perf_counter() - t) * 1e3, 2), "ms", flush=True)


probe("start")
for st in steps:
    t = time.perf_counter()
    if st == "per_integrator":
        bench.per_integrator(a, lib, s, 1.8e13, 1.965e9)
    elif st == "adaptive":
        bench.adaptive_rates(lib, s)
    elif st == "device":
        p0 = bench.problem_c(0)
        for _ in range(3):
            lib.ablmc_accumulate_device(C.byref(p0._c), 10, 0, 1 << 25)
        torch.cuda.synchronize()
    elif st == "mlmc":
        res = bench.mlmc_sweep(a)
        for k, v in res.items():
            print("sweep", k, round(v["seconds"] * 1e3, 2), "ms", flush=True)
    print("step", st, round(time.perf_counter() - t, 2), "s", flush=True)
    probe("after " + st)
