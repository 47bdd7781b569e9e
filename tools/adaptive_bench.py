"""Throughput of the adaptive sampler (steps actually taken per second) vs
the uniform-grid sampler on the same problem; run on the GPU box."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_1612_07717_b200 import ablmc, capi  # noqa: E402

lib = capi.load()
stream = torch.cuda.Stream()
lib.ablmc_set_stream(C.c_void_p(stream.cuda_stream))
out = {}
for ig in (ablmc.Integrator.se, ablmc.Integrator.gl, ablmc.Integrator.baoab):
    for adaptive in (False, True):
        for level in (0, 3):
            key = f"{ig.name}_{'adaptive' if adaptive else 'uniform'}_l{level}"
            if len(sys.argv) > 1 and key not in sys.argv[1:]:
                continue
            q = ablmc.QoISpec(kind=ablmc.QoIKind.smoothed_indicator)
            pr = ablmc.Problem.make(ablmc.ModelParams(), ig, q, 0.05, 0.1, 1.0, 40, 1,
                                    ablmc.SampleOptions(adaptive=adaptive, x_adapt=0.05))
            pc = C.byref(pr._c)
            n = 1 << 20
            lib.ablmc_accumulate_device(pc, level, 0, n)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(stream)
            lib.ablmc_accumulate_device(pc, level, 0, n)
            e.record(stream)
            torch.cuda.synchronize()
            ms = s.elapsed_time(e)
            import numpy as np
            sy, sy2 = np.zeros(1), np.zeros(1)
            acc = capi.LevelStatsC()
            acc.level, acc.dim = level, 1
            acc.sum_y = sy.ctypes.data_as(C.POINTER(C.c_double))
            acc.sum_y2 = sy2.ctypes.data_as(C.POINTER(C.c_double))
            assert lib.ablmc_fetch_device_result(pc, level, C.byref(acc)) == 0
            out[key] = {"ms": ms, "samples": n, "steps": acc.cost_steps,
                        "steps_per_s": acc.cost_steps / (ms * 1e-3),
                        "samples_per_s": n / (ms * 1e-3), "failed": acc.failed}
            print(key, json.dumps(out[key]), flush=True)
json.dump(out, open("gpurun_out/adaptive_bench.json", "w"), indent=1)
