"""MLMC wall time vs sampler-kernel time: how much of a run_mlmc call is
outside the library's kernels (host driver, launch latency, the per-round
synchronisation).  BASELINE config 3 problem (BAOAB, reference profile,
x0 = 0.5, u0 = 0.1, T = 1, M0 = 1, seed 42).  The driver wall is the C
driver's own clock (best of 5 plain runs); the kernel time is the sum of the
kernel durations of one run in the CUDA activity trace (CUPTI via
torch.profiler), which stays accurate under the tracer's launch overhead.

  python tools/mlmc_profile.py > profiles/r2_mlmc_profile.txt
"""
import json
import sys
import tempfile

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, '.')
from paper_1612_07717_b200 import ablmc  # noqa: E402

ablmc.init(0)
pr = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.baoab, ablmc.QoISpec(), 0.5, 0.1,
                        1.0, 1, 42)
for _ in range(3):
    ablmc.run_mlmc(pr, 1e-4)  # warm-up: context, workspaces
for eps in (1e-4, 3e-5, 1e-5):
    plain = min(ablmc.run_mlmc(pr, eps).wall_seconds for _ in range(5)) * 1e3
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        r = ablmc.run_mlmc(pr, eps)
        torch.cuda.synchronize()
    with tempfile.NamedTemporaryFile(suffix=".json") as f:
        prof.export_chrome_trace(f.name)
        ev = json.load(open(f.name))["traceEvents"]
    ks = sorted((e for e in ev if e.get("ph") == "X" and e.get("cat") == "kernel"),
                key=lambda e: e["ts"])
    kern = sum(e["dur"] for e in ks) * 1e-3
    # device-busy time: the union of the kernel intervals (a batch's levels
    # run concurrently on their lanes, so their durations overlap)
    busy, end = 0.0, None
    for e in ks:
        b, f = e["ts"], e["ts"] + e["dur"]
        if end is None or b > end:
            busy += f - b
            end = f
        elif f > end:
            busy += f - end
            end = f
    busy *= 1e-3
    print(f"eps {eps:g}: driver wall {plain:.3f} ms, kernels {kern:.3f} ms summed over {len(ks)} "
          f"launches, device busy {busy:.3f} ms -> {100 * (1 - busy / plain):.1f}% of the driver "
          f"wall with no kernel running; N_l {[s.n for s in r.level_stats]}")
