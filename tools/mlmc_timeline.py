"""GPU timeline of one run_mlmc call (BASELINE config 3 problem) from the
CUDA activity trace (torch.profiler / CUPTI): kernels and copies with their
start/end times, the gaps between them, and the share of the driver's wall
time during which no kernel of the library runs.

  python tools/mlmc_timeline.py [eps] > profiles/r2_mlmc_timeline.txt
"""
import json
import sys
import tempfile

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_1612_07717_b200 import ablmc  # noqa: E402

eps = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-4
ablmc.init(0)
pr = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.baoab, ablmc.QoISpec(), 0.5, 0.1,
                        1.0, 1, 42)
for _ in range(3):
    ablmc.run_mlmc(pr, eps)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    r = ablmc.run_mlmc(pr, eps)
    torch.cuda.synchronize()
with tempfile.NamedTemporaryFile(suffix=".json") as f:
    prof.export_chrome_trace(f.name)
    ev = json.load(open(f.name))["traceEvents"]
gpu = sorted((e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")),
             key=lambda e: e["ts"])
rt = sorted((e for e in ev if e.get("ph") == "X" and e.get("cat") == "cuda_runtime"), key=lambda e: e["ts"])
t0 = min(e["ts"] for e in gpu + rt)
print(f"eps {eps:g}: driver wall {r.wall_seconds * 1e6:.0f} us, N_l {[s.n for s in r.level_stats]}")
busy = sum(e["dur"] for e in gpu if e["cat"] == "kernel")
span = gpu[-1]["ts"] + gpu[-1]["dur"] - gpu[0]["ts"]
print(f"GPU activities: {len(gpu)}, kernel time {busy:.0f} us, first->last activity {span:.0f} us, "
      f"kernel share of that span {100 * busy / span:.1f}%")
prev_end = None
for e in gpu:
    gap = "" if prev_end is None else f"gap {e['ts'] - prev_end:7.1f} us"
    name = e["name"].split("(")[0][-48:]
    print(f"  {e['ts'] - t0:9.1f} +{e['dur']:7.1f} us  {e['cat']:10s} {name:48s} {gap}")
    prev_end = e["ts"] + e["dur"]
agg = {}
for e in rt:
    agg.setdefault(e["name"], [0, 0.0])
    agg[e["name"]][0] += 1
    agg[e["name"]][1] += e["dur"]
print("CUDA runtime calls (count, total us):")
for k, (n, d) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:12]:
    print(f"  {k:40s} {n:5d} {d:9.1f}")
