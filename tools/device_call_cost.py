import ctypes as C, sys, time
sys.path.insert(0, ".")
import torch
from paper_1612_07717_b200 import ablmc, capi
lib = capi.load()
stream = torch.cuda.Stream(); lib.ablmc_set_stream(C.c_void_p(stream.cuda_stream))
for ig in (ablmc.Integrator.se, ablmc.Integrator.baoab):
    pr = ablmc.Problem.make(ablmc.ModelParams(), ig, ablmc.QoISpec(), 0.5, 0.1, 1.0, 1, 42)
    pc = C.byref(pr._c)
    for n in (256, 65536, 1 << 20, 1 << 22):
        for _ in range(20): lib.ablmc_accumulate_device(pc, 0, 0, n)
        torch.cuda.synchronize()
        # host time per call (no sync) and device time per call
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter(); s.record(stream)
        for _ in range(200): lib.ablmc_accumulate_device(pc, 0, 0, n)
        e.record(stream); host = (time.perf_counter() - t) / 200
        torch.cuda.synchronize()
        print(f"{ig.name} level 0 n={n}: host {host*1e6:.1f} us/call issue, device {s.elapsed_time(e)/200*1e3:.1f} us/call")
