import ctypes as C, sys, time
sys.path.insert(0, '.')
from paper_1612_07717_b200 import ablmc, capi
lib = capi.load()
pr = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.baoab, ablmc.QoISpec(), 0.5, 0.1, 1.0, 1, 42)
ablmc.run_mlmc(pr, 1e-4)
for eps in (1e-4, 3e-5):
    lib.ablmc_set_profiling(1)
    t = time.perf_counter(); r = ablmc.run_mlmc(pr, eps); wall = time.perf_counter() - t
    tot = C.c_double(); cnt = C.c_int64()
    lib.ablmc_level_kernel_times(C.byref(tot), C.byref(cnt))
    lib.ablmc_set_profiling(0)
    print(f"eps {eps}: wall {wall*1e3:.2f} ms, K1 total {tot.value:.2f} ms over {cnt.value} launches, N {[s.n for s in r.level_stats]}")
