import time, sys
sys.path.insert(0,'.')
from paper_1612_07717_b200 import ablmc
pr = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.baoab, ablmc.QoISpec(), 0.5, 0.1, 1.0, 1, 42)
for n in (1000, 10000, 100000, 1000000):
    for level in (0, 3):
        st = ablmc.LevelStats().init(level, pr.h_level(level), 1)
        ablmc.accumulate_samples(st, 0, n, pr, level)
        t = time.perf_counter()
        for i in range(20):
            ablmc.accumulate_samples(st, 0, n, pr, level)
        dt = (time.perf_counter() - t) / 20
        print(f"n={n} level={level}: {dt*1e6:.1f} us/call")
t = time.perf_counter(); r = ablmc.run_mlmc(pr, 1e-4); print("mlmc 1e-4", (time.perf_counter()-t)*1e3, "ms", [s.n for s in r.level_stats])
