import sys, time
sys.path.insert(0, '.')
from paper_1612_07717_b200 import ablmc
ablmc.init(0)
pr = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator.baoab, ablmc.QoISpec(), 0.5, 0.1, 1.0, 1, 42)
for eps in (1e-4, 3e-5, 3e-5, 1e-5, 1e-5, 3e-6, 3e-6):
    t = time.perf_counter(); r = ablmc.run_mlmc(pr, eps); dt = time.perf_counter() - t
    print(eps, round(dt * 1e3, 2), 'ms', round(r.wall_seconds * 1e3, 2), r.levels_used, flush=True)
