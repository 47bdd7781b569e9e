"""Small invocations of every kernel family (uniform / adaptive x QoI kinds x
integrators, oracle-mode states, fp32 and extension profiles, MLMC driver)
with ragged tiles: a quick crash / error sweep on the GPU box."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_1612_07717_b200 import ablmc  # noqa: E402

Ig = ablmc.Integrator
mp = ablmc.ModelParams()
for ig in Ig:
    for qoi in (ablmc.QoISpec(), ablmc.QoISpec(kind=ablmc.QoIKind.smoothed_indicator),
                ablmc.QoISpec(kind=ablmc.QoIKind.binned_field,
                              bin_edges=ablmc.equidistant_edges(64, 1.0))):
        for opt in (ablmc.SampleOptions(), ablmc.SampleOptions(adaptive=True, x_adapt=0.1)):
            pr = ablmc.Problem.make(mp, ig, qoi, 0.05, 0.1, 1.0, 8, 3, opt)
            for level in (0, 2):
                st = ablmc.LevelStats().init(level, pr.h_level(level), pr.dim())
                ablmc.accumulate_samples(st, 5, 3000, pr, level)  # ragged tiles
            ablmc.simulate_pairs(pr, 2, 0, 300)
            ablmc.simulate_paths(pr, 8, 0, 300)
    pr = ablmc.Problem.make(mp, ig, ablmc.QoISpec(), 0.5, 0.1, 1.0, 8, 3)
    ablmc.simulate_pairs(pr, 2, 0, 100, xi=np.random.default_rng(0).normal(size=(100, 32)))
    for kw in (dict(fp32=True), dict(profile=ablmc.Profile.floored, random_u0=True),
               dict(profile=ablmc.Profile.constant)):
        pr = ablmc.Problem.make(mp, ig, ablmc.QoISpec(), 0.5, 0.1, 1.0, 8, 3, **kw)
        st = ablmc.LevelStats().init(2, pr.h_level(2), 1)
        ablmc.accumulate_samples(st, 0, 3000, pr, 2)
r = ablmc.run_mlmc(ablmc.Problem.make(mp, Ig.gl, ablmc.QoISpec(), 0.05, 0.1, 1.0, 40, 1), 3e-3)
print("kernel_sweep ok", r.estimate[0])
