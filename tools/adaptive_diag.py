"""Diagnose device vs oracle differences of adaptive pairs (GPU box)."""
import sys
sys.path[:0] = ["tests", "."]
import numpy as np
import oracle_lib as O
from paper_1612_07717_b200 import ablmc

Ig = ablmc.Integrator
cfgs = [dict(ig=Ig.gl, x0=0.012, m0=20, xa=0.3, level=4, signs=False, n=8),
        dict(ig=Ig.gl, x0=0.05, m0=40, xa=0.05, level=2, signs=True, n=96)]
for cfg in cfgs:
    pr = ablmc.Problem.make(ablmc.ModelParams(), cfg["ig"], ablmc.QoISpec(), cfg["x0"], 0.1, 1.0,
                            cfg["m0"], 31, ablmc.SampleOptions(signs_on=cfg["signs"], adaptive=True,
                                                               x_adapt=cfg["xa"]))
    c = pr._c
    level = cfg["level"]
    M = c.m0 << level
    got = ablmc.simulate_pairs(pr, level, 1000, cfg["n"])
    for i in range(cfg["n"]):
        xi = ablmc.normals(c.seed, level, 1000 + i, 0, 256 * M + 257)
        xg = np.array(O.orc_normals(c.seed, level, 1000 + i, 0, 64))
        rc, f, cc, st = O.orc_pair_adaptive(c.integrator, c.params, c.x0, c.u0, c.T, c.T / M,
                                            c.x_adapt, c.seed, level, 1000 + i, c.signs_on, xi=xi)
        rc2, f2, cc2, st2 = O.orc_pair_adaptive(c.integrator, c.params, c.x0, c.u0, c.T, c.T / M,
                                                c.x_adapt, c.seed, level, 1000 + i, c.signs_on)
        g = got[i]
        d = abs(g["fx"] - f.x) + abs(g["cx"] - cc.x)
        if d > 1e-9 or i < 2:
            print(cfg["ig"].name, level, i, "dev", g["fx"], g["cx"], g["fpar"], g["fn"], g["cpar"],
                  g["cn"])
            print("   orc(devxi)", f.x, cc.x, f.parity, f.n_refl, cc.parity, cc.n_refl, st, rc)
            print("   orc(glibc)", f2.x, cc2.x, f2.parity, f2.n_refl, cc2.parity, cc2.n_refl, st2, rc2)
            print("   max|xi dev - glibc| over 64:", np.max(np.abs(xi[:64] - xg)))
