"""Hex snapshot of level sums over a spread of configurations (uniform and
adaptive, every QoI kind, ragged and multi-super-block counts): run before and
after a change to the reduction to prove bit-identical results.
usage: python tools/bits_snapshot.py OUT.json"""
import json
import sys

sys.path.insert(0, ".")
from paper_1612_07717_b200 import ablmc  # noqa: E402

Ig = ablmc.Integrator
SB = 1 << 22
out = {}
for ig in Ig:
    for qname, q in (("mean", ablmc.QoISpec()),
                     ("smooth", ablmc.QoISpec(kind=ablmc.QoIKind.smoothed_indicator)),
                     ("bins64", ablmc.QoISpec(kind=ablmc.QoIKind.binned_field,
                                              bin_edges=ablmc.equidistant_edges(64, 1.0)))):
        for adaptive in (False, True):
            if adaptive and qname == "bins64" and ig == Ig.baoab:
                continue
            pr = ablmc.Problem.make(ablmc.ModelParams(), ig, q, 0.3, 0.1, 1.0, 4, 11,
                                    ablmc.SampleOptions(adaptive=adaptive, x_adapt=0.2))
            for level, first, count in ((0, 0, 1000), (2, 7, 3 * 4096 + 5),
                                        (1, 3, SB + 12345 if not adaptive else 70000)):
                if adaptive and count > 100000:
                    continue
                st = ablmc.LevelStats().init(level, pr.h_level(level), pr.dim())
                ablmc.accumulate_samples(st, first, count, pr, level)
                out[f"{ig.name}-{qname}-{'ad' if adaptive else 'un'}-l{level}-{count}"] = [
                    [v.hex() for v in st.sum_y[:8]], [v.hex() for v in st.sum_y2[:8]], st.n,
                    st.failed, st.cost_steps]
pr = ablmc.Problem.make(ablmc.ModelParams(), Ig.se, ablmc.QoISpec(), 0.5, 0.1, 1.0, 1, 42)
st = ablmc.LevelStats().init(10, pr.h_level(10), 1)
ablmc.accumulate_samples(st, 0, 2 * SB + 999, pr, 10)
out["se-l10-2sb"] = [[v.hex() for v in st.sum_y], [v.hex() for v in st.sum_y2], st.n, st.cost_steps]
st = ablmc.LevelStats().init(0, 1 / 7, 1)
ablmc.accumulate_paths(st, 3, 50000, pr, 7, 31)
out["paths"] = [[v.hex() for v in st.sum_y], st.n, st.cost_steps]
json.dump(out, open(sys.argv[1], "w"), indent=0)
print(len(out), "entries")
