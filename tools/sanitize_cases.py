"""Small calls through every kernel family of libablmc_b200.so, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck): the uniform
sampler (levels 0-5, every integrator, scalar and binned QoIs, fp32-state),
the state kernels, the adaptive sampler and one small MLMC run.  Sizes are
ragged (not multiples of a tile) on purpose.  usage (GPU box):
  compute-sanitizer --tool memcheck python tools/sanitize_cases.py [family ...]
"""
import sys

sys.path.insert(0, ".")
from paper_1612_07717_b200 import ablmc  # noqa: E402

A = ablmc
fam = set(sys.argv[1:]) or {"level", "binned", "fp32", "states", "adaptive", "mlmc"}
A.init(0)
P = A.ModelParams()
n_calls = 0


def acc(pr, level, first, count):
    global n_calls
    st = A.LevelStats().init(level, pr.h_level(level), pr.dim())
    A.accumulate_samples(st, first, count, pr, level)
    n_calls += 1
    return st


if "level" in fam:
    for ig in A.Integrator:
        for q in (A.QoISpec(), A.QoISpec(kind=A.QoIKind.smoothed_indicator),
                  A.QoISpec(kind=A.QoIKind.raw_indicator)):
            pr = A.Problem.make(P, ig, q, 0.05, 0.1, 1.0, 1, 7)
            for level, count in ((0, 5001), (1, 4099), (2, 1027), (5, 777)):
                st = acc(pr, level, 3, count)
                assert st.n + st.failed == count
        # the reference's default M0 = 40 and a release at the ground
        pr = A.Problem.make(P, ig, A.QoISpec(), 0.0, 0.1, 1.0, 40, 11)
        acc(pr, 1, 0, 513)
        # the extension profiles
        for prof in (A.Profile.constant, A.Profile.floored):
            pr = A.Problem.make(P, ig, A.QoISpec(), 0.5, 0.0, 1.0, 1, 5, profile=prof,
                                random_u0=True)
            acc(pr, 3, 0, 1500)
    # several levels in one batch (the concurrent lanes)
    pr = A.Problem.make(P, A.Integrator.baoab, A.QoISpec(), 0.5, 0.0, 1.0, 1, 3)
    reqs = [(A.LevelStats().init(l, pr.h_level(l), 1), 0, 3000 >> l, l) for l in range(5)]
    A.accumulate_levels(reqs, pr)
    n_calls += 1

if "binned" in fam:
    for bins in (64, 300):
        q = A.QoISpec(kind=A.QoIKind.binned_field, delta=0.02,
                      bin_edges=A.equidistant_edges(bins, 1.0))
        for ig in (A.Integrator.se, A.Integrator.gl):
            pr = A.Problem.make(P, ig, q, 0.01, 0.1, 1.0, 1, 9)
            for level, count in ((0, 4100), (3, 1030)):
                st = acc(pr, level, 0, count)
                assert st.n + st.failed == count

if "fp32" in fam:
    for ig in A.Integrator:
        pr = A.Problem.make(P, ig, A.QoISpec(), 0.5, 0.1, 1.0, 1, 7, fp32=True)
        acc(pr, 4, 0, 2049)

if "states" in fam:
    for ig in A.Integrator:
        pr = A.Problem.make(P, ig, A.QoISpec(), 0.05, 0.1, 1.0, 1, 7)
        A.simulate_pairs(pr, 3, 0, 700)
        A.simulate_paths(pr, 8, 0, 700)
        n_calls += 2

if "adaptive" in fam:
    for ig in A.Integrator:
        pr = A.Problem.make(P, ig, A.QoISpec(), 0.05, 0.1, 1.0, 40, 7,
                            A.SampleOptions(adaptive=True, x_adapt=0.05))
        for level, count in ((0, 1500), (2, 700)):
            st = acc(pr, level, 0, count)
            assert st.n + st.failed == count

if "mlmc" in fam:
    pr = A.Problem.make(P, A.Integrator.gl, A.QoISpec(), 0.5, 0.0, 1.0, 1, 42)
    r = A.run_mlmc(pr, 2e-3, A.MlmcOptions(pilot_n=2000, init_n=500))
    n_calls += 1
    assert r.levels_used >= 1

A.finalize()
print(f"sanitize_cases: {n_calls} calls ok ({' '.join(sorted(fam))})")
