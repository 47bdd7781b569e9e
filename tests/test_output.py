"""Driver-facing formats: result.json schema v1 and the
CSV tables must be byte-identical to the reference's own writers
(output.hpp, compiled unmodified into oracle/_ref with the nlohmann/json this
image ships).  Pure host formatting: runs on CPU."""
import ctypes as C

import numpy as np
import pytest

import oracle_lib as O
from paper_1612_07717_b200 import ablmc, capi

P = C.POINTER
R = O.ref()
needs_ref = pytest.mark.skipif(R is None, reason="oracle/_ref not built")


def ref_text(fn, *args):
    fn.restype = C.c_int64
    n = fn(*args, None, 0)
    buf = C.create_string_buffer(n + 1)
    fn(*args, buf, n + 1)
    return buf.raw[:n].decode()


TRICKY = [0.0, 1.0, 0.1, 1e-5, 1e-4, 123456789012345.0, 1e16, 2.5e-310, -3.75, 1 / 3,
          6.02214076e23, 5e-324, 0.5549485498861402]


def synthetic_result(dim, n_levels, rng, warnings_mask):
    r = capi.RunResultC()
    est = rng.normal(size=dim)
    err = np.abs(rng.normal(size=dim)) * 1e-4
    sy = rng.normal(size=(capi.ABLMC_MAX_LEVELS, dim)) * 1e3
    sy2 = np.abs(rng.normal(size=(capi.ABLMC_MAX_LEVELS, dim))) * 1e5
    sy[0, 0] = TRICKY[int(rng.integers(len(TRICKY)))]
    r.est_vec = est.ctypes.data_as(P(C.c_double))
    r.err_vec = err.ctypes.data_as(P(C.c_double))
    r.level_sum_y_vec = sy.ctypes.data_as(P(C.c_double))
    r.level_sum_y2_vec = sy2.ctypes.data_as(P(C.c_double))
    r.levels_used = n_levels - 1
    r.n_levels = n_levels
    r.estimate, r.stat_error = est[0], err[0]
    r.bias_estimate, r.alpha, r.c1 = 4.8e-5, 1.9913, 0.0123
    r.total_cost_steps, r.pilot_cost_steps, r.failed_samples = 14135138554, 55569251, 3
    r.wall_seconds = 0.3242277
    r.warnings_mask = warnings_mask
    for l in range(n_levels):
        r.level_n[l] = int(rng.integers(1, 10**10))
        r.level_failed[l] = int(rng.integers(0, 3))
        r.level_cost[l] = int(rng.integers(1, 10**12))
        r.level_h[l] = 1.0 / (40 << l)
    return r, (est, err, sy, sy2)


@needs_ref
@pytest.mark.parametrize("case", range(8))
def test_result_json_byte_identical(case):
    rng = np.random.default_rng(case)
    dim = [1, 1, 20, 64, 1, 3, 1, 8][case]
    cfg = ablmc.RunConfig(method=ablmc.Method(case % 2), integrator=ablmc.Integrator(case % 3),
                          qoi_kind=ablmc.QoIKind.binned_field if dim > 1 else ablmc.QoIKind.mean_position,
                          qoi_bins=max(dim, 20), eps=TRICKY[case + 2], seed=2**64 - 1 - case,
                          m0=40 << case, fixed_n=case * 1000, timings=bool(case % 3),
                          coupling_signs=case != 4, workers=case + 1, output_dir=f"out/{case}",
                          x0=0.05 * (case + 1), u0=-0.1 * case)
    r, keep = synthetic_result(dim, 1 + case % 5, rng, case % 4)
    cc = cfg.c()
    ours = ablmc._text(ablmc.lib().ablmc_result_json, C.byref(cc), C.byref(r), dim)
    theirs = ref_text(R.ref_result_json, C.byref(cc), C.byref(r), C.c_int64(dim))
    assert ours == theirs
    assert ours.endswith("}\n") and '"schema_version": 1' in ours


@needs_ref
def test_csv_writers_byte_identical():
    rng = np.random.default_rng(3)
    rows = [ablmc.DecayRow(l, 1 / (40 << l), float(rng.random()) * 10 ** -l, TRICKY[l % len(TRICKY)],
                           0.0, int(rng.integers(1, 10**9)), int(rng.integers(1, 10**12)))
            for l in range(9)]
    ours = ablmc.variance_decay_csv(rows)
    arr = (capi.DecayRowC * len(rows))()
    for a, r in zip(arr, rows):
        a.level, a.h, a.var_y, a.mean_y, a.se_mean, a.n, a.cost_steps = (
            r.level, r.h, r.var_y, r.mean_y, r.se_mean, r.n, r.cost_steps)
    assert ours == ref_text(R.ref_variance_decay_csv, arr, len(rows))
    cost = [ablmc.CostRow(e, ablmc.Method(i % 2), ablmc.Integrator(i % 3), 10**i, 0.25 * i,
                          0.13 + i, 1e-4 / (i + 1)) for i, e in enumerate([1e-3, 3e-4, 1e-4, 3e-5])]
    for timings in (True, False):
        ours = ablmc.cost_sweep_csv(cost, timings)
        arr = (capi.CostRowC * len(cost))()
        for a, r in zip(arr, cost):
            a.eps, a.method, a.integrator, a.cost_steps = r.eps, int(r.method), int(r.integrator), r.cost_steps
            a.wall_seconds, a.estimate, a.stat_error = r.wall_seconds, r.estimate, r.stat_error
        assert ours == ref_text(R.ref_cost_sweep_csv, arr, len(cost), int(timings))
    edges = ablmc.equidistant_edges(64, 1.0)
    conc = list(rng.random(64))
    se = list(rng.random(64) * 1e-3)
    e = (C.c_double * 65)(*edges)
    assert ablmc.pdf_csv(edges, conc, se) == ref_text(R.ref_pdf_csv, e, 65, (C.c_double * 64)(*conc),
                                                      (C.c_double * 64)(*se))


@pytest.mark.parametrize("case", range(8))
def test_result_json_read_back(case):
    """output_record_from_json (output.hpp:47-81,125-159): the product reads a
    result.json back to the same record (re-emitted text byte-identical), and
    the reference's own reader agrees byte for byte (the resume path: per-level
    sums reloaded, sampling continues at index n + failed)."""
    rng = np.random.default_rng(100 + case)
    dim = [1, 1, 20, 64, 1, 3, 1, 8][case]
    cfg = ablmc.RunConfig(method=ablmc.Method(case % 2), integrator=ablmc.Integrator(case % 3),
                          qoi_kind=ablmc.QoIKind.binned_field if dim > 1 else ablmc.QoIKind.smoothed_indicator,
                          qoi_bins=max(dim, 20), eps=TRICKY[case + 2], seed=2**64 - 1 - case,
                          m0=40 << case, fixed_n=case * 1000, timings=bool(case % 3),
                          adaptive=case == 5, coupling_signs=case != 4, workers=case + 1,
                          output_dir=f"out/{case}", x0=0.05 * (case + 1), u0=-0.1 * case)
    r, keep = synthetic_result(dim, 1 + case % 5, rng, case % 4)
    cc = cfg.c()
    text = ablmc._text(ablmc.lib().ablmc_result_json, C.byref(cc), C.byref(r), dim)
    cfg2, res2 = ablmc.read_result_json(text)
    assert cfg2 == cfg
    assert len(res2.estimate) == dim and len(res2.level_stats) == 1 + case % 5
    assert ablmc.result_json(cfg2, res2) == text
    if R is not None:
        assert ref_text(R.ref_result_json_roundtrip, text.encode()) == text


def test_result_json_reader_errors():
    cfg = ablmc.RunConfig()
    r, keep = synthetic_result(1, 2, np.random.default_rng(0), 0)
    text = ablmc._text(ablmc.lib().ablmc_result_json, C.byref(cfg.c()), C.byref(r), 1)
    with pytest.raises(RuntimeError, match="schema version 2"):
        ablmc.read_result_json(text.replace('"schema_version": 1', '"schema_version": 2'))
    with pytest.raises(ValueError):
        ablmc.read_result_json(text.replace('"gl"', '"rk4"'))
    with pytest.raises(ValueError):
        ablmc.read_result_json("{not json")
