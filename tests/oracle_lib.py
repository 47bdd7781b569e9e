"""ctypes access to the parity checkers under oracle/ (TEST INFRASTRUCTURE).

* ``orc()`` — oracle/build/libablmc_oracle.so, the C restatement.
* ``ref()`` — oracle/_ref/libablmc_ref.so, the unmodified reference headers
  behind an extern "C" shim (None if it was never built).
Both share the C-ABI structs of include/ablmc_b200.h (paper_1612_07717_b200.capi).
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

from paper_1612_07717_b200 import capi

ROOT = Path(__file__).resolve().parents[1]
ORC_SO = ROOT / "oracle" / "build" / "libablmc_oracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libablmc_ref.so"

P = C.POINTER
_orc = None
_ref = None


def _ensure_built() -> None:
    if not ORC_SO.exists():
        subprocess.run(["make", "-s", "-f", str(ROOT / "oracle" / "Makefile")], check=True)


class OrcState(C.Structure):
    _fields_ = [("x", C.c_double), ("u", C.c_double), ("parity", C.c_int), ("n_refl", C.c_int64)]


class OrcCoeffs(C.Structure):
    _fields_ = [("sigma_u2", C.c_double), ("lambda_", C.c_double), ("sigma", C.c_double),
                ("dsigma_u2", C.c_double)]


def orc() -> C.CDLL:
    global _orc
    if _orc is None:
        _ensure_built()
        L = C.CDLL(str(ORC_SO))
        sig = {
            "orc_philox4x32": (None, [P(C.c_uint32), P(C.c_uint32), P(C.c_uint32)]),
            "orc_splitmix64": (C.c_uint64, [C.c_uint64]),
            "orc_stream_key": (None, [C.c_uint64, C.c_uint32, P(C.c_uint32)]),
            "orc_bits_to_unit": (C.c_double, [C.c_uint32, C.c_uint32]),
            "orc_normal_at": (C.c_double, [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64]),
            "orc_coarse_noise_se": (C.c_double, [C.c_double, C.c_double, C.c_int, C.c_int, C.c_int]),
            "orc_coarse_noise_gl": (C.c_double, [C.c_double, C.c_double, C.c_double, C.c_double,
                                                 C.c_int, C.c_int, C.c_int]),
            "orc_sde_coeffs": (OrcCoeffs, [C.c_double, P(capi.ModelParamsC)]),
            "orc_dv_dx": (C.c_double, [P(OrcCoeffs), C.c_double]),
            "orc_reflect": (C.c_int, [P(C.c_double), P(C.c_double), C.c_double, P(C.c_int),
                                      P(C.c_int64), P(C.c_int)]),
            "orc_se_stability_limit": (C.c_double, [P(capi.ModelParamsC)]),
            "orc_step": (C.c_int, [C.c_int, P(OrcState), C.c_double, C.c_double,
                                   P(capi.ModelParamsC), C.c_int, P(C.c_int)]),
            "orc_simulate_pair": (C.c_int, [C.c_int, P(capi.ModelParamsC), C.c_double, C.c_double,
                                            C.c_double, C.c_int64, C.c_uint64, C.c_uint32,
                                            C.c_uint64, P(C.c_double), C.c_int, P(OrcState),
                                            P(OrcState)]),
            "orc_simulate_path": (C.c_int, [C.c_int, P(capi.ModelParamsC), C.c_double, C.c_double,
                                            C.c_double, C.c_int64, C.c_uint64, C.c_uint32,
                                            C.c_uint64, P(C.c_double), P(OrcState)]),
            "orc_simulate_pair_adaptive": (C.c_int, [C.c_int, P(capi.ModelParamsC), C.c_double,
                                                     C.c_double, C.c_double, C.c_double,
                                                     C.c_double, C.c_uint64, C.c_uint32,
                                                     C.c_uint64, P(C.c_double), C.c_int,
                                                     P(OrcState), P(OrcState), P(C.c_int64)]),
            "orc_simulate_path_adaptive": (C.c_int, [C.c_int, P(capi.ModelParamsC), C.c_double,
                                                     C.c_double, C.c_double, C.c_double,
                                                     C.c_double, C.c_uint64, C.c_uint32,
                                                     C.c_uint64, P(C.c_double), P(OrcState),
                                                     P(C.c_int64)]),
            "orc_set_device_math": (None, [C.c_int]),
            "orc_set_profile": (None, [C.c_int, C.c_double, C.c_double, C.c_double, C.c_double,
                                       C.c_double]),
            "orc_build_smoothing_polynomial": (C.c_int, [C.c_int, P(C.c_double)]),
            "orc_evaluate": (None, [P(capi.QoISpecC), P(C.c_double), C.c_int, C.c_double,
                                    P(C.c_double)]),
            "orc_accumulate_samples": (C.c_int, [P(capi.ProblemC), C.c_int, C.c_int64, C.c_int64,
                                                 P(capi.LevelStatsC)]),
            "orc_accumulate_paths": (C.c_int, [P(capi.ProblemC), C.c_int64, C.c_uint32, C.c_int64,
                                               C.c_int64, P(capi.LevelStatsC)]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        _orc = L
    return _orc


def ref() -> C.CDLL | None:
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            return None
        L = C.CDLL(str(REF_SO))
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_philox4x32": (None, [P(C.c_uint32), P(C.c_uint32), P(C.c_uint32)]),
            "ref_splitmix64": (C.c_uint64, [C.c_uint64]),
            "ref_normals": (None, [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_int64,
                                   P(C.c_double)]),
            "ref_sde_coeffs": (None, [C.c_double, P(capi.ModelParamsC), P(C.c_double)]),
            "ref_model_values": (C.c_int, [C.c_double, C.c_double, P(capi.ModelParamsC),
                                           P(C.c_double)]),
            "ref_se_stability_limit": (C.c_double, [P(capi.ModelParamsC)]),
            "ref_coarse_noise_se": (C.c_double, [C.c_double, C.c_double, C.c_int, C.c_int, C.c_int]),
            "ref_coarse_noise_gl": (C.c_double, [C.c_double, C.c_double, C.c_double, C.c_double,
                                                 C.c_int, C.c_int, C.c_int]),
            "ref_reflect": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_int, C.c_int64,
                                      P(C.c_double), P(C.c_int), P(C.c_int64)]),
            "ref_step": (C.c_int, [C.c_int, P(capi.PathStateC), C.c_double, C.c_double,
                                   P(capi.ModelParamsC), C.c_int, P(C.c_int)]),
            "ref_extended_path": (None, [C.c_int, P(capi.ModelParamsC), C.c_double, C.c_double,
                                         C.c_double, C.c_int64, P(C.c_double), P(C.c_double),
                                         P(C.c_int)]),
            "ref_pair_states": (None, [P(capi.ProblemC), C.c_int, C.c_int64, C.c_int64,
                                       P(capi.PairStateC)]),
            "ref_path_states": (None, [P(capi.ProblemC), C.c_int64, C.c_uint32, C.c_int64,
                                       C.c_int64, P(capi.PathStateC)]),
            "ref_build_smoothing_polynomial": (C.c_int, [C.c_int, P(C.c_double)]),
            "ref_evaluate": (None, [P(capi.QoISpecC), C.c_double, P(C.c_double)]),
            "ref_accumulate_samples": (C.c_int, [P(capi.ProblemC), C.c_int, C.c_int64, C.c_int64,
                                                 C.c_int, P(capi.LevelStatsC), P(C.c_double)]),
            "ref_accumulate_paths": (C.c_int, [P(capi.ProblemC), C.c_int64, C.c_uint32, C.c_int64,
                                               C.c_int64, C.c_int, P(capi.LevelStatsC),
                                               P(C.c_double)]),
            "ref_decay_sweep": (C.c_int, [P(capi.ProblemC), C.c_int, C.c_int, C.c_int64, C.c_int,
                                          P(capi.DecayRowC)]),
            "ref_run_mlmc": (C.c_int, [P(capi.ProblemC), C.c_double, P(capi.MlmcOptionsC),
                                       C.c_int, P(capi.RunResultC)]),
            "ref_run_stmc": (C.c_int, [P(capi.ProblemC), C.c_int64, C.c_double, C.c_int64,
                                       C.c_int, P(capi.RunResultC)]),
            "ref_cost_sweep": (C.c_int, [P(capi.ProblemC), C.c_int, P(C.c_double), C.c_int,
                                         C.c_double, C.c_double, C.c_int, P(capi.CostRowC)]),
            "ref_result_json": (C.c_int64, [P(capi.RunConfigC), P(capi.RunResultC), C.c_int64,
                                            C.c_char_p, C.c_int64]),
            "ref_variance_decay_csv": (C.c_int64, [P(capi.DecayRowC), C.c_int, C.c_char_p,
                                                   C.c_int64]),
            "ref_cost_sweep_csv": (C.c_int64, [P(capi.CostRowC), C.c_int, C.c_int, C.c_char_p,
                                               C.c_int64]),
            "ref_pdf_csv": (C.c_int64, [P(C.c_double), C.c_int, P(C.c_double), P(C.c_double),
                                        C.c_char_p, C.c_int64]),
        }
        for k, (r, a) in sig.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        _ref = L
    return _ref


# ------------------------------------------------------------ convenience
def default_params(**kw) -> capi.ModelParamsC:
    p = capi.ModelParamsC(1.3, 0.5, 0.2, 1.0, 0.01, 1.0, 1.0)
    for k, v in kw.items():
        setattr(p, k, v)
    return p


class Stats:
    """Host LevelStats buffers usable by orc/ref/product accumulate calls."""

    def __init__(self, dim: int = 1, level: int = 0, h: float = 0.0):
        self.sum_y = np.zeros(dim)
        self.sum_y2 = np.zeros(dim)
        self.c = capi.LevelStatsC()
        self.c.level, self.c.h, self.c.dim = level, h, dim
        self.c.sum_y = self.sum_y.ctypes.data_as(P(C.c_double))
        self.c.sum_y2 = self.sum_y2.ctypes.data_as(P(C.c_double))

    @property
    def n(self):
        return self.c.n

    @property
    def failed(self):
        return self.c.failed

    @property
    def cost_steps(self):
        return self.c.cost_steps


def orc_normals(seed, level, idx, k0, n):
    L = orc()
    return np.array([L.orc_normal_at(seed, level, idx, k0 + j) for j in range(n)])


def ref_normals(seed, level, idx, k0, n):
    out = np.zeros(n)
    ref().ref_normals(seed, level, idx, k0, n, out.ctypes.data_as(P(C.c_double)))
    return out


def orc_pair(ig, params, x0, u0, T, M, seed, level, idx, xi=None, signs_on=1):
    f, c = OrcState(), OrcState()
    xp = None
    if xi is not None:
        xi = np.ascontiguousarray(xi, dtype=np.float64)
        xp = xi.ctypes.data_as(P(C.c_double))
    rc = orc().orc_simulate_pair(ig, C.byref(params), x0, u0, T, M, seed, level, idx, xp,
                                 signs_on, C.byref(f), C.byref(c))
    return rc, f, c


def orc_path(ig, params, x0, u0, T, M, seed, level, idx, xi=None):
    s = OrcState()
    xp = None
    if xi is not None:
        xi = np.ascontiguousarray(xi, dtype=np.float64)
        xp = xi.ctypes.data_as(P(C.c_double))
    rc = orc().orc_simulate_path(ig, C.byref(params), x0, u0, T, M, seed, level, idx, xp,
                                 C.byref(s))
    return rc, s


def _xi_ptr(xi):
    if xi is None:
        return None, None
    xi = np.ascontiguousarray(xi, dtype=np.float64)
    return xi, xi.ctypes.data_as(P(C.c_double))


def orc_pair_adaptive(ig, params, x0, u0, T, h_base, x_adapt, seed, level, idx, signs_on=1,
                      xi=None):
    """xi: explicit NoiseStream::next() sequence (long enough for the pair's
    data-dependent draw count), else the Philox stream."""
    f, c, n = OrcState(), OrcState(), C.c_int64(0)
    keep, xp = _xi_ptr(xi)
    rc = orc().orc_simulate_pair_adaptive(ig, C.byref(params), x0, u0, T, h_base, x_adapt, seed,
                                          level, idx, xp, signs_on, C.byref(f), C.byref(c),
                                          C.byref(n))
    return rc, f, c, n.value


def orc_path_adaptive(ig, params, x0, u0, T, h_base, x_adapt, seed, level, idx, xi=None):
    s, n = OrcState(), C.c_int64(0)
    keep, xp = _xi_ptr(xi)
    rc = orc().orc_simulate_path_adaptive(ig, C.byref(params), x0, u0, T, h_base, x_adapt, seed,
                                          level, idx, xp, C.byref(s), C.byref(n))
    return rc, s, n.value
