"""ctypes declarations of the C ABI in ``include/ablmc_b200.h``.

Loads the in-tree ``libablmc_b200.so``; there is no fallback: if the library
is missing the import of the product API raises.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libablmc_b200.so"

ABLMC_OK = 0
ABLMC_ERR_INVALID_ARGUMENT = 1
ABLMC_ERR_RUNTIME = 2
ABLMC_ERR_SAMPLE_FAILURE = 3
ABLMC_ERR_CUDA = 4
ABLMC_ERR_NO_DEVICE = 5
ABLMC_SUPERBLOCK = 1 << 22
ABLMC_NCOUNTS = 3  # {n, failed, cost_steps} per super-block partial
ABLMC_MAX_LEVELS = 24
ABLMC_NCCL_ID_BYTES = 128

SE, GL, BAOAB = 0, 1, 2
QOI_MEAN_POSITION, QOI_SMOOTHED_INDICATOR, QOI_RAW_INDICATOR, QOI_BINNED_FIELD = 0, 1, 2, 3
PROFILE_REFERENCE, PROFILE_CONSTANT, PROFILE_FLOORED = 0, 1, 2


class ModelParamsC(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("kappa_sigma", "kappa_tau", "u_star", "H", "eps_reg", "x_ref", "noise_scale")]


class QoISpecC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("r", C.c_int32), ("a", C.c_double), ("b", C.c_double),
                ("delta", C.c_double), ("n_edges", C.c_int32), ("_pad", C.c_int32),
                ("bin_edges", C.POINTER(C.c_double))]


class ProblemC(C.Structure):
    _fields_ = [("params", ModelParamsC), ("integrator", C.c_int32), ("signs_on", C.c_int32),
                ("qoi", QoISpecC), ("x0", C.c_double), ("u0", C.c_double), ("T", C.c_double),
                ("m0", C.c_int64), ("seed", C.c_uint64), ("adaptive", C.c_int32),
                ("profile", C.c_int32), ("x_adapt", C.c_double), ("random_u0", C.c_int32),
                ("fp32", C.c_int32), ("const_sigma_u", C.c_double), ("const_tau", C.c_double),
                ("sigma_floor", C.c_double), ("tau_min", C.c_double), ("tau_max", C.c_double)]


class LevelStatsC(C.Structure):
    _fields_ = [("level", C.c_int32), ("_pad", C.c_int32), ("h", C.c_double), ("dim", C.c_int64),
                ("sum_y", C.POINTER(C.c_double)), ("sum_y2", C.POINTER(C.c_double)),
                ("n", C.c_int64), ("failed", C.c_int64), ("cost_steps", C.c_int64)]


class PathStateC(C.Structure):
    _fields_ = [("x", C.c_double), ("u", C.c_double), ("parity", C.c_int32), ("ok", C.c_int32),
                ("n_refl", C.c_int64)]


class PairStateC(C.Structure):
    _fields_ = [("fine", PathStateC), ("coarse", PathStateC)]


class MlmcOptionsC(C.Structure):
    _fields_ = [("pilot_n", C.c_int64), ("pilot_levels_max", C.c_int32), ("l_max", C.c_int32),
                ("init_n", C.c_int64), ("use_bias_fit", C.c_int32), ("_pad", C.c_int32),
                ("alpha", C.c_double), ("c1", C.c_double)]


_L = ABLMC_MAX_LEVELS


class RunResultC(C.Structure):
    _fields_ = [("levels_used", C.c_int32), ("n_levels", C.c_int32), ("estimate", C.c_double),
                ("stat_error", C.c_double), ("bias_estimate", C.c_double), ("alpha", C.c_double),
                ("c1", C.c_double), ("total_cost_steps", C.c_int64),
                ("pilot_cost_steps", C.c_int64), ("failed_samples", C.c_int64),
                ("wall_seconds", C.c_double), ("n_warnings", C.c_int32), ("_pad", C.c_int32),
                ("level_n", C.c_int64 * _L), ("level_failed", C.c_int64 * _L),
                ("level_cost", C.c_int64 * _L), ("level_h", C.c_double * _L),
                ("level_sum_y", C.c_double * _L), ("level_sum_y2", C.c_double * _L),
                ("est_vec", C.POINTER(C.c_double)), ("err_vec", C.POINTER(C.c_double)),
                ("level_sum_y_vec", C.POINTER(C.c_double)),
                ("level_sum_y2_vec", C.POINTER(C.c_double)),
                ("warnings_mask", C.c_int32), ("_pad2", C.c_int32)]


class CostRowC(C.Structure):
    _fields_ = [("eps", C.c_double), ("method", C.c_int32), ("integrator", C.c_int32),
                ("cost_steps", C.c_int64), ("wall_seconds", C.c_double), ("estimate", C.c_double),
                ("stat_error", C.c_double)]


class RunConfigC(C.Structure):
    _fields_ = [("model", ModelParamsC), ("method", C.c_int32), ("integrator", C.c_int32),
                ("qoi_kind", C.c_int32), ("qoi_r", C.c_int32), ("qoi_a", C.c_double),
                ("qoi_b", C.c_double), ("qoi_delta", C.c_double), ("qoi_bins", C.c_int32),
                ("adaptive", C.c_int32), ("T", C.c_double), ("m0", C.c_int64),
                ("eps", C.c_double), ("fixed_n", C.c_int64), ("seed", C.c_uint64),
                ("x0", C.c_double), ("u0", C.c_double), ("x_adapt", C.c_double),
                ("coupling_signs", C.c_int32), ("workers", C.c_int32), ("timings", C.c_int32),
                ("_pad", C.c_int32), ("output_dir", C.c_char_p)]


class DecayRowC(C.Structure):
    _fields_ = [("level", C.c_int32), ("_pad", C.c_int32), ("h", C.c_double), ("var_y", C.c_double),
                ("mean_y", C.c_double), ("se_mean", C.c_double), ("n", C.c_int64),
                ("cost_steps", C.c_int64)]


P = C.POINTER
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, P(C.c_double), C.c_int64, P(C.c_double))
# name -> (restype, argtypes): every symbol include/ablmc_b200.h declares.
SIGNATURES = {
    "ablmc_set_collective": (C.c_int, [C.c_int, C.c_int, ALLGATHER_FN, C.c_void_p]),
    "ablmc_nccl_unique_id": (C.c_int, [P(C.c_ubyte)]),
    "ablmc_init_group": (C.c_int, [C.c_int, C.c_int, C.c_int, P(C.c_ubyte)]),
    "ablmc_init_devices": (C.c_int, [C.c_int, P(C.c_int)]),
    "ablmc_init_loopback": (C.c_int, [C.c_int, C.c_int]),
    "ablmc_group_info": (C.c_int, [P(C.c_int), P(C.c_int), P(C.c_int), P(C.c_int)]),
    "ablmc_last_collective_count": (C.c_int64, []),
    "ablmc_gather_layout": (C.c_int, [C.c_int, C.c_int, C.c_int, P(C.c_int64), P(C.c_int64),
                                      P(C.c_int64), P(C.c_int64)]),
    "ablmc_merge_gathered": (C.c_int, [C.c_int, C.c_int, C.c_int, P(C.c_int64), P(C.c_double),
                                       P(P(LevelStatsC))]),
    "ablmc_abi_version": (C.c_int, []),
    "ablmc_init": (C.c_int, [C.c_int]),
    "ablmc_finalize": (C.c_int, []),
    "ablmc_last_error": (C.c_char_p, []),
    "ablmc_set_stream": (C.c_int, [C.c_void_p]),
    "ablmc_problem_defaults": (None, [P(ProblemC)]),
    "ablmc_problem_validate": (C.c_int, [P(ProblemC)]),
    "ablmc_h_level": (C.c_double, [P(ProblemC), C.c_int]),
    "ablmc_qoi_dim": (C.c_int64, [P(ProblemC)]),
    "ablmc_check_se_stability": (C.c_int, [P(ProblemC), C.c_double]),
    "ablmc_check_failure_budget": (C.c_int, [P(LevelStatsC)]),
    "ablmc_accumulate_samples": (C.c_int, [P(ProblemC), C.c_int, C.c_int64, C.c_int64,
                                           P(LevelStatsC)]),
    "ablmc_accumulate_levels": (C.c_int, [P(ProblemC), C.c_int, P(C.c_int), P(C.c_int64),
                                          P(C.c_int64), P(P(LevelStatsC))]),
    "ablmc_accumulate_paths": (C.c_int, [P(ProblemC), C.c_int64, C.c_uint32, C.c_int64,
                                         C.c_int64, P(LevelStatsC)]),
    "ablmc_num_superblocks": (C.c_int64, [C.c_int64]),
    "ablmc_accumulate_partials": (C.c_int, [P(ProblemC), C.c_int, C.c_int64, C.c_uint32,
                                            C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                            P(C.c_double), P(C.c_int64)]),
    "ablmc_merge_partials": (C.c_int, [P(ProblemC), C.c_int, C.c_int64, C.c_int64,
                                       P(C.c_double), P(C.c_int64), P(LevelStatsC)]),
    "ablmc_accumulate_device": (C.c_int, [P(ProblemC), C.c_int, C.c_int64, C.c_int64]),
    "ablmc_fetch_device_result": (C.c_int, [P(ProblemC), C.c_int, P(LevelStatsC)]),
    "ablmc_copy_device_result": (C.c_int, [C.c_void_p, C.c_void_p]),
    "ablmc_last_launch_count": (C.c_int64, []),
    "ablmc_set_profiling": (C.c_int, [C.c_int]),
    "ablmc_level_kernel_times": (C.c_int, [P(C.c_double), P(C.c_int64)]),
    "ablmc_probe_fp64_rate": (C.c_int, [P(C.c_double)]),
    "ablmc_selftest_fastmath": (C.c_int, [C.c_int64, C.c_uint64, P(C.c_uint64)]),
    "ablmc_release_coeffs": (C.c_int, [P(ProblemC), P(C.c_double)]),
    "ablmc_pair_states": (C.c_int, [P(ProblemC), C.c_int, C.c_int64, C.c_int64, P(C.c_double),
                                    P(PairStateC)]),
    "ablmc_path_states": (C.c_int, [P(ProblemC), C.c_int64, C.c_uint32, C.c_int64, C.c_int64,
                                    P(C.c_double), P(PathStateC)]),
    "ablmc_normals": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, C.c_int64,
                                P(C.c_double)]),
    "ablmc_mlmc_options_defaults": (None, [P(MlmcOptionsC)]),
    "ablmc_run_mlmc": (C.c_int, [P(ProblemC), C.c_double, P(MlmcOptionsC), P(RunResultC)]),
    "ablmc_run_stmc": (C.c_int, [P(ProblemC), C.c_int64, C.c_double, C.c_int64,
                                 P(RunResultC)]),
    "ablmc_decay_sweep": (C.c_int, [P(ProblemC), C.c_int, C.c_int, C.c_int64, P(DecayRowC)]),
    "ablmc_cost_sweep": (C.c_int, [P(ProblemC), C.c_int, P(C.c_double), C.c_int, C.c_double,
                                   C.c_double, P(CostRowC)]),
    "ablmc_fit_power_law": (C.c_int, [P(C.c_double), P(C.c_double), C.c_int, P(C.c_double),
                                     P(C.c_double)]),
    "ablmc_estimate_bias_constants": (C.c_int, [P(C.c_double), P(C.c_double), P(C.c_double),
                                                C.c_int, P(C.c_double), P(C.c_double),
                                                P(C.c_double)]),
    "ablmc_choose_levels": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_int64, C.c_double,
                                      C.c_int, P(C.c_int)]),
    "ablmc_allocate_samples": (C.c_int, [P(C.c_double), P(C.c_double), C.c_int, C.c_double,
                                         P(C.c_int64)]),
    "ablmc_build_smoothing_polynomial": (C.c_int, [C.c_int, P(C.c_double)]),
    "ablmc_adaptive_step_size": (C.c_double, [C.c_double, C.c_double, C.c_double,
                                              P(ModelParamsC)]),
    "ablmc_run_config_defaults": (None, [P(RunConfigC)]),
    "ablmc_result_json": (C.c_int64, [P(RunConfigC), P(RunResultC), C.c_int64, C.c_char_p,
                                      C.c_int64]),
    "ablmc_read_result_json": (C.c_int, [C.c_char_p, P(RunConfigC), P(RunResultC), P(C.c_int64),
                                         C.c_char_p, C.c_int64]),
    "ablmc_read_result_json_error": (C.c_char_p, []),
    "ablmc_variance_decay_csv": (C.c_int64, [P(DecayRowC), C.c_int, C.c_char_p, C.c_int64]),
    "ablmc_cost_sweep_csv": (C.c_int64, [P(CostRowC), C.c_int, C.c_int, C.c_char_p, C.c_int64]),
    "ablmc_pdf_csv": (C.c_int64, [P(C.c_double), C.c_int, P(C.c_double), P(C.c_double),
                                  C.c_char_p, C.c_int64]),
}

_lib = None


def load(path: os.PathLike | str | None = None) -> C.CDLL:
    """Load the product library; raises (no fallback) when it is missing."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    # ABLMC_LIB: an alternative in-tree build of the same library (A/B tuning runs)
    p = Path(path) if path else Path(os.environ.get("ABLMC_LIB") or LIB_PATH)
    if not p.exists():
        raise ImportError(
            f"{p} is missing: build it with `python -m paper_1612_07717_b200.build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib
