"""Python mirror of the reference's ablmc API for the device level sampler.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/ablmc): ``ModelParams`` (model.hpp:28-48),
``QoISpec`` (qoi.hpp:107-142), ``Problem`` (estimators.hpp:26-94),
``LevelStats`` (stats.hpp:26-88), ``accumulate_samples`` (stats.hpp:96-136),
``check_failure_budget`` (stats.hpp:139-143), ``run_mlmc`` / ``run_stmc`` /
``decay_sweep`` (estimators.hpp:230-431).  Every sampling call goes through
the C ABI of ``libablmc_b200.so`` (sm_100a kernels); nothing here computes a
sample on the CPU.

Exceptions: std::invalid_argument -> ``ValueError``; std::runtime_error ->
``RuntimeError``; SampleFailureError -> ``SampleFailureError``; CUDA / no
device -> ``CudaError``.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import capi

_P = C.pointer


class SampleFailureError(RuntimeError):
    """More than 0.01% of a level's samples failed (stats.hpp:19-22)."""


class CudaError(RuntimeError):
    """CUDA failure or no usable sm_100a device."""


class Integrator(enum.IntEnum):
    se = capi.SE
    gl = capi.GL
    baoab = capi.BAOAB


class QoIKind(enum.IntEnum):
    mean_position = capi.QOI_MEAN_POSITION
    smoothed_indicator = capi.QOI_SMOOTHED_INDICATOR
    raw_indicator = capi.QOI_RAW_INDICATOR
    binned_field = capi.QOI_BINNED_FIELD


class Profile(enum.IntEnum):
    reference = capi.PROFILE_REFERENCE
    constant = capi.PROFILE_CONSTANT  # extension (BASELINE config 1), parity unpinned
    floored = capi.PROFILE_FLOORED    # extension (BASELINE configs 2-5 as written), parity unpinned


def lib() -> C.CDLL:
    return capi.load()


def _check(rc: int) -> None:
    if rc == capi.ABLMC_OK:
        return
    msg = lib().ablmc_last_error().decode()
    if rc == capi.ABLMC_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == capi.ABLMC_ERR_RUNTIME:
        raise RuntimeError(msg)
    if rc == capi.ABLMC_ERR_SAMPLE_FAILURE:
        raise SampleFailureError(msg)
    raise CudaError(msg)


def init(device: int = -1) -> None:
    _check(lib().ablmc_init(device))


def init_devices(n: int, devices: Sequence[int] | None = None) -> None:
    """Drive n GPUs from this process (the reference's single-process
    fan-out, stats.hpp:120-135): every accumulate call, and so every driver
    iteration, shards its super-blocks over them and exchanges the partials
    in ONE NCCL all-gather (include/ablmc_b200.h, multi-GPU sharding)."""
    devs = None if devices is None else (C.c_int * n)(*[int(d) for d in devices])
    _check(lib().ablmc_init_devices(int(n), devs))


def init_loopback(n: int, device: int = 0) -> None:
    """Verification transport: n ranks sharing ONE device, the all-gather as
    device-to-device copies (include/ablmc_b200.h, ablmc_init_loopback)."""
    _check(lib().ablmc_init_loopback(int(n), int(device)))


def nccl_unique_id() -> bytes:
    """ncclUniqueId for ablmc_init_group (rank 0 creates it and ships it)."""
    buf = (C.c_ubyte * capi.ABLMC_NCCL_ID_BYTES)()
    _check(lib().ablmc_nccl_unique_id(buf))
    return bytes(buf)


def init_group(device: int, rank: int, world: int, unique_id: bytes) -> None:
    """One process per GPU: join the library's own NCCL communicator."""
    if len(unique_id) != capi.ABLMC_NCCL_ID_BYTES:
        raise ValueError("unique_id must be ABLMC_NCCL_ID_BYTES long")
    buf = (C.c_ubyte * capi.ABLMC_NCCL_ID_BYTES).from_buffer_copy(unique_id)
    _check(lib().ablmc_init_group(int(device), int(rank), int(world), buf))


def group_info() -> dict:
    m, r, w, n = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    lib().ablmc_group_info(C.byref(m), C.byref(r), C.byref(w), C.byref(n))
    return {"mode": m.value, "rank": r.value, "world": w.value, "n_local": n.value}


def last_collective_count() -> int:
    return int(lib().ablmc_last_collective_count())


def finalize() -> None:
    _check(lib().ablmc_finalize())


def set_stream(cuda_stream: int | None) -> None:
    """Launch on this cudaStream_t (e.g. ``torch.cuda.Stream().cuda_stream``).
    0/None selects the library's own stream (NOT the legacy default stream)."""
    lib().ablmc_set_stream(C.c_void_p(cuda_stream) if cuda_stream else None)


@dataclass
class ModelParams:  # model.hpp:28-35
    kappa_sigma: float = 1.3
    kappa_tau: float = 0.5
    u_star: float = 0.2
    H: float = 1.0
    eps_reg: float = 0.01
    x_ref: float = 1.0
    noise_scale: float = 1.0

    def validate(self) -> None:  # model.hpp:37-47
        p = Problem.make(self, Integrator.gl, QoISpec(), 0.5, 0.0, 1.0, 1, 0, validate=False)
        _check(lib().ablmc_problem_validate(_P(p._c)))

    def c(self) -> capi.ModelParamsC:
        return capi.ModelParamsC(self.kappa_sigma, self.kappa_tau, self.u_star, self.H,
                                 self.eps_reg, self.x_ref, self.noise_scale)


def equidistant_edges(bins: int, H: float) -> list[float]:  # qoi.hpp:144-151
    if bins < 1:
        raise ValueError("equidistant_edges: bins must be >= 1")
    e = [H * float(i) / float(bins) for i in range(bins + 1)]
    e[0], e[-1] = 0.0, H
    return e


@dataclass
class QoISpec:  # qoi.hpp:107-113
    kind: QoIKind = QoIKind.mean_position
    a: float = 0.1055
    b: float = 0.1555
    r: int = 4
    delta: float = 0.1
    bin_edges: Sequence[float] = field(default_factory=list)

    def size(self) -> int:
        return len(self.bin_edges) - 1 if self.kind == QoIKind.binned_field else 1


@dataclass
class SampleOptions:  # coupling.hpp:216-221
    signs_on: bool = True
    adaptive: bool = False
    x_adapt: float = 0.05


class Problem:
    """Problem (estimators.hpp:26-94) as a C descriptor; build with make()."""

    def __init__(self) -> None:
        self._c = capi.ProblemC()
        lib().ablmc_problem_defaults(_P(self._c))
        self._edges = None
        self.qoi = QoISpec()

    @staticmethod
    def make(params: ModelParams, ig: Integrator, qoi: QoISpec, x0: float, u0: float, T: float,
             m0: int, seed: int, opt: SampleOptions | None = None, *,
             profile: Profile = Profile.reference, random_u0: bool = False,
             const_sigma_u: float = 1.3, const_tau: float = 0.1, sigma_floor: float = 1e-3,
             tau_min: float = 1e-5, tau_max: float = 1.0, fp32: bool = False,
             validate: bool = True) -> "Problem":
        opt = opt or SampleOptions()
        pr = Problem()
        c = pr._c
        c.params = params.c()
        c.integrator = int(ig)
        c.signs_on = 1 if opt.signs_on else 0
        c.adaptive = 1 if opt.adaptive else 0
        c.x_adapt = opt.x_adapt
        c.qoi.kind = int(qoi.kind)
        c.qoi.a, c.qoi.b, c.qoi.r, c.qoi.delta = qoi.a, qoi.b, int(qoi.r), qoi.delta
        if qoi.kind == QoIKind.binned_field:
            pr._edges = (C.c_double * len(qoi.bin_edges))(*qoi.bin_edges)
            c.qoi.n_edges = len(qoi.bin_edges)
            c.qoi.bin_edges = C.cast(pr._edges, C.POINTER(C.c_double))
        c.x0, c.u0, c.T, c.m0, c.seed = x0, u0, T, int(m0), int(seed) & ((1 << 64) - 1)
        c.profile = int(profile)
        c.random_u0 = 1 if random_u0 else 0
        c.fp32 = 1 if fp32 else 0  # fp32-state variant (BASELINE config 5), statistical parity only
        c.const_sigma_u, c.const_tau = const_sigma_u, const_tau
        c.sigma_floor, c.tau_min, c.tau_max = sigma_floor, tau_min, tau_max
        pr.qoi = qoi
        if validate:
            _check(lib().ablmc_problem_validate(_P(c)))
        return pr

    # accessors mirroring the reference's public fields
    @property
    def integrator(self) -> Integrator:
        return Integrator(self._c.integrator)

    @property
    def m0(self) -> int:
        return self._c.m0

    @property
    def T(self) -> float:
        return self._c.T

    @property
    def seed(self) -> int:
        return self._c.seed

    def with_seed(self, seed: int) -> "Problem":
        q = Problem()
        C.memmove(C.addressof(q._c), C.addressof(self._c), C.sizeof(capi.ProblemC))
        q._edges, q.qoi = self._edges, self.qoi
        q._c.seed = int(seed)
        return q

    def dim(self) -> int:
        return int(lib().ablmc_qoi_dim(_P(self._c)))

    def h_level(self, level: int) -> float:  # estimators.hpp:39
        return self._c.T / float(self._c.m0 << level)

    def check_se_stability(self, h: float) -> None:  # estimators.hpp:86-93
        _check(lib().ablmc_check_se_stability(_P(self._c), h))


class LevelStats:
    """LevelStats (stats.hpp:26-88) with numpy sums."""

    def __init__(self) -> None:
        self.init(0, 0.0, 1)

    def init(self, level: int, h: float, dim: int) -> "LevelStats":
        self.level, self.h, self.dim = int(level), float(h), int(dim)
        self.sum_y = np.zeros(self.dim)
        self.sum_y2 = np.zeros(self.dim)
        self.n = self.failed = self.cost_steps = 0
        return self

    def attempts(self) -> int:
        return self.n + self.failed

    def add(self, y: Sequence[float], steps: int) -> None:  # stats.hpp:46-53
        for i in range(self.dim):
            self.sum_y[i] += y[i]
            self.sum_y2[i] += y[i] * y[i]
        self.n += 1
        self.cost_steps += steps

    def merge(self, o: "LevelStats") -> None:  # stats.hpp:55-63
        self.sum_y += o.sum_y
        self.sum_y2 += o.sum_y2
        self.n += o.n
        self.failed += o.failed
        self.cost_steps += o.cost_steps

    def mean(self, i: int = 0) -> float:
        return float(self.sum_y[i]) / float(self.n)

    def variance(self, i: int = 0) -> float:  # stats.hpp:67-71
        if self.n < 2:
            return 0.0
        m = float(self.sum_y[i]) / float(self.n)
        return max(0.0, (float(self.sum_y2[i]) - float(self.n) * m * m) / float(self.n - 1))

    def max_variance(self) -> float:
        return max([0.0] + [self.variance(i) for i in range(self.dim)])

    def max_abs_mean(self) -> float:
        return max([0.0] + [abs(self.mean(i)) for i in range(self.dim)])

    def std_error(self, i: int = 0) -> float:
        return (self.variance(i) / float(self.n)) ** 0.5 if self.n > 0 else 0.0

    # C view sharing the numpy buffers (add-merge happens in place)
    def _view(self) -> capi.LevelStatsC:
        v = capi.LevelStatsC()
        v.level, v.h, v.dim = self.level, self.h, self.dim
        v.sum_y = self.sum_y.ctypes.data_as(C.POINTER(C.c_double))
        v.sum_y2 = self.sum_y2.ctypes.data_as(C.POINTER(C.c_double))
        v.n, v.failed, v.cost_steps = self.n, self.failed, self.cost_steps
        return v

    def _take(self, v: capi.LevelStatsC) -> None:
        self.n, self.failed, self.cost_steps = v.n, v.failed, v.cost_steps


def accumulate_samples(acc: LevelStats, first: int, count: int, pr: Problem, level: int) -> None:
    """Device replacement for ``accumulate_samples(acc, first, count, workers,
    pr.level_sampler(level))`` (stats.hpp:96-136, estimators.hpp:60-72)."""
    if acc.dim != pr.dim():
        raise ValueError("LevelStats dim does not match the QoI size")
    v = acc._view()
    _check(lib().ablmc_accumulate_samples(_P(pr._c), int(level), int(first), int(count), _P(v)))
    acc._take(v)


def accumulate_levels(requests: Sequence[tuple], pr: Problem) -> None:
    """Several accumulate_samples calls in one device batch: requests are
    (acc, first, count, level) tuples; each acc ends as after its own call."""
    n = len(requests)
    views = [r[0]._view() for r in requests]
    lv = (C.c_int * n)(*[int(r[3]) for r in requests])
    fs = (C.c_int64 * n)(*[int(r[1]) for r in requests])
    cs = (C.c_int64 * n)(*[int(r[2]) for r in requests])
    ptrs = (C.POINTER(capi.LevelStatsC) * n)(*[_P(v) for v in views])
    _check(lib().ablmc_accumulate_levels(_P(pr._c), n, lv, fs, cs, ptrs))
    for r, v in zip(requests, views):
        r[0]._take(v)


def accumulate_paths(acc: LevelStats, first: int, count: int, pr: Problem, M: int,
                     stream_level: int = 0) -> None:
    """Device replacement for ``accumulate_samples(..., pr.path_sampler(M, stream_level))``."""
    v = acc._view()
    _check(lib().ablmc_accumulate_paths(_P(pr._c), int(M), int(stream_level), int(first),
                                        int(count), _P(v)))
    acc._take(v)


def check_failure_budget(acc: LevelStats) -> None:  # stats.hpp:139-143
    v = acc._view()
    _check(lib().ablmc_check_failure_budget(_P(v)))


# --------------------------------------------------------------- sharding
def num_superblocks(count: int) -> int:
    return int(lib().ablmc_num_superblocks(int(count)))


def accumulate_partials(pr: Problem, level: int, first: int, count: int, sb_begin: int,
                        sb_end: int, M: int = 0, stream_level: int = 0):
    """Super-block partials [sb_begin, sb_end) -> (sums[n,2*dim], counts[n,2])."""
    n = sb_end - sb_begin
    dim = pr.dim()
    sums = np.zeros((max(n, 0), 2 * dim))
    counts = np.zeros((max(n, 0), capi.ABLMC_NCOUNTS), dtype=np.int64)  # n, failed, cost_steps
    _check(lib().ablmc_accumulate_partials(
        _P(pr._c), int(level), int(M), int(stream_level), int(first), int(count), int(sb_begin),
        int(sb_end), sums.ctypes.data_as(C.POINTER(C.c_double)),
        counts.ctypes.data_as(C.POINTER(C.c_int64))))
    return sums, counts


def merge_partials(acc: LevelStats, pr: Problem, level: int, sums: np.ndarray, counts: np.ndarray,
                   M: int = 0) -> None:
    sums = np.ascontiguousarray(sums, dtype=np.float64)
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    v = acc._view()
    _check(lib().ablmc_merge_partials(_P(pr._c), int(level), int(M), int(sums.shape[0]),
                                      sums.ctypes.data_as(C.POINTER(C.c_double)),
                                      counts.ctypes.data_as(C.POINTER(C.c_int64)), _P(v)))
    acc._take(v)


def gather_layout(dim: int, world: int, n_sb: Sequence[int]) -> tuple[int, int, list[int]]:
    """(rows per rank, row width in doubles, first row of each request) of
    the all-gather block of a batch of requests of n_sb[q] super-blocks
    (include/ablmc_b200.h)."""
    n = len(n_sb)
    cs = (C.c_int64 * max(n, 1))(*[int(c) for c in n_sb])
    rows, width = C.c_int64(), C.c_int64()
    base = (C.c_int64 * max(n, 1))()
    _check(lib().ablmc_gather_layout(int(dim), int(world), n, cs, C.byref(rows), C.byref(width),
                                     base))
    return rows.value, width.value, list(base)[:n]


def merge_gathered(accs: Sequence[LevelStats], n_sb: Sequence[int], world: int,
                   recv: np.ndarray) -> None:
    """Merge all ranks' gathered blocks (recv, rank-major) into accs in
    global super-block order -- the library's post-all-gather step."""
    n = len(accs)
    dim = accs[0].dim
    recv = np.ascontiguousarray(recv, dtype=np.float64)
    views = [a._view() for a in accs]
    cs = (C.c_int64 * n)(*[int(c) for c in n_sb])
    ptrs = (C.POINTER(capi.LevelStatsC) * n)(*[_P(v) for v in views])
    _check(lib().ablmc_merge_gathered(int(dim), int(world), n, cs,
                                      recv.ctypes.data_as(C.POINTER(C.c_double)), ptrs))
    for a, v in zip(accs, views):
        a._take(v)


# ------------------------------------------------------------- oracle mode
PAIR_DTYPE = np.dtype([("fx", "f8"), ("fu", "f8"), ("fpar", "i4"), ("fok", "i4"), ("fn", "i8"),
                       ("cx", "f8"), ("cu", "f8"), ("cpar", "i4"), ("cok", "i4"), ("cn", "i8")])
PATH_DTYPE = np.dtype([("x", "f8"), ("u", "f8"), ("parity", "i4"), ("ok", "i4"), ("n_refl", "i8")])


def simulate_pairs(pr: Problem, level: int, first: int, count: int,
                   xi: Optional[np.ndarray] = None) -> np.ndarray:
    """simulate_pair (coupling.hpp:64-105) for samples [first, first+count).
    xi[count, M_f]: host-supplied normals (oracle mode), else Philox."""
    out = np.zeros(count, dtype=PAIR_DTYPE)
    xp = None
    if xi is not None:
        xi = np.ascontiguousarray(xi, dtype=np.float64)
        if xi.shape != (count, pr.m0 << level):
            raise ValueError("xi must have shape (count, m0 << level)")
        xp = xi.ctypes.data_as(C.POINTER(C.c_double))
    _check(lib().ablmc_pair_states(_P(pr._c), int(level), int(first), int(count), xp,
                                   out.ctypes.data_as(C.POINTER(capi.PairStateC))))
    return out


def simulate_paths(pr: Problem, M: int, first: int, count: int, stream_level: int = 0,
                   xi: Optional[np.ndarray] = None) -> np.ndarray:
    out = np.zeros(count, dtype=PATH_DTYPE)
    xp = None
    if xi is not None:
        xi = np.ascontiguousarray(xi, dtype=np.float64)
        if xi.shape != (count, M):
            raise ValueError("xi must have shape (count, M)")
        xp = xi.ctypes.data_as(C.POINTER(C.c_double))
    _check(lib().ablmc_path_states(_P(pr._c), int(M), int(stream_level), int(first), int(count),
                                   xp, out.ctypes.data_as(C.POINTER(capi.PathStateC))))
    return out


def normals(seed: int, level: int, idx: int, k0: int, n: int) -> np.ndarray:
    """NoiseStream(seed, level, idx).normal_at(k0 + j) on the device (noise.hpp:57-75)."""
    out = np.zeros(n)
    _check(lib().ablmc_normals(int(seed), int(level), int(idx), int(k0), int(n),
                               out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


# ----------------------------------------------------------------- drivers
@dataclass
class MlmcOptions:  # estimators.hpp:271-278
    pilot_n: int = 10000
    pilot_levels_max: int = 4
    init_n: int = 1000
    l_max: int = 16
    bias_fit: Optional[tuple[float, float]] = None  # (alpha, c1)


WARNINGS = ("Var[Y_1] >= Var[Y_0]/2: coarsest level M_0 is too coarse to pay off",
            "sample allocation did not converge in 64 rounds")  # estimators.hpp:352-373


@dataclass
class RunResult:  # estimators.hpp:197-210
    estimate: list
    stat_error: list
    bias_estimate: float
    alpha: float
    c1: float
    levels_used: int
    level_stats: list
    total_cost_steps: int
    pilot_cost_steps: int
    failed_samples: int
    wall_seconds: float
    warnings: list
    c: capi.RunResultC = field(repr=False, default=None)  # C view (for the format writers)
    _keep: tuple = field(repr=False, default=())


def _new_result(dim: int):
    r = capi.RunResultC()
    est, err = np.zeros(dim), np.zeros(dim)
    sy = np.zeros((capi.ABLMC_MAX_LEVELS, dim))
    sy2 = np.zeros((capi.ABLMC_MAX_LEVELS, dim))
    r.est_vec = est.ctypes.data_as(C.POINTER(C.c_double))
    r.err_vec = err.ctypes.data_as(C.POINTER(C.c_double))
    r.level_sum_y_vec = sy.ctypes.data_as(C.POINTER(C.c_double))
    r.level_sum_y2_vec = sy2.ctypes.data_as(C.POINTER(C.c_double))
    return r, (est, err, sy, sy2)


def _result(r: capi.RunResultC, keep) -> RunResult:
    est, err, sy, sy2 = keep
    dim = est.shape[0]
    levels = []
    for l in range(r.n_levels):
        st = LevelStats().init(l, r.level_h[l], dim)
        st.sum_y[:], st.sum_y2[:] = sy[l], sy2[l]
        st.n, st.failed, st.cost_steps = r.level_n[l], r.level_failed[l], r.level_cost[l]
        levels.append(st)
    warnings = [w for i, w in enumerate(WARNINGS) if r.warnings_mask >> i & 1]
    return RunResult(list(est), list(err), r.bias_estimate, r.alpha, r.c1, r.levels_used, levels,
                     r.total_cost_steps, r.pilot_cost_steps, r.failed_samples, r.wall_seconds,
                     warnings, r, keep)


def run_mlmc(pr: Problem, eps: float, o: MlmcOptions | None = None) -> RunResult:
    o = o or MlmcOptions()
    oc = capi.MlmcOptionsC()
    lib().ablmc_mlmc_options_defaults(_P(oc))
    oc.pilot_n, oc.pilot_levels_max, oc.init_n, oc.l_max = o.pilot_n, o.pilot_levels_max, o.init_n, o.l_max
    if o.bias_fit is not None:
        oc.use_bias_fit, (oc.alpha, oc.c1) = 1, o.bias_fit
    r, keep = _new_result(pr.dim())
    _check(lib().ablmc_run_mlmc(_P(pr._c), float(eps), _P(oc), _P(r)))
    return _result(r, keep)


def run_stmc(pr: Problem, M_L: int, eps: float, fixed_n: int = 0) -> RunResult:
    r, keep = _new_result(pr.dim())
    _check(lib().ablmc_run_stmc(_P(pr._c), int(M_L), float(eps), int(fixed_n), _P(r)))
    return _result(r, keep)


@dataclass
class DecayRow:  # estimators.hpp:403-411
    level: int
    h: float
    var_y: float
    mean_y: float
    se_mean: float
    n: int
    cost_steps: int


def decay_sweep(pr: Problem, l_min: int, l_max: int, n_per_level: int) -> list[DecayRow]:
    rows = (capi.DecayRowC * (l_max - l_min + 1))()
    _check(lib().ablmc_decay_sweep(_P(pr._c), int(l_min), int(l_max), int(n_per_level), rows))
    return [DecayRow(r.level, r.h, r.var_y, r.mean_y, r.se_mean, r.n, r.cost_steps) for r in rows]


def _dbl(v: Sequence[float]):
    return (C.c_double * len(v))(*[float(x) for x in v])


def fit_power_law(h: Sequence[float], v: Sequence[float]) -> tuple[float, float]:
    """estimators.hpp:107-123 -> (exponent, log_prefactor) (host, in the library)."""
    if len(h) != len(v):
        raise ValueError("fit_power_law: need at least two points")
    e, lp = C.c_double(), C.c_double()
    _check(lib().ablmc_fit_power_law(_dbl(h), _dbl(v), len(h), C.byref(e), C.byref(lp)))
    return e.value, lp.value


@dataclass
class BiasFit:  # estimators.hpp:131-137
    alpha: float = 1.0
    c1: float = 0.0
    c_y: float = 0.0

    def bias_at(self, h: float) -> float:
        return self.c1 * h ** self.alpha


def estimate_bias_constants(h: Sequence[float], mean_abs: Sequence[float],
                            std_err: Sequence[float]) -> BiasFit:
    """estimators.hpp:142-161; RuntimeError when some |E[Y_l]| <= 3 SE."""
    if not (len(h) == len(mean_abs) == len(std_err)):
        raise ValueError("estimate_bias_constants: ragged input")
    a, c1, cy = C.c_double(), C.c_double(), C.c_double()
    _check(lib().ablmc_estimate_bias_constants(_dbl(h), _dbl(mean_abs), _dbl(std_err), len(h),
                                               C.byref(a), C.byref(c1), C.byref(cy)))
    return BiasFit(a.value, c1.value, cy.value)


def choose_levels(alpha: float, c1: float, eps: float, m0: int, T: float, l_max: int = 16) -> int:
    """estimators.hpp:163-175."""
    L = C.c_int()
    _check(lib().ablmc_choose_levels(float(alpha), float(c1), float(eps), int(m0), float(T),
                                     int(l_max), C.byref(L)))
    return L.value


def allocate_samples(var: Sequence[float], h: Sequence[float], eps: float) -> list[int]:
    """estimators.hpp:177-190."""
    if len(var) != len(h):
        raise ValueError("allocate_samples: ragged input")
    out = (C.c_int64 * len(h))()
    _check(lib().ablmc_allocate_samples(_dbl(var), _dbl(h), len(h), float(eps), out))
    return list(out)


def build_smoothing_polynomial(r: int) -> list[float]:
    """qoi.hpp:31-77: coefficients of g_r (r + 2 of them)."""
    out = (C.c_double * 16)()
    _check(lib().ablmc_build_smoothing_polynomial(int(r), out))
    return list(out)[: int(r) + 2]


def adaptive_step_size(x: float, h: float, x_adapt: float, params: ModelParams) -> float:
    """timeline.hpp:18-23."""
    p = params.c()
    return lib().ablmc_adaptive_step_size(float(x), float(h), float(x_adapt), _P(p))


def variance_decay_slope(rows: Sequence[DecayRow]) -> float:  # estimators.hpp:434-441
    return fit_power_law([r.h for r in rows], [r.var_y for r in rows])[0]


# ------------------------------------------------------ cost sweep / formats
class Method(enum.IntEnum):  # estimators.hpp:163
    stmc = 0
    mlmc = 1


@dataclass
class CostRow:  # estimators.hpp:443-451
    eps: float
    method: Method
    integrator: Integrator
    cost_steps: int
    wall_seconds: float
    estimate: float
    stat_error: float


def cost_sweep(pr: Problem, method: Method, eps_values: Sequence[float],
               fit: tuple[float, float]) -> list[CostRow]:
    """estimators.hpp:456-485 over the device sampler; fit = (alpha, c1)."""
    eps = (C.c_double * len(eps_values))(*eps_values)
    rows = (capi.CostRowC * len(eps_values))()
    _check(lib().ablmc_cost_sweep(_P(pr._c), int(method), eps, len(eps_values), float(fit[0]),
                                  float(fit[1]), rows))
    return [CostRow(r.eps, Method(r.method), Integrator(r.integrator), r.cost_steps,
                    r.wall_seconds, r.estimate, r.stat_error) for r in rows]


@dataclass
class RunConfig:  # config.hpp:18-40 (the fields result.json records)
    model: ModelParams = field(default_factory=ModelParams)
    method: Method = Method.mlmc
    integrator: Integrator = Integrator.gl
    qoi_kind: QoIKind = QoIKind.mean_position
    qoi_a: float = 0.1055
    qoi_b: float = 0.1555
    qoi_r: int = 4
    qoi_delta: float = 0.1
    qoi_bins: int = 20
    T: float = 1.0
    m0: int = 40
    eps: float = 1e-3
    fixed_n: int = 0
    seed: int = 12345
    x0: float = 0.05
    u0: float = 0.1
    adaptive: bool = False
    x_adapt: float = 0.05
    coupling_signs: bool = True
    workers: int = 1
    timings: bool = True
    output_dir: str = "."

    def c(self) -> capi.RunConfigC:
        k = capi.RunConfigC()
        k.model = self.model.c()
        k.method, k.integrator, k.qoi_kind, k.qoi_r = (int(self.method), int(self.integrator),
                                                       int(self.qoi_kind), int(self.qoi_r))
        k.qoi_a, k.qoi_b, k.qoi_delta, k.qoi_bins = self.qoi_a, self.qoi_b, self.qoi_delta, int(self.qoi_bins)
        k.adaptive, k.T, k.m0, k.eps = int(self.adaptive), self.T, int(self.m0), self.eps
        k.fixed_n, k.seed, k.x0, k.u0, k.x_adapt = (int(self.fixed_n), int(self.seed), self.x0,
                                                    self.u0, self.x_adapt)
        k.coupling_signs, k.workers, k.timings = (int(self.coupling_signs), int(self.workers),
                                                  int(self.timings))
        k.output_dir = self.output_dir.encode()
        return k


def _text(fn, *args) -> str:
    n = fn(*args, None, 0)
    if n < 0:
        raise ValueError("format writer failed")
    buf = C.create_string_buffer(int(n) + 1)
    fn(*args, buf, n + 1)
    return buf.raw[:n].decode()


def result_json(cfg: RunConfig, r: RunResult) -> str:
    """result.json text (output.hpp:91-123,213-219), byte-identical to the reference."""
    cc = cfg.c()
    return _text(lib().ablmc_result_json, _P(cc), _P(r.c), len(r.estimate))


def read_result_json(text: str) -> tuple:
    """output_record_from_json (output.hpp:47-81,125-159): (RunConfig, RunResult)
    from result.json text -- reload the per-level sums to resume a run."""
    d = C.c_int64()
    raw = text.encode()
    rc = lib().ablmc_read_result_json(raw, None, None, C.byref(d), None, 0)
    if rc != 0:
        msg = lib().ablmc_read_result_json_error().decode()
        raise RuntimeError(msg) if rc == capi.ABLMC_ERR_RUNTIME else ValueError(msg)
    r, keep = _new_result(int(d.value))
    k = capi.RunConfigC()
    buf = C.create_string_buffer(4096)
    _check(lib().ablmc_read_result_json(raw, _P(k), _P(r), C.byref(d), buf, 4096))
    m = k.model
    cfg = RunConfig(ModelParams(m.kappa_sigma, m.kappa_tau, m.u_star, m.H, m.eps_reg, m.x_ref,
                                m.noise_scale), Method(k.method), Integrator(k.integrator),
                    QoIKind(k.qoi_kind), k.qoi_a, k.qoi_b, k.qoi_r, k.qoi_delta, k.qoi_bins, k.T,
                    k.m0, k.eps, k.fixed_n, k.seed, k.x0, k.u0, bool(k.adaptive), k.x_adapt,
                    bool(k.coupling_signs), k.workers, bool(k.timings), buf.value.decode())
    return cfg, _result(r, keep)


def write_result_json(cfg: RunConfig, r: RunResult, directory) -> str:
    from pathlib import Path
    d = Path(directory)
    d.mkdir(parents=True, exist_ok=True)
    path = d / "result.json"
    path.write_bytes(result_json(cfg, r).encode())
    return str(path)


def variance_decay_csv(rows: Sequence[DecayRow]) -> str:  # output.hpp:184-191
    arr = (capi.DecayRowC * len(rows))()
    for a, r in zip(arr, rows):
        a.level, a.h, a.var_y, a.mean_y, a.se_mean, a.n, a.cost_steps = (
            r.level, r.h, r.var_y, r.mean_y, r.se_mean, r.n, r.cost_steps)
    return _text(lib().ablmc_variance_decay_csv, arr, len(rows))


def cost_sweep_csv(rows: Sequence[CostRow], timings: bool = True) -> str:  # output.hpp:193-200
    arr = (capi.CostRowC * len(rows))()
    for a, r in zip(arr, rows):
        a.eps, a.method, a.integrator, a.cost_steps = r.eps, int(r.method), int(r.integrator), r.cost_steps
        a.wall_seconds, a.estimate, a.stat_error = r.wall_seconds, r.estimate, r.stat_error
    return _text(lib().ablmc_cost_sweep_csv, arr, len(rows), int(timings))


def pdf_csv(edges: Sequence[float], concentration: Sequence[float],
            std_error: Sequence[float]) -> str:  # output.hpp:202-209
    e = (C.c_double * len(edges))(*edges)
    cc = (C.c_double * len(concentration))(*concentration)
    se = (C.c_double * len(std_error))(*std_error)
    return _text(lib().ablmc_pdf_csv, e, len(edges), cc, se)
