#!/usr/bin/env python
"""Benchmark of the B200 coupled MLMC level sampler (BASELINE.json metric:
coupled fine path-steps/s per level, % of the FP64 roofline).

Workload (BASELINE.json configs[4], "C5"): reference profile (kappa_sigma
1.3, kappa_tau 0.5, u* 0.2, H 1, eps_reg 0.01), z0 = 500 m (x0 = 0.5),
u0 = 0.1, T = 1000 s (T = 1), M0 = 1, level l = 10 (1024 fine + 512 coarse
steps), symplectic Euler, fp64, mean-position QoI, Philox seed 42, N coupled
paths per GPU (default 2^25).  One step = one accumulate_samples call over
the N paths (level sampler + moment reduction).  Weak scaling: rank r owns
sample indices [r N, (r+1) N) (contiguous super-blocks), and for N > 1 the
per-rank moments meet in one NCCL all-gather per step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--paths N] [--impl reference]
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# Algorithmic FP64-pipe ops per coupled fine path-step.
W_ALG = {0: 181.0, 1: 273.0, 2: 416.0}
IG_NAME = {0: "se", 1: "gl", 2: "baoab"}
LEVEL = 10
SEED = 42


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--paths", type=int, default=1 << 25, help="coupled paths per GPU per step")
    ap.add_argument("--integrator", default="se", choices=["se", "gl", "baoab"])
    ap.add_argument("--level", type=int, default=LEVEL)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target wall time of the CPU baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-step-seconds", type=float, default=None,
                    help="reference arm: CPU seconds per step (default: ~60 s over the run)")
    ap.add_argument("--force-dist", action="store_true",
                    help="use the NCCL process group and collectives even at world size 1")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the per-integrator lines and the MLMC time-to-eps sweep")
    ap.add_argument("--mlmc-eps", default="1e-4,3e-5,1e-5,3e-6",
                    help="config-3 tolerances (nondimensional: eps[m] / 1000 m)")
    return ap.parse_args()


def problem_c(ig: int):
    from paper_1612_07717_b200 import ablmc
    return ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator(ig), ablmc.QoISpec(), 0.5, 0.1,
                              1.0, 1, SEED)


class _RefProblem:
    """The C5 problem descriptor for the reference arm, filled field by field
    (the reference's defaults: model.hpp:29-35, qoi.hpp:108-112,
    estimators.hpp:27-36, coupling.hpp:218-220) WITHOUT the product library:
    the reference arm must not map libablmc_b200.so."""

    def __init__(self, ig: int):
        from paper_1612_07717_b200 import capi  # ctypes structs only; loads nothing
        c = capi.ProblemC()
        c.params = capi.ModelParamsC(1.3, 0.5, 0.2, 1.0, 0.01, 1.0, 1.0)
        c.integrator, c.signs_on = ig, 1
        c.qoi.kind, c.qoi.r, c.qoi.a, c.qoi.b, c.qoi.delta = 0, 4, 0.1055, 0.1555, 0.1
        c.x0, c.u0, c.T, c.m0, c.seed = 0.5, 0.1, 1.0, 1, SEED
        c.adaptive, c.x_adapt, c.profile = 0, 0.05, 0
        self._c = c


def workload_config(a, world: int) -> dict:
    """`config` of BOTH arms (identical, so the driver can compare them): the
    C5 workload.  The CPU arm times a bounded sample of it (reported outside
    `config`); throughput per path-step does not depend on the path count."""
    Mf = 1 << a.level
    return {"workload": f"C5: level {a.level} coupled pair ({Mf} fine + {Mf // 2} coarse steps), "
                        f"{a.integrator}, reference profile, x0=0.5, u0=0.1, T=1, M0=1, "
                        f"mean-position QoI, Philox seed {SEED}",
            "paths_per_gpu": a.paths, "level": a.level, "integrator": a.integrator,
            "l2": "GPU arm: flushed between timed steps (256 MB write); path state is "
                  "register-resident",
            "parallelism": f"dp{world} (contiguous super-block shards, one native NCCL "
                           f"all-gather of the partials per step)"}


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ------------------------------------------------------------ CPU reference
def reference_sample(ig: int, level: int, target_s: float, threads: int, pr=None):
    """Time the reference's own accumulate_samples (oracle/_ref, unmodified
    headers, std::thread pool) on a bounded sample; returns (path-steps/s,
    samples, seconds)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O
    R = O.ref()
    if R is None:
        raise RuntimeError("oracle/_ref/libablmc_ref.so is missing (built by __graft_entry__.build)")
    pr = pr or problem_c(ig)
    Mf = 1 << level
    n = max(threads * 64, 4096)
    secs = C.c_double()
    while True:
        st = O.Stats(1)
        rc = R.ref_accumulate_samples(C.byref(pr._c), level, 0, n, threads, C.byref(st.c),
                                      C.byref(secs))
        if rc != 0:
            raise RuntimeError(R.ref_last_error().decode())
        if secs.value >= 0.5 * target_s or n > (1 << 30):
            break
        n = int(n * min(64.0, max(2.0, target_s / max(secs.value, 1e-3))))
    return n * Mf / secs.value, n, secs.value


def run_reference(a):
    """The reference arm: the unmodified reference's own accumulate_samples
    (oracle/_ref, std::thread pool on every host thread) on the C5 workload,
    each step a bounded sample of it.  Under torchrun only rank 0 runs.  The
    product library is never loaded here."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # rank 0 alone runs the CPU reference arm
    ig = {"se": 0, "gl": 1, "baoab": 2}[a.integrator]
    threads = host_threads()
    pr = _RefProblem(ig)
    step_s = a.ref_step_seconds or max(1.0, 60.0 / max(1, a.steps + a.warmup))  # run ~1-2 min
    rate, n, _ = reference_sample(ig, a.level, step_s, threads, pr)
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O
    R = O.ref()
    secs = C.c_double()
    times = []
    for i in range(a.warmup + a.steps):
        st = O.Stats(1)
        R.ref_accumulate_samples(C.byref(pr._c), a.level, i * n, n, threads, C.byref(st.c),
                                 C.byref(secs))
        if i >= a.warmup:
            times.append(secs.value)
    Mf = 1 << a.level
    t = statistics.mean(times)
    value = n * Mf / t
    sample = (f"{n} coupled paths x {Mf} fine steps per step (bounded sample of the workload); "
              f"reference accumulate_samples with {threads} worker threads")
    line = {
        "impl": "reference", "metric": "coupled fine path-steps/s (level sampler)",
        "value": value, "unit": "path-steps/s", "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (Philox seed 42)",
        "config": workload_config(a, a.gpus),
        "cpu_sample": {"paths_per_step": n, "note": "throughput per path-step does not depend on "
                       "the number of paths (independent samples)"},
        "cpu_baseline": {"value": value, "unit": "path-steps/s", "cores": threads,
                         "kind": "reference", "sample": sample},
        "e2e": {"value": value, "unit": "path-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, device: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------- extra measurements
def _k1_profile() -> dict:
    tp = ROOT / "profiles" / "k1_ncu.json"
    return json.loads(tp.read_text()) if tp.exists() else {}


def per_integrator(a, lib, stream, peak, clock_hz=None):
    """Level-10 coupled throughput of all three integrators (2^23 paths, one
    warm-up + 2 timed accumulate calls each, CUDA events on the stream)."""
    import torch
    out = {}
    n = 1 << 23
    for ig in (0, 1, 2):
        pr = problem_c(ig)
        pc = C.byref(pr._c)
        lib.ablmc_accumulate_device(pc, a.level, 0, n)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record(stream)
        for _ in range(2):
            lib.ablmc_accumulate_device(pc, a.level, 0, n)
        e.record(stream)
        torch.cuda.synchronize()
        rate = 2 * n * (1 << a.level) / (s.elapsed_time(e) * 1e-3)
        w_exec = _k1_profile().get(IG_NAME[ig], {}).get("fp64_instr_per_path_step")
        out[IG_NAME[ig]] = {"path_steps_per_s": rate, "W_executed_ncu": w_exec,
                            "roofline_frac": rate * w_exec / peak if w_exec else None,
                            "W_alg": W_ALG[ig], "roofline_frac_W_alg": rate * W_ALG[ig] / peak,
                            "paths": n}
    # fp32-state variant (BASELINE config 5; statistical parity only)
    from paper_1612_07717_b200 import ablmc
    for ig in (0, 1, 2):
        pr = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator(ig), ablmc.QoISpec(), 0.5,
                                0.1, 1.0, 1, SEED, fp32=True)
        pc = C.byref(pr._c)
        lib.ablmc_accumulate_device(pc, a.level, 0, n)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record(stream)
        for _ in range(2):
            lib.ablmc_accumulate_device(pc, a.level, 0, n)
        e.record(stream)
        torch.cuda.synchronize()
        rate = 2 * n * (1 << a.level) / (s.elapsed_time(e) * 1e-3)
        row = {"path_steps_per_s": rate, "paths": n}
        # W32 roofline: FP32-pipe arithmetic instructions per
        # path-step (ncu, profiles/k1_ncu.json) against the 128-lane FFMA pipe
        # at the SM clock of this run; the variant is issue-bound, so the issue
        # fraction (all instructions / 4 SMSPs x 1 warp-instr per cycle) and
        # the MUFU (XU) count are reported beside it
        prof = _k1_profile().get(IG_NAME[ig] + "_fp32_state")
        if prof and clock_hz:
            w32, ins = prof["fp32_instr_per_path_step"], prof["instr_per_path_step"]
            row.update({"W32_fp32_pipe": w32, "mufu_per_path_step": prof["mufu_per_path_step"],
                        "instr_per_path_step": ins,
                        "roofline_frac_fp32_pipe": rate * w32 / (148 * 128 * clock_hz),
                        "issue_frac": rate * ins / 32 / (148 * 4 * clock_hz),
                        "ncu_pct": {k: prof[k] for k in ("issue_active_pct", "fma_pipe_pct",
                                                          "alu_pipe_pct", "xu_pipe_pct")},
                        "source": prof["source"]})
        out[IG_NAME[ig] + "_fp32_state"] = row
    out["adaptive"] = adaptive_rates(lib, stream)
    return out


def adaptive_rates(lib, stream):
    """adaptive (non-nested) level 3, defaults (x0 =
    0.05, u0 = 0.1, T = 1, M0 = 40, x_adapt = 0.05, smoothed indicator); steps
    actually taken per second on the B200 (2^20 samples) and by the reference's
    own accumulate_samples on all host threads (bounded sample)."""
    import numpy as np
    import torch
    from paper_1612_07717_b200 import ablmc, capi
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O
    R = O.ref()
    threads = host_threads()
    out = {}
    level = 3
    for ig in (0, 1, 2):
        q = ablmc.QoISpec(kind=ablmc.QoIKind.smoothed_indicator)
        pr = ablmc.Problem.make(ablmc.ModelParams(), ablmc.Integrator(ig), q, 0.05, 0.1, 1.0, 40,
                                SEED, ablmc.SampleOptions(adaptive=True, x_adapt=0.05))
        pc = C.byref(pr._c)
        n = 1 << 20
        lib.ablmc_accumulate_device(pc, level, 0, n)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record(stream)
        lib.ablmc_accumulate_device(pc, level, 0, n)
        e.record(stream)
        torch.cuda.synchronize()
        sy, sy2 = np.zeros(1), np.zeros(1)
        acc = capi.LevelStatsC()
        acc.level, acc.dim = level, 1
        acc.sum_y = sy.ctypes.data_as(C.POINTER(C.c_double))
        acc.sum_y2 = sy2.ctypes.data_as(C.POINTER(C.c_double))
        lib.ablmc_fetch_device_result(pc, level, C.byref(acc))
        gpu = acc.cost_steps / (s.elapsed_time(e) * 1e-3)
        row = {"steps_per_s": gpu, "samples": n, "mean_steps_per_sample": acc.cost_steps / n}
        if R is not None:
            st = O.Stats(1)
            secs = C.c_double()
            m = 4096 * threads
            R.ref_accumulate_samples(pc, level, 0, m, threads, C.byref(st.c), C.byref(secs))
            row["cpu_reference_steps_per_s"] = st.cost_steps / secs.value
            row["cpu_reference_threads"] = threads
            row["speedup_vs_cpu_reference"] = gpu / row["cpu_reference_steps_per_s"]
        out[IG_NAME[ig]] = row
    return out


def _timed_level(lib, stream, pr, level, n, reps=1):
    """(ms per accumulate call, samples, cost_steps) for one device level."""
    import numpy as np
    import torch
    from paper_1612_07717_b200 import capi
    pc = C.byref(pr._c)
    lib.ablmc_accumulate_device(pc, level, 0, n)  # warm-up (workspace growth)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record(stream)
    for _ in range(reps):
        lib.ablmc_accumulate_device(pc, level, 0, n)
    e.record(stream)
    torch.cuda.synchronize()
    dim = pr.dim()
    sy, sy2 = np.zeros(dim), np.zeros(dim)
    acc = capi.LevelStatsC()
    acc.level, acc.dim = level, dim
    acc.sum_y = sy.ctypes.data_as(C.POINTER(C.c_double))
    acc.sum_y2 = sy2.ctypes.data_as(C.POINTER(C.c_double))
    lib.ablmc_fetch_device_result(pc, level, C.byref(acc))
    return s.elapsed_time(e) / reps, acc.n, acc.cost_steps


def configs_sweep(lib, stream):
    """BASELINE.json configs 1, 2 and 4 on one B200 (nondimensional units:
    H = 1000 m, T = 1000 s, velocities in m/s; DESIGN.md §7 for the
    extension profiles).  Each level is one device accumulate call of N
    samples (config 4 bounded to 2^22 paths per level instead of 2e8, to keep
    the default run short; throughput is per path, so it extrapolates)."""
    import torch
    from paper_1612_07717_b200 import ablmc
    out = {}
    mp = ablmc.ModelParams()
    # config 1: homogeneous OU (constant sigma_w = 1.3, tau = 0.1), z0 = H/2,
    # w0 ~ N(0, sigma_w^2), SE, l = 3 with M_f = 8, N = 1e5, QoI z_T
    pr = ablmc.Problem.make(mp, ablmc.Integrator.se, ablmc.QoISpec(), 0.5, 0.0, 1.0, 1, SEED,
                            profile=ablmc.Profile.constant, random_u0=True)
    ms, n, cost = _timed_level(lib, stream, pr, 3, 100000, reps=20)
    out["config1_homogeneous_ou_se_l3"] = {"ms_per_level_call": ms, "paths": n,
                                           "path_steps_per_s": n * 8 / (ms * 1e-3)}
    # config 2: floored / clamped inhomogeneous profile, w0 ~ N(0, sigma_w(z0)^2),
    # z0 = H/2, levels 0..8, M0 = 1, N = 1e6 per level, all three integrators
    c2 = {}
    for ig in ablmc.Integrator:
        pr = ablmc.Problem.make(mp, ig, ablmc.QoISpec(), 0.5, 0.0, 1.0, 1, SEED,
                                profile=ablmc.Profile.floored, random_u0=True)
        rows = []
        total_ms = 0.0
        for level in range(9):
            ms, n, cost = _timed_level(lib, stream, pr, level, 1000000)
            total_ms += ms
            rows.append({"level": level, "ms": ms, "cost_steps": cost})
        # the same nine levels as ONE accumulate_levels batch through the public
        # API (what one MLMC allocation round is: the levels run on concurrent
        # lanes, one synchronisation, host LevelStats out): wall time, best of 3
        walls = []
        for _ in range(4):
            reqs = [(ablmc.LevelStats().init(l, pr.h_level(l), 1), 0, 1000000, l) for l in range(9)]
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ablmc.accumulate_levels(reqs, pr)
            walls.append((time.perf_counter() - t0) * 1e3)
        assert [r[0].cost_steps for r in reqs] == [r["cost_steps"] for r in rows]
        c2[ig.name] = {"levels": rows, "total_ms": total_ms,
                       "one_batch_wall_ms": min(walls[1:]),
                       "fine_path_steps_per_s_level8": 1e6 * 256 / (rows[-1]["ms"] * 1e-3)}
    out["config2_floored_levels0to8_1e6"] = c2
    # config 4: release at z0 = 10 m, 64-bin smoothed concentration field,
    # GL, levels 0..10, floored profile
    q = ablmc.QoISpec(kind=ablmc.QoIKind.binned_field, bin_edges=ablmc.equidistant_edges(64, 1.0))
    pr = ablmc.Problem.make(mp, ablmc.Integrator.gl, q, 0.01, 0.0, 1.0, 1, SEED,
                            profile=ablmc.Profile.floored, random_u0=True)
    n4 = 1 << 22
    rows = []
    for level in range(11):
        ms, n, cost = _timed_level(lib, stream, pr, level, n4)
        rows.append({"level": level, "ms": ms, "paths_per_s": n / (ms * 1e-3)})
    # config 5 throughput against N (the headline runs 2^25 per GPU)
    pr = ablmc.Problem.make(mp, ablmc.Integrator.se, ablmc.QoISpec(), 0.5, 0.1, 1.0, 1, SEED)
    out["config5_se_l10_n_sweep"] = {}
    for n in (10**6, 10**7, 10**8):
        ms, ok, cost = _timed_level(lib, stream, pr, 10, n)
        out["config5_se_l10_n_sweep"][f"{n:.0e}"] = {"ms": ms, "path_steps_per_s": ok * 1024 / (ms * 1e-3)}
    out["config4_z0_10m_64bins_gl"] = {
        "paths_per_level": n4, "levels": rows,
        "projected_seconds_2e8_paths_x_11_levels": sum(2e8 / r["paths_per_s"] for r in rows)}
    return out


def mlmc_sweep(a):
    """BASELINE config 3: full MLMC driver (reference run_mlmc semantics,
    estimators.hpp:284-397) on the reference profile, BAOAB, x0 = 0.5,
    u0 = 0.1, T = 1, M0 = 1, mean position, for each tolerance; wall time of
    the whole driver (host allocation loop + device level sampler)."""
    from paper_1612_07717_b200 import ablmc, capi
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_lib as O
    R = O.ref()
    threads = host_threads()
    res = {}
    pr = problem_c(2)
    for eps in [float(e) for e in a.mlmc_eps.split(",") if e]:
        times = []
        for _ in range(3):  # best of 3 (host-side wall clock of the whole driver)
            t0 = time.perf_counter()
            r = ablmc.run_mlmc(pr, eps)
            times.append(time.perf_counter() - t0)
        t = min(times)
        row = {"seconds": t, "seconds_all": times, "estimate": r.estimate[0], "stat_error": r.stat_error[0],
               "bias_estimate": r.bias_estimate, "levels": r.levels_used,
               "N_l": [st.n for st in r.level_stats], "total_cost_steps": r.total_cost_steps,
               "eps_m": eps * 1000.0}
        # StMC at the finest resolved level M0 2^L (estimators.hpp:230-269)
        t0 = time.perf_counter()
        s = ablmc.run_stmc(pr, 1 << r.levels_used, eps)
        row["stmc_seconds"] = time.perf_counter() - t0
        row["stmc_cost_steps"] = s.total_cost_steps
        # the reference's own CPU run_mlmc, all host threads, bounded to eps >= 1e-5
        if R is not None and eps >= 1e-5:
            o = capi.MlmcOptionsC()
            ablmc.lib().ablmc_mlmc_options_defaults(C.byref(o))
            rr = capi.RunResultC()
            t0 = time.perf_counter()
            rc = R.ref_run_mlmc(C.byref(pr._c), eps, C.byref(o), threads, C.byref(rr))
            if rc == 0:
                row["reference_cpu_seconds"] = time.perf_counter() - t0
                row["reference_cpu_estimate"] = rr.estimate
                row["reference_cpu_threads"] = threads
        res[f"{eps:g}"] = row
    return res


# ---------------------------------------------------------------- B200 arm
def run_b200(a):
    import torch
    import torch.distributed as dist
    from paper_1612_07717_b200 import ablmc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dist_on = world > 1 or a.force_dist
    if dist_on and "RANK" not in os.environ:
        # --force-dist outside torchrun: a one-rank group on the loopback
        os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                          MASTER_PORT=str(free_port()))
    if dist_on:
        # torch.distributed is the plumbing here (barriers, max over ranks,
        # shipping the NCCL unique id); the data path is the library's own NCCL
        # communicator.  NCCL's own log lines ("NCCL version ..." with this
        # image's NCCL_DEBUG=VERSION) go to stderr: stdout carries only the
        # JSON line.
        sys.stdout.flush()
        saved = os.dup(1)
        os.dup2(2, 1)
        try:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            dist.barrier()
            ablmc.init(local)
            from paper_1612_07717_b200.sharding import init_nccl_group
            init_nccl_group()  # native group: ablmc_init_group(local, rank, world, id)
        finally:
            sys.stdout.flush()
            os.dup2(saved, 1)
            os.close(saved)
    else:
        ablmc.init(local)
    # A dedicated (non-default) stream shared by torch and the library, so the
    # CUDA events below bracket exactly the library's kernels.
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ablmc.set_stream(stream.cuda_stream)
    lib = ablmc.lib()

    ig = {"se": 0, "gl": 1, "baoab": 2}[a.integrator]
    level = a.level
    Mf = 1 << level
    N = a.paths
    pr = problem_c(ig)
    pc = C.byref(pr._c)

    def barrier():
        if dist_on:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if not dist_on:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # > 126 MB L2

    def device_step():
        # the whole job's index range [0, world N): in the native group each
        # rank samples its contiguous super-blocks ([r N, (r+1) N) when N is a
        # multiple of 2^22), then ONE all-gather of the partials and the
        # ordered device merge -- every rank ends with the job's moments
        rc = lib.ablmc_accumulate_device(pc, level, 0, world * N)
        if rc:
            ablmc._check(rc)
        return lib.ablmc_last_launch_count(), lib.ablmc_last_collective_count()

    # ---- value: device-resident, CUDA events on the launching stream
    for _ in range(a.warmup):
        device_step()
    barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(a.steps)]
    launches = collectives = 0
    k1_ms, k1_n = C.c_double(), C.c_int64()
    lib.ablmc_level_kernel_times(C.byref(k1_ms), C.byref(k1_n))  # reset
    lib.ablmc_set_profiling(1)
    with ClockSampler(local) as clk:
        for i in range(a.steps):
            flush.zero_()  # L2 flush between timed iterations (outside the events)
            barrier()
            ev[i][0].record(stream)
            nl, nc = device_step()
            ev[i][1].record(stream)
            launches += nl
            collectives += nc
        barrier()
    lib.ablmc_set_profiling(0)
    lib.ablmc_level_kernel_times(C.byref(k1_ms), C.byref(k1_n))
    ms = [s.elapsed_time(e) for s, e in ev]
    total_ms = max_over_ranks(sum(ms))
    k1_avg_ms = k1_ms.value / max(1, k1_n.value)
    k1_share = k1_ms.value / sum(ms)
    steps_per_launch = N * Mf * a.steps / max(1, k1_n.value)
    ms_per_step = total_ms / a.steps
    value = world * N * Mf / (ms_per_step * 1e-3)

    # moments of the last step (sanity: E[Y_10] of the whole job, every rank)
    acc = ablmc.LevelStats().init(level, pr.h_level(level), 1)
    v = acc._view()
    ablmc._check(lib.ablmc_fetch_device_result(pc, level, C.byref(v)))
    acc._take(v)

    fp64_rate = C.c_double()
    ablmc._check(lib.ablmc_probe_fp64_rate(C.byref(fp64_rate)))
    peak = fp64_rate.value
    # dominant kernel (K1, the fused level sampler): FP64-pipe instructions
    # per coupled fine path-step as executed (ncu, profiles/k1_ncu.json: the
    # floor of the bit-exact algorithm as implemented) x path-steps per launch
    # / its average launch duration (CUDA events on its stream)
    traffic, w_exec = None, None
    tp = ROOT / "profiles" / "k1_ncu.json"
    if tp.exists():
        prof = json.loads(tp.read_text()).get(IG_NAME[ig], {})
        if "dram_bytes_per_path_step" in prof:
            traffic = prof["dram_bytes_per_path_step"] * steps_per_launch
            w_exec = prof["fp64_instr_per_path_step"]
    kernel_rate = steps_per_launch / (k1_avg_ms * 1e-3)  # path-steps/s inside K1
    w = w_exec if w_exec is not None else W_ALG[ig]
    achieved = kernel_rate * w

    # ---- e2e: the public API call a user makes (accumulate_samples into a
    # host LevelStats) over the whole job's index range [0, world N): with the
    # native group the library splits it by super-blocks and all-gathers the
    # partials once per call; host<->device traffic inside the timed region
    e2e_times = []
    n_sb = ablmc.num_superblocks(world * N)
    for i in range(a.warmup + a.steps):
        barrier()
        t0 = time.perf_counter()
        e2e_acc = ablmc.LevelStats().init(level, pr.h_level(level), 1)
        ablmc.accumulate_samples(e2e_acc, 0, world * N, pr, level)
        t1 = time.perf_counter()
        if i >= a.warmup:
            e2e_times.append(t1 - t0)
    e2e_t = max_over_ranks(statistics.mean(e2e_times))
    e2e_value = world * N * Mf / e2e_t
    h2d = C.sizeof(pr._c)  # the problem descriptor (kernel parameters) per call
    # the gathered block (all ranks' partial rows + status rows) or, on one
    # device, this rank's super-block partials
    rows = (n_sb + world - 1) // world
    d2h = (world * (rows + 1) * (2 + 3) * 8) if dist_on else n_sb * (2 + 3) * 8

    if rank != 0:
        if dist_on:
            dist.barrier()
            ablmc.init(local)
            dist.destroy_process_group()
        return

    line = {
        "metric": "coupled fine path-steps/s (level sampler)", "value": value,
        "unit": "path-steps/s", "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (Philox seed 42)",
        "config": workload_config(a, world),
        "e2e": {"value": e2e_value, "unit": "path-steps/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": int(launches),
        "collectives": {"per_step": collectives / a.steps,
                        "kind": "ncclAllGather on the library's own communicator" if dist_on
                                else "none (one device)"},
        "roofline": {"bound": "fp64", "achieved": achieved / 1e12, "peak": peak / 1e12,
                     "unit": "FP64 Tops/s (pipe lane-ops)", "frac": achieved / peak,
                     "traffic": traffic,
                     "kernel": "k_level (K1, fused coupled level sampler)",
                     "kernel_avg_ms": k1_avg_ms, "kernel_share_of_step": k1_share,
                     "path_steps_per_launch": steps_per_launch,
                     "W_executed_ncu": w_exec, "W_alg_survey": W_ALG[ig],
                     "frac_W_alg_survey": kernel_rate * W_ALG[ig] / peak,
                     "note": f"achieved = coupled fine path-steps per K1 launch x W = {w:.1f} "
                             "FP64-pipe instructions per path-step as executed (ncu, "
                             "profiles/k1_ncu.json: DFMA/DMUL/DADD/DSETP/MUFU64 of the bit-exact "
                             "algorithm) / K1 launch time, i.e. the FP64-pipe utilisation; "
                             "frac_W_alg_survey uses SURVEY.md 8(d)'s libdevice-based count "
                             f"{W_ALG[ig]:.0f} instead; peak = DFMA probe measured in this run "
                             "(MEASURED_PEAKS.json has no FP64 entry); traffic = ncu DRAM bytes "
                             "per path-step x path-steps per launch"},
        "clocks": clk.summary(),
        "estimate": {"mean_y": acc.mean(), "n": acc.n, "failed": acc.failed},
    }
    if not a.no_extras and world == 1:
        sm = clk.summary()["sm_mhz"]
        line["per_integrator"] = per_integrator(a, lib, stream, fp64_rate.value,
                                                sm * 1e6 if sm else None)
        line["mlmc_time_to_eps"] = mlmc_sweep(a)
        line["baseline_configs"] = configs_sweep(lib, stream)
    if not a.no_cpu_baseline and world == 1:
        threads = host_threads()
        rate, n_cpu, secs = reference_sample(ig, level, a.cpu_seconds, threads)
        rate1, n1, secs1 = reference_sample(ig, level, 3.0, 1)  # also 1 thread
        line["cpu_baseline"] = {"value": rate, "unit": "path-steps/s", "cores": threads,
                                "kind": "reference",
                                "sample": f"{n_cpu} coupled paths x {Mf} fine steps in {secs:.1f} s, "
                                          f"reference accumulate_samples, {threads} threads",
                                "single_thread": {"value": rate1, "paths": n1, "seconds": secs1}}
    print(json.dumps(line), flush=True)
    if dist_on:
        dist.barrier()
        ablmc.init(local)
        dist.destroy_process_group()


def free_port() -> int:
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_spawn(a) -> None:
    """`bench.py --gpus N` outside torchrun: re-exec under
    torch.distributed.run with one rank per GPU (the driver may also launch
    it under torchrun itself; then WORLD_SIZE is set and nothing happens)."""
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1", "--master-port",
               str(free_port()), str(Path(__file__).resolve()), *sys.argv[1:]]
        os.execv(sys.executable, cmd)


def main():
    a = parse()
    maybe_spawn(a)
    if a.impl == "reference":
        run_reference(a)
    else:
        run_b200(a)


if __name__ == "__main__":
    main()
