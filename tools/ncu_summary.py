"""Summarise an ncu --set full report of the level-sampler kernel into a text
file for profiles/: key throughput metrics, stall reasons and the dynamic
SASS opcode mix per coupled fine path-step.
usage: python tools/ncu_summary.py REPORT.ncu-rep PATH_STEPS_PER_LAUNCH > out.txt"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, path_steps = sys.argv[1], float(sys.argv[2])


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units, vals = raw[0], raw[1], raw[2]
get = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
print(f"report: {rep}")
print(f"kernel: {get.get('Kernel Name', ('?',))[0]}")
keys = ["gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum"]
for k in keys:
    if k in get:
        print(f"  {k:62s} {get[k][0]} {get[k][1]}")
st = [(float(v), h) for h, v in zip(hdr, vals) if "smsp__pcsamp_warps_issue_stalled" in h
      and not h.endswith("not_issued") and re.match(r"^[0-9.]+$", v or "")]
tot = sum(v for v, _ in st) or 1
print("stall reasons (share of pc samples):")
for v, h in sorted(st, reverse=True)[:10]:
    print(f"  {v / tot * 100:5.1f}%  {h.replace('smsp__pcsamp_warps_issue_stalled_', '')}")
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
h = src[1]
ia, isrc = h.index("Instructions Executed"), h.index("Source")
cnt = collections.Counter()
for r in src[2:]:
    if len(r) > ia and r[ia]:
        s = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip())
        cnt[(s.split()[0] if s else "?").split(".")[0]] += int(r[ia])
total = sum(cnt.values())
print(f"dynamic SASS per coupled fine path-step (thread instructions), total {total * 32 / path_steps:.1f}:")
fp64 = sum(cnt[o] for o in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX")) * 32 / path_steps
print(f"  FP64-pipe (DFMA+DMUL+DADD+DSETP+DMNMX): {fp64:.1f}")
fp32 = sum(cnt[o] for o in ("FFMA", "FMUL", "FADD", "FSETP", "FMNMX", "FSWZADD")) * 32 / path_steps
print(f"  FP32 arithmetic (FFMA+FMUL+FADD+FSETP+FMNMX): {fp32:.1f}")
print(f"  MUFU (XU): {cnt['MUFU'] * 32 / path_steps:.1f}")
for op, n in cnt.most_common(24):
    print(f"  {op:8s} {n * 32 / path_steps:7.2f}")
