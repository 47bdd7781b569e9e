"""Register-file read census of one kernel from an ncu source page (SASS,
with per-instruction execution counts and stall samples):

    python tools/rf_reads.py SASS.csv[.gz] PATH_STEPS_PER_LAUNCH

For every executed instruction it counts the 32-bit vector-register source
reads (RZ, uniform registers, constant-bank operands and immediates are free;
an operand marked .reuse is served by the operand reuse cache; 64-bit
operands of DFMA/DMUL/DADD/DSETP/DMNMX, I2F.*64 and the addend of IMAD.WIDE
read two registers; a register named in several operand slots is read once) and reports, per coupled fine path-step, the reads by
opcode class next to the instruction counts, plus the instructions that
collect the most `dispatch_stall` and `math_pipe_throttle` samples.  The
microbenchmark tools/microbench/fp64_issue.cu measures how many reads per
cycle an SMSP sustains alongside the FP64 pipe."""
import collections
import csv
import gzip
import io
import re
import sys

path, steps = sys.argv[1], float(sys.argv[2])
raw = (gzip.open(path, "rt") if path.endswith(".gz") else open(path)).read()
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
REG = re.compile(r"(-|\|)?\bR(\d+)(\.reuse)?\b")
D64 = ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX")

reads = collections.Counter()
instr = collections.Counter()
stalls = collections.Counter()
per_ins = []
tot_samples = 0
for r in rows[2:]:
    if len(r) <= ci["Instructions Executed"] or not r[ci["Instructions Executed"]]:
        continue
    n = int(r[ci["Instructions Executed"]])
    src = r[ci["Source"]].strip()
    s = re.sub(r"^@!?U?P\w+\s+", "", src)
    op_full = s.split()[0] if s else "?"
    op = op_full.split(".")[0]
    operands = s[len(op_full):].split(",")
    # destination: first operand for everything but stores / compares into predicates
    srcs = operands
    if op not in ("ST", "STS", "STG", "RED", "ATOM", "BRA", "EXIT", "BAR") and operands:
        first = operands[0]
        if REG.search(first) and not op.endswith("SETP"):
            srcs = operands[1:]
    k = 0
    seen = set()
    for j, o in enumerate(srcs):
        for m in REG.finditer(o):
            if m.group(3):  # .reuse
                continue
            if m.group(2) in seen:  # the same register in several slots is read once
                continue            # (fp64_issue.cu: DFMA(d, d, d) runs at the full rate)
            seen.add(m.group(2))
            w = 1
            if op in D64:
                w = 2
            elif op == "I2F" and "64" in op_full.split(".", 1)[-1] and ".F64." not in op_full + ".":
                w = 2 if ".U64" in op_full or ".S64" in op_full else 1
            elif op == "IMAD" and ".WIDE" in op_full and j == 2:
                w = 2
            k += w
    cls = op if op in D64 or op in ("MUFU", "LOP3", "IMAD", "FSEL", "ISETP", "VIADD", "SEL", "LDC",
                                    "LDCU", "SHF", "IADD3", "LEA", "I2F") else "other"
    reads[cls] += k * n
    instr[cls] += n
    sd = int(r[ci["stall_dispatch"]] or 0)
    sm = int(r[ci["stall_math"]] or 0)
    stalls["dispatch"] += sd
    stalls["math"] += sm
    tot_samples += int(r[ci["# Samples"]] or 0)
    per_ins.append((sd, sm, n, k, src))

print(f"per coupled fine path-step (warp-level counts x 32 / path-steps):")
print(f"  {'class':8s} {'instr':>8s} {'reg reads':>10s}")
T_i = T_r = 0.0
for cls in sorted(instr, key=lambda c: -reads[c]):
    i, rr = instr[cls] * 32 / steps, reads[cls] * 32 / steps
    T_i += i
    T_r += rr
    print(f"  {cls:8s} {i:8.1f} {rr:10.1f}")
print(f"  {'total':8s} {T_i:8.1f} {T_r:10.1f}   ({T_r / T_i:.2f} reads per instruction)")
print(f"stall samples: dispatch {stalls['dispatch']}, math {stalls['math']} of {tot_samples}")
print("top dispatch-stall instructions (dispatch, math, executed, reads, source):")
for sd, sm, n, k, src in sorted(per_ins, reverse=True)[:25]:
    print(f"  {sd:7d} {sm:7d} {n:10d} {k:2d}  {src}")
