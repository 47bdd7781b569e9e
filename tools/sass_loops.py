"""Static SASS census of the loops in one kernel of libablmc_b200.so:
for every backward branch, the opcode mix of the loop body.
usage: python tools/sass_loops.py MANGLED_NAME_REGEX"""
import collections
import re
import subprocess
import sys

lib = "paper_1612_07717_b200/libablmc_b200.so"
pat = re.compile(sys.argv[1])
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
for f in funcs[1:]:
    name = f.split("\n", 1)[0].strip()
    if not pat.search(name):
        continue
    ins = []
    for line in f.splitlines():
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    addr = {a: i for i, (a, _) in enumerate(ins)}
    print(name[:120], len(ins), "instructions")
    for i, (a, s) in enumerate(ins):
        m = re.search(r"BRA\s+(?:`?\(?)?0x([0-9a-f]+)", s)
        if m and "BRA" in s:
            t = int(m.group(1), 16)
            if t < a and t in addr:
                body = ins[addr[t]:i + 1]
                c = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", x).split()[0].split(".")[0]
                                        for _, x in body)
                fp64 = sum(c[k] for k in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX"))
                print(f"  loop {t:#x}-{a:#x}: {len(body)} instr, fp64 {fp64}: " +
                      ", ".join(f"{k} {v}" for k, v in c.most_common(18)))
    break
