#!/bin/bash
# Per-level accumulate time of the device sampler (reference profile, x0 = 0.5,
# M0 = 1, 2^22 samples per call; level 10 with 2^23) for SE/GL/BAOAB: one
# JSON line per (integrator, level).  usage: bash tools/level_sweep.sh > out.jsonl
cd "${GRAFT_REPO_ROOT:-.}"
for l in 0 1 2 3 4 6 8; do for ig in se gl baoab; do
  timeout 60 python tools/level_bench.py --ig $ig --level $l --n 4194304 --reps 5 2>&1 | tail -1
done; done
for ig in se gl baoab; do timeout 120 python tools/level_bench.py --ig $ig --level 10 --n 8388608 --reps 3 2>&1 | tail -1; done
