#!/bin/bash
# A/B: level_bench per library variant (paper_1612_07717_b200/variants/lib_<name>.so)
# usage: bash tools/ab_run.sh NAME... (base = the default build)
cd "${GRAFT_REPO_ROOT:-.}"
for lib in "$@"; do
  if [ $lib = base ]; then L=""; else L=paper_1612_07717_b200/variants/lib_$lib.so; fi
  for ig in se gl baoab; do
    echo -n "$lib "; ABLMC_LIB=$L timeout 120 python tools/level_bench.py --ig $ig --n 8388608 --reps 3 2>&1 | tail -1
  done
done
