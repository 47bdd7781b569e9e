#!/bin/bash
# A/B of library variants at given levels: "lib ig level ms" per line.
# usage: bash tools/ab_levels.sh "0 1" base u2 ...   (n = 2^22 samples, 10 reps)
cd "${GRAFT_REPO_ROOT:-.}"
levels=$1; shift
for lib in "$@"; do
  if [ $lib = base ]; then L=""; else L=paper_1612_07717_b200/variants/lib_$lib.so; fi
  for l in $levels; do for ig in se gl baoab; do
    ABLMC_LIB=$L timeout 120 python tools/level_bench.py --ig $ig --level $l --n 4194304 --reps 10 2>&1 | tail -1 | \
      python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$lib', d['ig'], d['level'], round(d['ms'], 4))" 2>&1
  done; done
done
