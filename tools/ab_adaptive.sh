#!/bin/bash
# A/B of library variants on the adaptive sampler (tools/adaptive_bench.py keys).
# usage: bash tools/ab_adaptive.sh base ad192 ...
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for lib in "$@"; do
  if [ $lib = base ]; then L=""; else L=paper_1612_07717_b200/variants/lib_$lib.so; fi
  for rep in 1 2; do
  ABLMC_LIB=$L timeout 300 python tools/adaptive_bench.py se_adaptive_l3 gl_adaptive_l3 baoab_adaptive_l3 se_adaptive_l0 2>&1 | \
    grep adaptive_l | python -c "
import sys, json
for line in sys.stdin:
    k, d = line.split(' ', 1); d = json.loads(d)
    print('$lib', k, round(d['ms'], 3), 'ms', '%.3e steps/s' % d['steps_per_s'])"
  done
done
