#!/bin/bash
# A/B: level_bench per library variant, then GPU tests on the variants
cd $GRAFT_REPO_ROOT
for lib in base icd icdr; do
  if [ $lib = base ]; then L=""; else L=paper_1612_07717_b200/variants/lib_$lib.so; fi
  for ig in se gl baoab; do
    echo -n "$lib "; ABLMC_LIB=$L timeout 120 python tools/level_bench.py --ig $ig --n 8388608 --reps 3 2>&1 | tail -1
  done
done
for lib in icd icdr; do
  echo "== tests $lib"; ABLMC_LIB=paper_1612_07717_b200/variants/lib_$lib.so timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
done
