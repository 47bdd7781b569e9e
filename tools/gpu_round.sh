#!/bin/bash
# One GPU session: device tests, per-integrator K1 throughput, ncu captures of
# K1 (SE/GL/BAOAB, level 10, 2^20 paths).  usage: bash tools/gpu_round.sh TAG
cd "${GRAFT_REPO_ROOT:-.}"
tag=${1:-r}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
for ig in se gl baoab; do
  timeout 120 python tools/level_bench.py --ig $ig --n 8388608 --reps 3 >> gpurun_out/${tag}_level.jsonl 2>&1
done
if [ "${NCU:-1}" = 1 ]; then
  for ig in se gl baoab; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_level -c 1 -f \
      -o gpurun_out/${tag}_k1_$ig python tools/level_bench.py --ig $ig --n 1048576 --reps 1 \
      > gpurun_out/${tag}_ncu_$ig.log 2>&1
    python tools/ncu_summary.py gpurun_out/${tag}_k1_$ig.ncu-rep 1073741824 > gpurun_out/${tag}_ncu_k_level_${ig}_l10.txt 2>&1
    ls -la gpurun_out/${tag}_k1_$ig.ncu-rep >> gpurun_out/${tag}_ncu_$ig.log
    [ $ig = se ] || rm -f gpurun_out/${tag}_k1_$ig.ncu-rep   # stay under gpurun's 64 MiB copy-back
  done
fi
