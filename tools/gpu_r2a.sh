#!/bin/bash
# Round-2 batch A: FP64 issue microbenchmark, fp32-variant tests and rates,
# ncu captures (fp32 K1 x3, K4 config 4, K1 SE l10 with source-level stalls),
# summarised on the box (tools/ncu_summary.py); reports kept under /tmp.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r2a; R=/tmp/r2a; mkdir -p $O $R
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fi tools/microbench/fp64_issue.cu && timeout 120 /tmp/fi > $O/fp64_issue.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_extensions.py -q -s -p no:cacheprovider -k fp32 > $O/fp32_tests.log 2>&1
for ig in se gl baoab; do timeout 60 python tools/level_bench.py --ig $ig --level 10 --n 8388608 --fp32 --reps 3 | tail -1; done > $O/fp32_rates.jsonl 2>&1
for l in 0 5 10; do timeout 120 python tools/level_bench.py --ig gl --level $l --n 4194304 --x0 0.01 --profile floored --random-u0 --bins 64 --reps 3 | tail -1; done > $O/k4_rates.jsonl 2>&1
for ig in se gl baoab; do
  timeout 600 ncu --set full --clock-control none -k regex:k_level -c 1 -f -o $R/k1f32_$ig \
    python tools/level_bench.py --ig $ig --level 10 --n 1048576 --fp32 --reps 1 > $O/k1f32_${ig}_ncu.log 2>&1
  python tools/ncu_summary.py $R/k1f32_$ig.ncu-rep 1073741824 > $O/k1f32_${ig}_l10.txt 2>&1
done
for l in 0 10; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_binned -c 1 -f -o $R/k4_l$l \
    python tools/level_bench.py --ig gl --level $l --n 4194304 --x0 0.01 --profile floored --random-u0 --bins 64 --reps 1 > $O/k4_l${l}_ncu.log 2>&1
  python tools/ncu_summary.py $R/k4_l$l.ncu-rep 4194304 > $O/k4_l${l}.txt 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/level_bench.py --ig gl --level $l --n 4194304 --x0 0.01 --profile floored --random-u0 --bins 64 --reps 1 > $O/k4_l${l}_launches.csv 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_level -c 1 -f -o $R/k1_se_src \
  python tools/level_bench.py --ig se --level 10 --n 1048576 --reps 1 > $O/k1_se_src_ncu.log 2>&1
python tools/ncu_summary.py $R/k1_se_src.ncu-rep 1073741824 > $O/k1_se_src.txt 2>&1
ncu -i $R/k1_se_src.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > $O/k1_se_src_sass.csv.gz
ls -la $O; du -sh $O
