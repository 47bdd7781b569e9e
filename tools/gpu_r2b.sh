#!/bin/bash
# Round-2 batch B: K4 rewrite (fast delta division, unrolled g_r) parity and
# speed, SE 3-CTA variant A/B, full-size configs 3/4/5.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r2b; R=/tmp/r2b; mkdir -p $O $R
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_extensions.py tests/test_gpu_group.py -q -p no:cacheprovider > $O/tests.log 2>&1
for l in 0 5 10; do timeout 120 python tools/level_bench.py --ig gl --level $l --n 4194304 --x0 0.01 --profile floored --random-u0 --bins 64 --reps 3 | tail -1; done > $O/k4_rates.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_binned -c 1 -f -o $R/k4_l0 \
    python tools/level_bench.py --ig gl --level 0 --n 4194304 --x0 0.01 --profile floored --random-u0 --bins 64 --reps 1 > $O/k4_l0_ncu.log 2>&1
python tools/ncu_summary.py $R/k4_l0.ncu-rep 4194304 > $O/k4_l0.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    python tools/level_bench.py --ig gl --level 0 --n 4194304 --x0 0.01 --profile floored --random-u0 --bins 64 --reps 1 > $O/k4_l0_launches.csv 2>&1
bash tools/ab_run.sh base se3 > $O/ab_se3.txt 2>&1
timeout 900 python tools/full_configs.py --cpu > $O/full_configs.json 2> $O/full_configs.err
ls -la $O; tail -3 $O/tests.log
