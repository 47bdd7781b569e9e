#!/bin/bash
# Round-2 record: default bench (N=1), reference arm, ncu launch list of the
# bench command, K1 full captures (GL, BAOAB; SE has the source-level one).
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r2g; R=/tmp/r2g; mkdir -p $O $R
python bench.py > $O/bench.json 2> $O/bench.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench_se_l10.csv \
  python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > $O/ncu_bench.log 2>&1
for ig in gl baoab se; do
  timeout 900 ncu --set full --clock-control none -k regex:k_level -c 1 -f -o $R/k1_$ig \
    python tools/level_bench.py --ig $ig --level 10 --n 1048576 --reps 1 > $O/k1_${ig}_ncu.log 2>&1
  python tools/ncu_summary.py $R/k1_$ig.ncu-rep 1073741824 > $O/k1_${ig}_l10.txt 2>&1
done
python tools/mlmc_profile.py > $O/mlmc_profile.txt 2>&1
python tools/mlmc_timeline.py 1e-4 > $O/mlmc_timeline.txt 2>&1
ls -la $O
