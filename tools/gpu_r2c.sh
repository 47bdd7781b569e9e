#!/bin/bash
# Round-2 batch C: SE 3-CTA A/B; level-0 K1 source-level profile; MLMC wall vs K1.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r2c; R=/tmp/r2c; mkdir -p $O $R
bash tools/ab_run.sh base se3 > $O/ab_se3.txt 2>&1
for ig in se baoab; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_level -c 1 -f -o $R/k1_${ig}_l0 \
    python tools/level_bench.py --ig $ig --level 0 --n 4194304 --reps 1 > $O/k1_${ig}_l0_ncu.log 2>&1
python tools/ncu_summary.py $R/k1_${ig}_l0.ncu-rep 4194304 > $O/k1_${ig}_l0.txt 2>&1
ncu -i $R/k1_${ig}_l0.ncu-rep --page source --csv --print-source sass 2>&1 | gzip > $O/k1_${ig}_l0_sass.csv.gz
done
for l in 0 1 2 3; do for ig in se baoab; do timeout 60 python tools/level_bench.py --ig $ig --level $l --n 4194304 --reps 5 | tail -1; done; done > $O/low_levels.jsonl 2>&1
timeout 120 python tools/mlmc_profile.py > $O/mlmc_profile.txt 2>&1
ls -la $O
