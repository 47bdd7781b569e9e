#!/bin/bash
# ncu --set full with source-level stall sampling of one level-sampler kernel;
# exports the SASS source page (per-instruction stall samples) as CSV.
# usage: bash tools/gpu_prof_src.sh TAG KERNEL_REGEX -- <command>
cd "${GRAFT_REPO_ROOT:-.}"
tag=$1; kre=$2; shift 3
mkdir -p gpurun_out
"$@" > gpurun_out/${tag}_plain.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -c 1 -f \
  -o gpurun_out/${tag} "$@" > gpurun_out/${tag}_ncu.log 2>&1
ncu -i gpurun_out/${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_sass.csv 2>&1
ncu -i gpurun_out/${tag}.ncu-rep --page source --csv --print-source cuda > gpurun_out/${tag}_cuda.csv 2>&1
ls -la gpurun_out/${tag}*
