#!/usr/bin/env bash
# A/B variant of libablmc_b200.so that recompiles adaptive_kernels.cu only
# (other objects from the default build) -> paper_1612_07717_b200/variants/lib_<name>.so
# usage: tools/build_variant_ad.sh NAME [-DFOO=1 ...]
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
name="$1"; shift
csrc="$ROOT/paper_1612_07717_b200/csrc"; obj="$ROOT/paper_1612_07717_b200/build"
out="$ROOT/paper_1612_07717_b200/variants"; mkdir -p "$out"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off \
  -I"$ROOT/include" "$@" -Xptxas -v -c "$csrc/adaptive_kernels.cu" -o "/tmp/ak_$name.o" 2>"/tmp/ptx_ad_$name.txt"
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/lib_$name.so" "$obj/level_kernels.o" \
  "/tmp/ak_$name.o" "$obj/binned_kernels.o" "$obj/capi.o" "$obj/collective.o" "$obj/drivers.o" "$obj/output.o" -cudart static
awk '/Compiling entry/ {n=$0} /Used|spill/ {print n; print $0}' "/tmp/ptx_ad_$name.txt" \
  | grep -A2 "k_adaptive_persistentILi[012]ELi0ELb1ELi2" | grep -E "Used|spill" | sed "s/^/$name /"
