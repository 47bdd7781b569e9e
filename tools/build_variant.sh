#!/usr/bin/env bash
# Build an A/B variant of libablmc_b200.so with extra -D flags into
# paper_1612_07717_b200/variants/lib_<name>.so (git-ignored; travels with the
# gpurun snapshot; select it with ABLMC_LIB=...).  Needs the default build's
# objects (python -m paper_1612_07717_b200.build) for drivers.o / output.o.
# usage: tools/build_variant.sh NAME [-DFOO=1 ...]
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
name="$1"; shift
csrc="$ROOT/paper_1612_07717_b200/csrc"
obj="$ROOT/paper_1612_07717_b200/build"
out="$ROOT/paper_1612_07717_b200/variants"
mkdir -p "$out"
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-ffp-contract=off -I$ROOT/include"
$NV "$@" -Xptxas -v -c "$csrc/level_kernels.cu" -o "/tmp/lk_$name.o" 2>"/tmp/ptx_$name.txt"
$NV "$@" -Xptxas -v -c "$csrc/adaptive_kernels.cu" -o "/tmp/ak_$name.o" 2>>"/tmp/ptx_$name.txt"
$NV "$@" -c "$csrc/binned_kernels.cu" -o "/tmp/bk_$name.o"
$NV "$@" -c "$csrc/capi.cu" -o "/tmp/capi_$name.o"
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/lib_$name.so" "/tmp/lk_$name.o" \
  "/tmp/ak_$name.o" "/tmp/bk_$name.o" "/tmp/capi_$name.o" "$obj/collective.o" "$obj/drivers.o" \
  "$obj/output.o" \
  -cudart static
awk '/Compiling entry/ {n=$0} /Used|spill/ {print n; print $0}' "/tmp/ptx_$name.txt" \
  | grep -A1 "k_levelILi[012]ELi0ELb1ELb0" | grep -E "Used" | sed "s/^/$name /"
