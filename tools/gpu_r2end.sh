#!/bin/bash
# End-of-round-2 verification on a fresh box at HEAD: GPU tests, smoke,
# default bench, the same bench through the library's NCCL path at world
# size 1 (--force-dist: pack + ncclAllGather + grouped merge on every step),
# reference arm, ncu launch list of the bench command.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r2end; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 300 python bench.py --force-dist --no-extras --no-cpu-baseline > $O/bench_dist1.json 2> $O/bench_dist1.err
timeout 300 python bench.py --no-extras --no-cpu-baseline > $O/bench_plain.json 2> $O/bench_plain.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_bench_dist1.csv python bench.py --force-dist --no-extras --no-cpu-baseline \
  --steps 2 --warmup 3 > $O/ncu_dist1.log 2>&1
tail -3 $O/tests.log; tail -2 $O/smoke.log
for f in bench bench_dist1 bench_plain bench_ref; do echo "== $f"; cut -c1-500 $O/$f.json; tail -2 $O/$f.err; done
