#!/bin/bash
# Re-verification of the round-2 state on a fresh box: GPU tests, smoke,
# default bench, reference arm, level sweep.
cd "${GRAFT_REPO_ROOT:-.}"
O=gpurun_out/r2v; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; echo "tests rc=$?" >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
bash tools/level_sweep.sh > $O/level_sweep.jsonl 2>&1
timeout 300 python tools/adaptive_bench.py > $O/adaptive_bench.json 2>&1
tail -3 $O/tests.log; cat $O/smoke.log | tail -2; cat $O/bench.json | cut -c1-600
