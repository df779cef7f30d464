#!/bin/bash
# run the GPU suite + b>=6 timings against an experimental library build
for n in "$@"; do
  echo "== $n"
  SPINGP_LIB=tools/vart/lib_$n.so timeout 900 python -m pytest tests -q -m gpu -k "not in_tree_build" 2>&1 | grep -E "^FAILED|passed|failed" | head -20
  for c in cfg4 cfg5; do
  SPINGP_LIB=tools/vart/lib_$n.so timeout 300 python bench.py --config $c --points 1000000 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c 1M', d['ms_per_step'], d['kernels_ms_per_step'])" 2>&1 | tail -1
  done
done
