#!/bin/bash
# A/B of library build variants (tools/varlib/*.so, SPINGP_LIB) on cfg4 / cfg5 prefixes
for v in default tools/varlib/libB.so tools/varlib/libC.so; do
  if [ "$v" = default ]; then unset SPINGP_LIB; else export SPINGP_LIB=$PWD/$v; fi
  echo "== $v"
  python bench.py --config cfg4 --points 4000000 --steps 3 --warmup 3 --no-cpu-baseline --no-per-config 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg4 4M', d['ms_per_step'], d['kernels_ms_per_step'])"
  python bench.py --config cfg5 --points 2000000 --steps 2 --warmup 3 --no-cpu-baseline --no-per-config 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg5 2M', d['ms_per_step'], d['kernels_ms_per_step'])"
done
