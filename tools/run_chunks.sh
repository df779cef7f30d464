#!/bin/bash
# level-0 chunk-count sweep for the b >= 6 configs at full size (SPINGP_CHUNKS = target chunks)
for CH in 75776 32768 16384 8192; do
  echo "== chunks $CH"
  SPINGP_CHUNKS=$CH python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline --no-per-config 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg4', d['ms_per_step'], d['kernels_ms_per_step'])"
  SPINGP_CHUNKS=$CH python bench.py --config cfg5 --steps 2 --warmup 3 --no-cpu-baseline --no-per-config 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg5', d['ms_per_step'], d['kernels_ms_per_step'])"
done
