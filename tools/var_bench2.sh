#!/bin/bash
# chunk-count sweep for the b>=6 configs (experiment)
for cfg in cfg4 cfg5; do
  for c in 75776 151552 303104; do
    r=$(SPINGP_CHUNKS=$c timeout 300 python bench.py --config $cfg --points 1000000 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})" 2>&1 | tail -1)
    echo "$cfg chunks=$c: $r"
  done
done
