#!/bin/bash
# level-0 occupancy / chunk-count sweep (experiment): lib variant x SPINGP_CHUNKS
for v in main; do
  lib=tools/vart/lib_$v.so; [ $v = main ] && lib=paper_1610_08035_b200/libspingp_b200.so
  for c in 75776 113664 151552 227328; do
    r=$(SPINGP_LIB=$lib SPINGP_CHUNKS=$c timeout 120 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['kernels_ms_per_step'].items()})" 2>&1 | tail -1)
    echo "$v chunks=$c: $r"
  done
done
