#!/bin/bash
cat > /tmp/prof_team.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_1610_08035_b200 as P
from paper_1610_08035_b200 import datasets
name, n = sys.argv[1], int(sys.argv[2])
w = datasets.make(name, **({"n": n} if n else {}))
with P.Context(0) as ctx:
    for _ in range(2):
        ctx.eval(w.leaves, w.theta, w.t, w.y, w.sigma, grad=True, var="var" in w.outputs)
PY
for cfg in cfg4 cfg5; do
  n=0; [ $cfg = cfg5 ] && n=2000000
  for k in k_rev0_team k_fwd0_team; do
    ncu --set full --import-source on --clock-control none -k regex:"$k" -s 1 -c 1 -o /tmp/p_${cfg}_$k python /tmp/prof_team.py $cfg $n > gpurun_out/p_${cfg}_$k.log 2>&1
    ncu -i /tmp/p_${cfg}_$k.ncu-rep --page details --csv > gpurun_out/r02b_ncu_${cfg}_${k}_details.csv 2>/dev/null
    ncu -i /tmp/p_${cfg}_$k.ncu-rep --page raw --csv > gpurun_out/r02b_ncu_${cfg}_${k}_raw.csv 2>/dev/null
  done
done
