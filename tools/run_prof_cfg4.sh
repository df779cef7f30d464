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
  ncu --set full --import-source on --clock-control none -k regex:"k_(rev0|fwd0)_team|k_(fwd|rev)L_team" -s 4 -c 4 -o /tmp/p_$cfg python /tmp/prof_team.py $cfg $n > gpurun_out/p_$cfg.log 2>&1
  ncu -i /tmp/p_$cfg.ncu-rep --page details --csv > gpurun_out/r02b_ncu_${cfg}_details.csv 2>/dev/null
  ncu -i /tmp/p_$cfg.ncu-rep --page raw --csv > gpurun_out/r02b_ncu_${cfg}_raw.csv 2>/dev/null
done
