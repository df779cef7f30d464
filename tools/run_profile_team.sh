#!/bin/bash
# ncu captures of the b >= 6 team kernels (cfg4 and cfg5 prefixes) and the solve-operator
# chunk-count sweep.  Outputs under gpurun_out/.
set -x
for CH in 75776 40000 20000 10000 5000; do
  SPINGP_CHUNKS=$CH python tools/bench_solve.py 1000000 3 20 > gpurun_out/solve_ch$CH.json 2>&1
done
cat > /tmp/prof_team.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import paper_1610_08035_b200 as P
from paper_1610_08035_b200 import datasets
name, n = sys.argv[1], int(sys.argv[2])
w = datasets.make(name, n=n)
with P.Context(0) as ctx:
    for _ in range(2):
        ctx.eval(w.leaves, w.theta, w.t, w.y, w.sigma, grad=True, var="var" in w.outputs)
PY
ncu --set full --import-source on --clock-control none -k regex:k_rev0_team -s 1 -c 1 -o gpurun_out/ncu_rev0_team_cfg4 python /tmp/prof_team.py cfg4 1000000 > gpurun_out/ncu_rev0_team_cfg4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_fwd0_team -s 1 -c 1 -o gpurun_out/ncu_fwd0_team_cfg4 python /tmp/prof_team.py cfg4 1000000 > gpurun_out/ncu_fwd0_team_cfg4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_rev0_team -s 1 -c 1 -o gpurun_out/ncu_rev0_team_cfg5 python /tmp/prof_team.py cfg5 200000 > gpurun_out/ncu_rev0_team_cfg5.log 2>&1
# e2e pipeline pieces (cfg2 host-pointer call)
for pp in "4 2" "4 4" "8 4" "8 8" "16 8"; do set -- $pp
  SPINGP_PIPE_IN=$1 SPINGP_PIPE_OUT=$2 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-per-config > gpurun_out/e2e_pipe_$1_$2.json 2>&1
done
