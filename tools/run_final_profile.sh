#!/bin/bash
# Round-2 evidence run: bench (default + reference arm), ncu launch list of the bench
# command, ncu full sets of the dominant kernels (cfg2, cfg4, cfg5, solve operator).
set -x
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/final_launches_cfg2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_(rev0|fwd0|tree_coop|reduce)" -c 4 -o gpurun_out/final_ncu_cfg2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/final_ncu_cfg2.log 2>&1
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
ncu --set full --import-source on --clock-control none -k regex:"k_(rev0|fwd0)_team|k_upper" -s 3 -c 3 -o gpurun_out/final_ncu_cfg4 python /tmp/prof_team.py cfg4 0 > gpurun_out/final_ncu_cfg4.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"k_(rev0|fwd0)_team|k_upper" -s 3 -c 3 -o gpurun_out/final_ncu_cfg5 python /tmp/prof_team.py cfg5 2000000 > gpurun_out/final_ncu_cfg5.log 2>&1
cat > /tmp/prof_solve.py <<'PY'
import sys, os
sys.path.insert(0, os.path.join(os.getcwd(), "tools")); sys.path.insert(0, os.getcwd())
import bench_solve
print(bench_solve.measure(n=1_000_000, b=3, steps=3))
PY
ncu --set full --import-source on --clock-control none -k regex:"k_(fwdL|revL|tree)" -s 6 -c 6 -o gpurun_out/final_ncu_solve python /tmp/prof_solve.py > gpurun_out/final_ncu_solve.log 2>&1
