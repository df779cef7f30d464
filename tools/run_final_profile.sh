#!/bin/bash
# Round-2 evidence run: bench (default + reference arm), ncu launch list of the bench
# command, ncu full sets of the dominant kernels (cfg2, cfg4, cfg5, solve operator),
# kept as text pages (details + raw) so the output stays small.
set -x
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/final_launches_cfg2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/final_launches_cfg2.log 2>&1
cap() {  # name, kernel regex, skip, count, command...
  local name=$1 kr=$2 sk=$3 cn=$4; shift 4
  ncu --set full --import-source on --clock-control none -k regex:"$kr" -s $sk -c $cn -o /tmp/$name "$@" > gpurun_out/$name.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/${name}_details.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /dev/null 2>&1
}
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
cat > /tmp/prof_solve.py <<'PY'
import sys, os
sys.path.insert(0, os.path.join(os.getcwd(), "tools")); sys.path.insert(0, os.getcwd())
import bench_solve
print(bench_solve.measure(n=1_000_000, b=3, steps=3))
PY
cap final_ncu_cfg2 "k_(rev0|fwd0|tree_coop|reduce)" 0 4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-per-config
cap final_ncu_cfg4 "k_(rev0|fwd0)_team|k_upper" 3 3 python /tmp/prof_team.py cfg4 0
cap final_ncu_cfg5 "k_(rev0|fwd0)_team|k_upper" 3 3 python /tmp/prof_team.py cfg5 2000000
cap final_ncu_solve "k_solve_strip" 3 1 python /tmp/prof_solve.py
SPINGP_SOLVE_STRIP=0 python tools/stream_time.py tile-kernel > gpurun_out/final_stream_tile_time.log 2>&1
cap final_ncu_solve_partitioned "k_(fwdL|revL|tree)" 6 3 python /tmp/prof_solve.py
SPINGP_SS_STAMPS=1 python tools/stream_stamps.py > gpurun_out/final_stream_stamps.log 2>&1
ls -la gpurun_out
