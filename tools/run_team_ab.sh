python tools/team_check.py 1000000 50000 > gpurun_out/team_check2.log 2>&1
for c in cfg4 cfg5; do
  python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/r02_team_$c.json 2>gpurun_out/r02_team_$c.err
  SPINGP_TEAM=0 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/r02_thread_$c.json 2>&1
done
