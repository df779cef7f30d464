python tools/team_check.py 1000000 50000 > gpurun_out/team_check5.log 2>&1
for c in cfg4 cfg5; do
python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-per-config 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['kernels_ms_per_step'])" >> gpurun_out/team_check5.log
done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py tests/test_predict.py tests/test_gpu_three_way.py -m gpu -q -x >> gpurun_out/team_check5.log 2>&1
