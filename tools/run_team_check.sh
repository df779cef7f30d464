python tools/team_check.py 1000000 50000 > gpurun_out/team_check3.log 2>&1
python bench.py --config cfg4 --steps 3 --warmup 3 --no-cpu-baseline --no-per-config 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg4', d['ms_per_step'], d['kernels_ms_per_step'])" >> gpurun_out/team_check3.log
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "cfg4 or eval_matches" >> gpurun_out/team_check3.log 2>&1
