python -m paper_2407_16847_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "tiny or fp32 or paper_grid or small or edge" > gpurun_out/r02s_pytest.txt 2>&1; tail -2 gpurun_out/r02s_pytest.txt
for i in 1 2 3; do timeout 300 python bench.py --config tiny --steps 50 --warmup 5 --no-cpu-baseline --no-per-config 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('tiny', round(d['ms_per_step']*1e3,2), 'us')"; done
