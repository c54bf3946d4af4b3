#!/bin/bash
# GPU box: build, -m gpu tests, and bench lines of the given configs (default: longformer bigbird).
# usage: TAG=r02a bash tools/gpu_check.sh [configs...]
TAG=${TAG:-chk}
python -m paper_2407_16847_b200.build > gpurun_out/${TAG}_build.log 2>&1 || { cat gpurun_out/${TAG}_build.log; exit 1; }
timeout ${TEST_TIMEOUT:-900} python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/${TAG}_pytest.txt 2>&1
tail -5 gpurun_out/${TAG}_pytest.txt
for c in ${@:-longformer bigbird}; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/${TAG}_bench_$c.json').read().splitlines()[-1]); print('$c', round(d['value'],1), 'TF/s', round(d['ms_per_step']*1e3,1), 'us', 'frac', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'])" 2>/dev/null || tail -3 gpurun_out/${TAG}_bench_$c.err
done
