#!/bin/bash
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
timeout -s KILL 600 python -m pytest tests -m gpu -q -x -k "host or boundary" 2>&1 | tail -2
for i in 1 2; do
timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/r02zl_bench.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/r02zl_bench.json').read().splitlines()[-1]); print('longformer', round(d['value'],1), 'e2e', d['e2e'])"
done
