#!/bin/bash
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for c in longformer bigbird; do timeout -s KILL 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-per-config 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('$c', round(d['value'],1), round(d['ms_per_step']*1e3,1), 'us', d['config']['plan'])"; done
for c in longformer bigbird; do timeout -s KILL 300 python tools/shard_sim.py $c; done | tee gpurun_out/r02zt_shard_sim.jsonl
