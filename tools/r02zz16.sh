#!/bin/bash
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
timeout -s KILL 600 python bench.py > gpurun_out/r02zz16_bench_longformer.json 2> gpurun_out/r02zz16_bench.err
python -c "
import json;d=json.loads(open('gpurun_out/r02zz16_bench_longformer.json').read().splitlines()[-1]);print(round(d['value'],1), round(d['roofline']['frac'],4), d['config']['plan'])
for k,v in d['per_config'].items(): print(k, round(v['value'],1), round(v['ms_per_step']*1e3,1), round(v['roofline']['frac'],3), v['plan'].get('fused_d64'))" || tail -5 gpurun_out/r02zz16_bench.err
