#!/bin/bash
# final HEAD: full GPU suite, default bench line, smoke
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
timeout -s KILL 1200 python -m pytest tests -m gpu -q > gpurun_out/r02zz18_gpu_pytest.txt 2>&1; tail -1 gpurun_out/r02zz18_gpu_pytest.txt
timeout -s KILL 600 python bench.py > gpurun_out/r02zz18_bench_longformer.json 2>/dev/null
python -c "
import json;d=json.loads(open('gpurun_out/r02zz18_bench_longformer.json').read().splitlines()[-1]);print(round(d['value'],1), round(d['roofline']['frac'],4), round(d['e2e']['value'],2), d['clocks'])
for k,v in d['per_config'].items(): print(k, round(v['value'],1), round(v['ms_per_step']*1e3,1), round(v['roofline']['frac'],3))"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
