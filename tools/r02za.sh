#!/bin/bash
# Session-3 start: full GPU suite, every bench line, unfused timings at HEAD.
TAG=r02za
mkdir -p gpurun_out
python -m paper_2407_16847_b200.build > gpurun_out/${TAG}_build.log 2>&1 || { tail gpurun_out/${TAG}_build.log; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gpu_pytest.txt 2>&1
tail -3 gpurun_out/${TAG}_gpu_pytest.txt
timeout 600 python bench.py > gpurun_out/${TAG}_bench_longformer.json 2> gpurun_out/${TAG}_bench_longformer.err
tail -c 600 gpurun_out/${TAG}_bench_longformer.json
for c in bigbird sparse_transformer mistral tiny; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/${TAG}_bench_$c.json').read().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d['roofline']['frac'])"
done
timeout 600 python tools/bench_unfused.py --configs longformer,bigbird,sparse_transformer --iters 10 > gpurun_out/${TAG}_unfused.jsonl 2>&1
tail -3 gpurun_out/${TAG}_unfused.jsonl | cut -c1-400
