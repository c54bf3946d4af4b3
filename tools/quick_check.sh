#!/bin/bash
# quick GPU check: tc tests, full gpu parity, bench lines for all configs
python -m paper_2407_16847_b200.build > /dev/null
timeout 120 python -m pytest tests/test_gpu_tc_quick.py -x -q 2>&1 | tail -3
timeout 400 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in ${CONFIGS:-longformer bigbird sparse_transformer mistral}; do
  timeout 90 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['value'],1), 'TF/s', round(d['ms_per_step'],4), 'ms', d['roofline']['frac'])"
done
