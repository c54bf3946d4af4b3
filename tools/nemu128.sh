#!/bin/bash
# NEMU sweep for the d = 128 paired kernel (exponentials emulated on the FMA pipe per 32)
for n in 0 4 8 12; do
  SPLAT_EXTRA_NVCC_FLAGS="-DSPLAT_NEMU128=$n" python -m paper_2407_16847_b200.build --diag >/dev/null 2>&1
  ok=$(timeout 100 python -m pytest tests/test_gpu_tc_quick.py -x -q 2>&1 | tail -1)
  for c in mistral sparse_transformer; do
    r=$(timeout 90 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), d['clocks']['sm_mhz'])")
    echo "NEMU128=$n $c $r | $ok"
  done
done
python -m paper_2407_16847_b200.build --diag >/dev/null 2>&1
