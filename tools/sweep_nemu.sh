#!/bin/bash
# usage (GPU box): tools/sweep_nemu.sh "0 8 12 16" "longformer mistral"
for n in $1; do
  SPLAT_EXTRA_NVCC_FLAGS="-DSPLAT_NEMU=$n" python -m paper_2407_16847_b200.build --diag >/dev/null 2>&1
  ok=$(timeout 60 python -m pytest tests/test_gpu_tc_quick.py -x -q 2>&1 | tail -1)
  for c in $2; do
    r=$(timeout 60 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],4))")
    echo "NEMU=$n $c $r | $ok"
  done
done
