#!/bin/bash
# mbarrier try_wait suspend-time hint sweep (ns): fused Longformer + unfused R-SpMM
for f in "" "-DSPLAT_WAIT_HINT=2000" "-DSPLAT_WAIT_HINT=100000"; do
  SPLAT_EXTRA_NVCC_FLAGS="$f" python -m paper_2407_16847_b200.build --force > /dev/null 2>&1
  ok=$(timeout 100 python -m pytest tests/test_gpu_tc_quick.py -x -q 2>&1 | tail -1)
  r=$(timeout 90 python bench.py --config longformer --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1))")
  u=$(timeout 120 python tools/bench_unfused.py --configs longformer 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('spmm', round(d['rspmm']['ms'],3), 'sddmm', round(d['rsddmm']['ms'],3))")
  echo "flags='$f' fused $r | $u | $ok"
done
python -m paper_2407_16847_b200.build --force > /dev/null 2>&1
