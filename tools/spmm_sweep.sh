#!/bin/bash
# R-SpMM gather configuration sweep (warpgroups x rows per PARTIAL load batch)
for f in "" "-DSPLAT_UNF_RB=8" "-DSPLAT_UNF_RB=2"; do
  SPLAT_EXTRA_NVCC_FLAGS="$f" python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1
  ok=$(timeout 120 python -m pytest tests/test_gpu_parity.py -q -x -k "unfused_small" 2>&1 | tail -1)
  r=$(timeout 120 python tools/bench_unfused.py --configs longformer,sparse_transformer 2>/dev/null | python3 -c "
import json,sys
print(' '.join('%s=%.3f' % (json.loads(l)['config'][:4], json.loads(l)['rspmm']['ms']) for l in sys.stdin))")
  echo "flags='$f' $r | $ok"
done
python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1
