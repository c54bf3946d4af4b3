#!/bin/bash
# R-SpMM ring depths (d = 64): V ring x P staging stages
for v in "-DSPLAT_SPMM_KS64=3 -DSPLAT_SPMM_NSTG=4" "-DSPLAT_SPMM_KS64=2 -DSPLAT_SPMM_NSTG=5" "-DSPLAT_SPMM_KS64=2 -DSPLAT_SPMM_NSTG=4"; do
  SPLAT_EXTRA_NVCC_FLAGS="$v" python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1 || { echo "build fail $v"; continue; }
  SPLAT_LIB=diag timeout -s KILL 300 python tools/bench_unfused.py --configs longformer,bigbird --iters 10 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$v', d['config'], round(d['rspmm']['ms'],4), round(d['rspmm']['frac_hbm'],3))"
done
