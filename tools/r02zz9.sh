#!/bin/bash
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -k "unfused or small or rsddmm or residue or full or coverage or perm" 2>&1 | tail -2
timeout -s KILL 600 python tools/bench_unfused.py --configs longformer,bigbird,sparse_transformer --iters 10 > gpurun_out/r02zz9_unfused.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02zz9_unfused.jsonl'):
    try: d=json.loads(l)
    except Exception: continue
    print(d['config'], {k:(round(d[k]['ms'],3), round(d[k]['frac_hbm'],3)) for k in ('rsddmm','softmax','rspmm')})
PY
