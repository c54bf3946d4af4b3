#!/bin/bash
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests -m gpu -q -x -k "softmax or unfused or small or full or coverage" > gpurun_out/r02zz15_pytest.txt 2>&1; tail -1 gpurun_out/r02zz15_pytest.txt
timeout -s KILL 600 python tools/bench_unfused.py --configs longformer,bigbird,sparse_transformer --iters 10 > gpurun_out/r02zz15_unfused.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02zz15_unfused.jsonl'):
    try: d=json.loads(l)
    except Exception: continue
    print(d['config'], {k:(round(d[k]['ms'],3), round(d[k]['frac_hbm'],3)) for k in ('rsddmm','softmax','rspmm')})
PY
