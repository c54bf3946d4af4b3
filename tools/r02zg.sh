#!/bin/bash
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k "st_ or residue or sparse_transformer or softmax or small or unfused or full" 2>&1 | tail -2
timeout -s KILL 300 python bench.py --config sparse_transformer --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02zg_bench_st.json 2>/dev/null
python -c "import json; d=json.loads(open('gpurun_out/r02zg_bench_st.json').read().splitlines()[-1]); print('ST', d['value'], d['ms_per_step'], d['roofline']['frac'])"
timeout -s KILL 600 python tools/bench_unfused.py --configs longformer,bigbird,sparse_transformer --iters 10 > gpurun_out/r02zg_unfused.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02zg_unfused.jsonl'):
    try: d=json.loads(l)
    except Exception: continue
    print(d['config'], {k:(round(d[k]['ms'],3), round(d[k]['frac_hbm'],3)) for k in ('rsddmm','softmax','rspmm')})
PY
python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1
SPLAT_SOFTMAX_NOPIPE=1 SPLAT_LIB=diag timeout -s KILL 600 python tools/bench_unfused.py --configs longformer,bigbird --iters 10 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('nopipe', d['config'], round(d['softmax']['ms'],3), round(d['softmax']['frac_hbm'],3))"
