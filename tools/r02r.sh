TAG=r02r bash tools/r02_full.sh
timeout 900 python tools/bench_unfused.py --configs longformer,bigbird,sparse_transformer --iters 10 > gpurun_out/r02r_unfused.jsonl 2>&1; python -c "
import json
for l in open('gpurun_out/r02r_unfused.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['config'], {k:(round(d[k]['ms'],3), round(d[k]['frac_hbm'],3)) for k in ('rsddmm','softmax','rspmm')})
"
