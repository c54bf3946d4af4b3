for v in "-DSPLAT_SOFTMAX_ONLINE_MIN=2048" "-DSPLAT_SOFTMAX_ONLINE_MIN=0" "-DSPLAT_SOFTMAX_ONLINE_MIN=256"; do
  SPLAT_EXTRA_NVCC_FLAGS="$v" python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1
  echo "$v"
  SPLAT_LIB=diag timeout 300 python tools/bench_unfused.py --configs longformer,bigbird,sparse_transformer --iters 10 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['config'], {k:(round(d[k]['ms'],3), round(d[k]['frac_hbm'],3)) for k in ('softmax',)})
"
done
