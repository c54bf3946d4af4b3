for v in "" "-DSPLAT_SPMM_NOEXP"; do
  SPLAT_EXTRA_NVCC_FLAGS="$v" python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1 || echo "build fail $v"
  echo "variant: $v"
  SPLAT_LIB=diag timeout 300 python tools/bench_unfused.py --configs longformer,bigbird --iters 5 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['config'], {k:(round(d[k]['ms'],3), round(d[k]['frac_hbm'],3)) for k in ('rspmm',)})
"
done
SPLAT_EXTRA_NVCC_FLAGS="-DSPLAT_SPMM_NOEXP -DSPLAT_UNF_PROF" python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1
python tools/unf_prof.py longformer | grep -v "warp  [2-7] \|warp  9\|warp 1[0-5]\|warp 1[7-9]\|warp 2[1-3]"
