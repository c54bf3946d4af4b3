python -m paper_2407_16847_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "unfused or bf16 or residue or spmm" > gpurun_out/r02f_pytest.txt 2>&1; tail -2 gpurun_out/r02f_pytest.txt
timeout 600 python tools/bench_unfused.py --configs longformer,bigbird --iters 10 > gpurun_out/r02f_unfused.jsonl 2>&1; python -c "
import json
for l in open('gpurun_out/r02f_unfused.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['config'], {k:(round(d[k]['ms'],3), round(d[k]['frac_hbm'],3)) for k in ('rsddmm','softmax','rspmm')})
"
SPLAT_EXTRA_NVCC_FLAGS=-DSPLAT_UNF_PROF python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1
timeout 120 python tools/unf_prof.py longformer
