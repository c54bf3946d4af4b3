python -m paper_2407_16847_b200.build > /dev/null 2>&1
timeout 300 compute-sanitizer --tool memcheck python tools/spmm_case.py longformer 2 2>&1 | tail -1
timeout 300 compute-sanitizer --tool synccheck python tools/spmm_case.py bigbird 2 2>&1 | tail -1
timeout 300 compute-sanitizer --tool racecheck python tools/spmm_case.py longformer 2 2>&1 | grep SUMMARY
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "unfused or bf16 or residue or spmm" > gpurun_out/r02y_pytest.txt 2>&1; tail -1 gpurun_out/r02y_pytest.txt
timeout 600 python tools/bench_unfused.py --configs longformer,bigbird,sparse_transformer --iters 10 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['config'], {k:(round(d[k]['ms'],3), round(d[k]['frac_hbm'],3)) for k in ('rspmm',)})
"
