python -m paper_2407_16847_b200.build > /dev/null 2>&1
timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python tools/sanitize_case.py n512_d64 2>&1 | tail -3
timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python tools/sanitize_case.py st_d128 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q -x -k "unfused or bf16 or residue or spmm or paper_grid" > gpurun_out/r02e_pytest.txt 2>&1; tail -3 gpurun_out/r02e_pytest.txt
timeout 600 python tools/bench_unfused.py --configs longformer,bigbird,sparse_transformer --iters 10 > gpurun_out/r02e_unfused.jsonl 2>&1; python -c "
import json
for l in open('gpurun_out/r02e_unfused.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['config'], {k:(round(d[k]['ms'],3), round(d[k]['frac_hbm'],3)) for k in ('rsddmm','softmax','rspmm')})
"
timeout 120 ./tools/micro/tsx > gpurun_out/r02e_tsx.txt 2>&1; cat gpurun_out/r02e_tsx.txt
