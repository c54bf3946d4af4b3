python -m paper_2407_16847_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "unfused or bf16 or residue or spmm or softmax or paper_grid or tiny or fp32" > gpurun_out/r02n_pytest.txt 2>&1; tail -2 gpurun_out/r02n_pytest.txt
timeout 600 python tools/bench_unfused.py --configs longformer,bigbird,sparse_transformer --iters 10 > gpurun_out/r02n_unfused.jsonl 2>&1; python -c "
import json
for l in open('gpurun_out/r02n_unfused.jsonl'):
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['config'], {k:(round(d[k]['ms'],3), round(d[k]['frac_hbm'],3)) for k in ('rsddmm','softmax','rspmm')})
"
for c in longformer bigbird; do timeout 120 python tools/time_fused.py $c 20; done
