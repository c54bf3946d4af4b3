python -m paper_2407_16847_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "unfused or tiny or paper_grid or bigbird_unfused or mistral_unfused or fp32_wide or coverage" > gpurun_out/r02h_pytest.txt 2>&1; tail -3 gpurun_out/r02h_pytest.txt
timeout 600 python tools/bench_unfused.py --configs longformer,bigbird,sparse_transformer --iters 10 > gpurun_out/r02h_unfused.jsonl 2>&1; cat gpurun_out/r02h_unfused.jsonl | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d.get('config'), {k:(round(v['ms']*1e3,1), round(v.get('frac_hbm',0),3)) for k,v in d.items() if isinstance(v,dict) and 'ms' in v})
"
