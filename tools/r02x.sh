python -m paper_2407_16847_b200.build > /dev/null 2>&1
timeout 600 compute-sanitizer --tool racecheck --print-limit 2 python tools/spmm_case.py longformer 2 2>&1 | grep -E "SUMMARY|Race|Read access" | head -6
timeout 600 compute-sanitizer --tool synccheck python tools/spmm_case.py bigbird 2 2>&1 | tail -1
TAG=r02x bash tools/sanitize_all.sh
timeout 900 python -m pytest tests -m gpu -q -x -k "unfused or bf16 or fused or uniform or d64 or deterministic" > gpurun_out/r02x_pytest.txt 2>&1; tail -1 gpurun_out/r02x_pytest.txt
for c in longformer bigbird; do timeout 120 python tools/time_fused.py $c 20; done
timeout 600 python tools/bench_unfused.py --configs longformer,bigbird --iters 10 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(d['config'], {k:(round(d[k]['ms'],3), round(d[k]['frac_hbm'],3)) for k in ('rspmm',)})
"
