# softmax register-resident rows: parity (unfused tests) and timing vs the three-pass kernel
python -m paper_2407_16847_b200.build > /dev/null 2>&1
python -c "from paper_2407_16847_b200 import build; build.build(diag=True)" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "unfused or softmax or full_size" > gpurun_out/r02ad_pytest.txt 2>&1; tail -1 gpurun_out/r02ad_pytest.txt
for rc in 1 0; do
  echo "RC knob $rc"
  SPLAT_LIB=diag SPLAT_SOFTMAX_RC=$rc timeout 300 python tools/bench_unfused.py --max-bh 32 --configs longformer,bigbird,mistral 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: continue
    print(d['config'], 'softmax', round(d['softmax']['ms'], 4), round(d['softmax']['frac_hbm'], 3))"
done
