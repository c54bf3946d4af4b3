#!/bin/bash
# one-launch residue kernel: ncu source-level capture (sparse_transformer) + softmax timings after the register-path change
mkdir -p gpurun_out
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"mhsa_tc" -s 1 -c 1 \
    -o gpurun_out/r02ze_mix python bench.py --config sparse_transformer --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/r02ze_ncu.log 2>&1
ls -la gpurun_out/r02ze_mix.ncu-rep
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -x -k "softmax or small or unfused" 2>&1 | tail -2
timeout -s KILL 600 python tools/bench_unfused.py --configs longformer,bigbird,sparse_transformer --iters 10 > gpurun_out/r02ze_unfused.jsonl 2>&1
python - <<'PY'
import json
for l in open('gpurun_out/r02ze_unfused.jsonl'):
    try: d=json.loads(l)
    except Exception: continue
    print(d['config'], {k:(round(d[k]['ms'],3), round(d[k]['frac_hbm'],3)) for k in ('rsddmm','softmax','rspmm')})
PY
