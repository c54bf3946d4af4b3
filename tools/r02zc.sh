#!/bin/bash
# one-launch residue decomposition: parity tests, timing vs the two-launch form, DRAM traffic
mkdir -p gpurun_out
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k "st_ or residue or sparse_transformer" 2>&1 | tail -5
timeout -s KILL 300 python bench.py --config sparse_transformer --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02zc_bench_st.json 2>gpurun_out/r02zc_bench_st.err
python -c "import json; d=json.loads(open('gpurun_out/r02zc_bench_st.json').read().splitlines()[-1]); print('ST one-launch', d['value'], d['ms_per_step'], d['roofline']['frac'])" || tail -5 gpurun_out/r02zc_bench_st.err
python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1
SPLAT_LIB=diag TAGV=one timeout -s KILL 120 python tools/time_fused.py sparse_transformer 20
SPLAT_RESIDUE_2PASS=1 SPLAT_LIB=diag TAGV=two timeout -s KILL 120 python tools/time_fused.py sparse_transformer 20
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:mhsa_tc -c 6 \
   python bench.py --config sparse_transformer --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/r02zc_ncu.txt 2>&1
grep -E "mhsa_tc|dram__bytes|gpu__time" gpurun_out/r02zc_ncu.txt | tail -12
