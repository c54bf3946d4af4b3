#!/bin/bash
# early S(j+1) load in the d = 64 split kernel (A/B, diagnostics builds); HBM / PCIe bandwidth by
# direction; launch list of the headline bench command alone
mkdir -p gpurun_out
python tools/hbm_rw.py > gpurun_out/r02zk_hbm_rw.json 2>&1; cat gpurun_out/r02zk_hbm_rw.json
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02zk_launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-per-config > /dev/null 2>&1
VARIANTS="-DSPLAT_NEMU=12|-DSPLAT_EARLY_S" CONFIGS="longformer bigbird" STEPS=30 bash tools/sweep_diag.sh
SPLAT_EXTRA_NVCC_FLAGS="-DSPLAT_EARLY_S" python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1
SPLAT_LIB=diag timeout -s KILL 300 python -m pytest tests/test_gpu_tc_quick.py -q -x 2>&1 | tail -2
