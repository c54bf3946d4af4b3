#!/bin/bash
# d = 64 split kernel investigation: ncu source-level capture (Longformer) + ablation timings.
mkdir -p gpurun_out
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mhsa_split" -s 3 -c 1 \
    -o gpurun_out/r02zb_split python bench.py --config longformer --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02zb_ncu.log 2>&1
ls -la gpurun_out/r02zb_split.ncu-rep
VARIANTS="-DSPLAT_NEMU=12|-DSPLAT_X_NOSUM|-DSPLAT_X_NOMAX|-DSPLAT_X_NOSUM -DSPLAT_X_NOMAX|-DSPLAT_NEMU=0|-DSPLAT_NEMU=16" \
  CONFIGS="longformer bigbird" bash tools/sweep_diag.sh 2>&1 | tee gpurun_out/r02zb_ablate.txt
SPLAT_EXTRA_NVCC_FLAGS="" python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1
for m in 1 2 3 16 19; do SPLAT_TC_DEBUG=$m SPLAT_LIB=diag TAGV="dbg=$m" timeout 120 python tools/time_fused.py longformer 20; done 2>&1 | tee -a gpurun_out/r02zb_ablate.txt
