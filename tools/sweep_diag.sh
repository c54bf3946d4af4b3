#!/bin/bash
# GPU box: time the fused kernel of the given configs for several diagnostics builds.
# usage: VARIANTS="-DSPLAT_NEMU=0|-DSPLAT_NEMU=8" CONFIGS="longformer bigbird" bash tools/sweep_diag.sh
IFS='|' read -ra VS <<< "$VARIANTS"
for v in "${VS[@]}"; do
  SPLAT_EXTRA_NVCC_FLAGS="$v" python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  for c in ${CONFIGS:-longformer bigbird}; do
    SPLAT_LIB=diag TAGV="$v" timeout 300 python tools/time_fused.py $c ${STEPS:-20}
  done
done
