#!/bin/bash
# d = 128 kernel: exponentials emulated on the FMA pipe per 32 (NEMU128) on Mistral and Sparse-TF
for n in 4 0 8 12; do
  SPLAT_EXTRA_NVCC_FLAGS="-DSPLAT_NEMU128=$n" python -m paper_2407_16847_b200.build --diag >/dev/null 2>&1 || { echo "build fail $n"; continue; }
  for c in mistral sparse_transformer; do SPLAT_LIB=diag TAGV="NEMU128=$n" timeout -s KILL 200 python tools/time_fused.py $c 8; done
done
