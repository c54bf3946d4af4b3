#!/bin/bash
# host pipeline chunk count vs e2e time (diagnostics builds)
for n in 12 6 8 15 4; do
  SPLAT_EXTRA_NVCC_FLAGS="-DSPLAT_HOST_CHUNKS=$n" python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1 || continue
  for i in 1 2; do SPLAT_LIB=diag TAGV="chunks=$n" timeout -s KILL 120 python tools/e2e_time.py longformer; done
done
