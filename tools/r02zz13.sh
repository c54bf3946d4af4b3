#!/bin/bash
for v in "" "-DSPLAT_QPF"; do
  SPLAT_EXTRA_NVCC_FLAGS="$v" python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1 || { echo "build fail $v"; continue; }
  for i in 1 2; do for c in sparse_transformer mistral; do SPLAT_LIB=diag TAGV="[$v]" timeout -s KILL 200 python tools/time_fused.py $c 10; done; done
done
SPLAT_EXTRA_NVCC_FLAGS="-DSPLAT_QPF" python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1
SPLAT_LIB=diag timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -x -k "st_ or residue or mis or perm" 2>&1 | tail -1
