#!/bin/bash
SPLAT_EXTRA_NVCC_FLAGS="-DSPLAT_MMA_LIVE" python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1 || exit 1
SPLAT_LIB=diag timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -k "lf_ or bb_ or win_d64 or blocked_d64 or longformer or bigbird or split_k or tiny_n or st_res_d64 or strided_d64" 2>&1 | tail -1
for i in 1 2; do
  python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1
  for c in longformer bigbird; do SPLAT_LIB=diag TAGV=base timeout -s KILL 120 python tools/time_fused.py $c 40; done
  SPLAT_EXTRA_NVCC_FLAGS="-DSPLAT_MMA_LIVE" python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1
  for c in longformer bigbird; do SPLAT_LIB=diag TAGV=mmalive timeout -s KILL 120 python tools/time_fused.py $c 40; done
done
