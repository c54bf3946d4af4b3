#!/bin/bash
# one-launch residue decomposition: lag sweep and immediate-signal ablation (diagnostics builds)
python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1 || exit 1
for L in 2 4 6 8 12 16 24; do SPLAT_MIX_LAG=$L SPLAT_LIB=diag TAGV="lag=$L" timeout -s KILL 120 python tools/time_fused.py sparse_transformer 20; done
SPLAT_RESIDUE_2PASS=1 SPLAT_LIB=diag TAGV=two timeout -s KILL 120 python tools/time_fused.py sparse_transformer 20
SPLAT_EXTRA_NVCC_FLAGS="-DSPLAT_X_DEPNOW" python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1 || exit 1
for L in 2 4 8 12; do SPLAT_MIX_LAG=$L SPLAT_LIB=diag TAGV="depnow lag=$L" timeout -s KILL 120 python tools/time_fused.py sparse_transformer 20; done
