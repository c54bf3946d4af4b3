#!/bin/bash
# residue path after reverting the L2-only loads; one-launch experiment re-measured; d = 64 micro-variants
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
timeout -s KILL 120 python tools/time_fused.py sparse_transformer 30 | sed 's/^/product /'
python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1 || exit 1
SPLAT_LIB=diag timeout -s KILL 120 python tools/time_fused.py sparse_transformer 30 | sed 's/^/diag-2pass /'
for L in 4 8; do SPLAT_RESIDUE_1PASS=1 SPLAT_MIX_LAG=$L SPLAT_LIB=diag timeout -s KILL 120 python tools/time_fused.py sparse_transformer 30 | sed "s/^/diag-1pass lag=$L /"; done
VARIANTS="-DSPLAT_NEMU=12|-DSPLAT_X_LIVELD|-DSPLAT_RESCALE_T=16.0f|-DSPLAT_X_LIVELD -DSPLAT_RESCALE_T=16.0f" CONFIGS="longformer bigbird" STEPS=30 bash tools/sweep_diag.sh
