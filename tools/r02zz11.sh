#!/bin/bash
# d = 64 NEMU re-sweep on the final code (exponentials per 32 on the FMA pipe)
VARIANTS="-DSPLAT_NEMU=12|-DSPLAT_NEMU=8|-DSPLAT_NEMU=10|-DSPLAT_NEMU=14|-DSPLAT_NEMU=12" CONFIGS="longformer bigbird" STEPS=40 bash tools/sweep_diag.sh
