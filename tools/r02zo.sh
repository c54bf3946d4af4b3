#!/bin/bash
SPLAT_EXTRA_NVCC_FLAGS="-DSPLAT_UNF_PROF" python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1 || exit 1
timeout -s KILL 120 python tools/unf_prof_sddmm.py longformer
timeout -s KILL 120 python tools/unf_prof_sddmm.py bigbird
