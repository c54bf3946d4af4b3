#!/bin/bash
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -x -k "st_res or residue or sparse_transformer" 2>&1 | tail -2
python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1 || exit 1
for L in 2 4 8 16; do SPLAT_MIX_LAG=$L SPLAT_LIB=diag TAGV="lag=$L" timeout -s KILL 120 python tools/time_fused.py sparse_transformer 20; done
SPLAT_RESIDUE_2PASS=1 SPLAT_LIB=diag TAGV=two timeout -s KILL 120 python tools/time_fused.py sparse_transformer 20
