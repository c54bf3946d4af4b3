#!/bin/bash
python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1 || exit 1
for i in 1 2; do
SPLAT_LIB=diag TAGV=ksplit timeout -s KILL 120 python tools/e2e_time.py longformer
SPLAT_NO_KSPLIT=1 SPLAT_LIB=diag TAGV=noksplit timeout -s KILL 120 python tools/e2e_time.py longformer
done
