#!/bin/bash
# GPU box: one ncu --set full capture (source-level) of the kernel matching $2 in `bench.py --config $1`.
# usage: bash tools/ncu_one.sh <config> <kernel-regex> <tag> [skip]
cfg=$1; k=$2; tag=$3; skip=${4:-3}
python -m paper_2407_16847_b200.build > /dev/null
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$k" -s $skip -c 1 \
    -o gpurun_out/${tag} python bench.py --config $cfg --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}.log 2>&1
ls -la gpurun_out/${tag}.ncu-rep
