#!/bin/bash
# usage (on the GPU box): tools/prof.sh <config> <tag>   -> gpurun_out/prof_<tag>.ncu-rep
cfg=$1; tag=$2
ncu --set full --clock-control none --import-source on -k regex:mhsa_tc -s 2 -c 1 -o gpurun_out/prof_${tag} \
    python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_${tag}.log 2>&1
