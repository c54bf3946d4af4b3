#!/bin/bash
# usage (on the GPU box): tools/prof_unfused.sh <config> <kernel-regex> <tag> -> gpurun_out/prof_<tag>.ncu-rep
cfg=$1; k=$2; tag=$3
ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_${tag} \
    python tools/bench_unfused.py --configs $cfg --iters 1 > gpurun_out/ncu_${tag}.log 2>&1
