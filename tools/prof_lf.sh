#!/bin/bash
# ncu full + source of the fused kernel on longformer and mistral; NEMU sweep
python -m paper_2407_16847_b200.build --force > /dev/null
bash tools/prof.sh longformer lf_cur
bash tools/sweep_nemu.sh "4 8 12 16 20" "longformer" > gpurun_out/sweep_nemu.txt 2>&1
