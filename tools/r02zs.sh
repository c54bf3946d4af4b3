#!/bin/bash
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
for c in longformer bigbird sparse_transformer; do timeout -s KILL 300 python tools/shard_sim.py $c; done | tee gpurun_out/r02zs_shard_sim.jsonl
