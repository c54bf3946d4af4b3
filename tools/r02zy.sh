#!/bin/bash
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/r02zy_gpu_pytest.txt 2>&1; tail -2 gpurun_out/r02zy_gpu_pytest.txt
for c in longformer bigbird sparse_transformer; do timeout -s KILL 300 python tools/shard_sim.py $c; done > gpurun_out/r02zy_shard_sim.jsonl; cat gpurun_out/r02zy_shard_sim.jsonl
