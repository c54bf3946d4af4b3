#!/bin/bash
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for i in 1 2; do for c in longformer bigbird; do
 (cd ctrl && timeout -s KILL 120 python tools/time_fused.py $c 30 | sed 's/^/ctrl /')
 timeout -s KILL 120 python tools/time_fused.py $c 30 | sed 's/^/cur  /'
done; done
for c in longformer bigbird; do timeout -s KILL 300 python tools/shard_sim.py $c; done
