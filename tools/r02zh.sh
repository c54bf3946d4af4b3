#!/bin/bash
# A/B: paired-kernel residue path -- HEAD (ctrl), current (VM template + 8 maps), current with plain O_s / lse loads (ctrl2)
for i in 1 2; do
(cd ctrl && timeout -s KILL 120 python tools/time_fused.py sparse_transformer 30 | sed 's/^/ctrl  /')
timeout -s KILL 120 python tools/time_fused.py sparse_transformer 30 | sed 's/^/cur   /'
(cd ctrl2 && timeout -s KILL 120 python tools/time_fused.py sparse_transformer 30 | sed 's/^/ctrl2 /')
done
(cd ctrl && timeout -s KILL 120 python tools/time_fused.py mistral 5 | sed 's/^/ctrl  /')
timeout -s KILL 120 python tools/time_fused.py mistral 5 | sed 's/^/cur   /'
