#!/bin/bash
# timing of the fused kernel under debug modes: 1 = no MMAs, 2 = no softmax math, 16 = no K/V TMA
python -m paper_2407_16847_b200.build > /dev/null
for d in ${MODES:-0 1 2 3 16 19}; do
  r=$(SPLAT_TC_DEBUG=$d timeout 60 python bench.py --config ${CFG:-longformer} --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,1),'us')")
  echo "dbg=$d $r"
done
