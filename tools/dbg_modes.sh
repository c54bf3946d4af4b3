#!/bin/bash
# timing of the fused kernel under debug modes (1 = no MMAs, 2 = no softmax math) and build flags
for fl in "" "-DSPLAT_SPIN" "-DSPLAT_WAIT_HINT=20" "-DSPLAT_WAIT_HINT=200"; do
  SPLAT_EXTRA_NVCC_FLAGS="$fl" python -m paper_2407_16847_b200.build --force > /dev/null
  for d in 0 3; do
    r=$(SPLAT_TC_DEBUG=$d timeout 60 python bench.py --config ${CFG:-longformer} --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,1),'us')")
    echo "flags='$fl' dbg=$d $r"
  done
done
