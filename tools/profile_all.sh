#!/bin/bash
# Round profile pass (GPU box): bench lines for every config (default one with the CPU
# baseline), the launch list of the default bench command, and one ncu --set full capture of the
# fused kernel(s) per config.  Outputs under gpurun_out/ (summarised into profiles/ by hand).
TAG=${TAG:-r01b}
python -m paper_2407_16847_b200.build > /dev/null
timeout 600 python bench.py > gpurun_out/${TAG}_bench_longformer.json 2> gpurun_out/${TAG}_bench_longformer.err
for c in bigbird sparse_transformer mistral tiny; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2>/dev/null
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for c in longformer bigbird mistral; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mhsa_(split|tc)" -s 3 -c 1 \
      -o gpurun_out/${TAG}_prof_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mhsa_tc" -s 6 -c 2 \
    -o gpurun_out/${TAG}_prof_sparse_transformer python bench.py --config sparse_transformer --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out | tail -20
# unfused primitives (Longformer): one ncu --set full capture each, and their timings
for k in rsddmm softmax rspmm; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/${TAG}_prof_unf_$k python tools/bench_unfused.py --configs longformer --iters 2 > /dev/null 2>&1
done
timeout 600 python tools/bench_unfused.py --configs longformer,bigbird,sparse_transformer --iters 10 > gpurun_out/${TAG}_unfused.jsonl 2>&1
