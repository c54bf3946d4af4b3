#!/bin/bash
# Session-3 checkpoint on the committed code: full GPU suite, all bench lines, launch list, ncu --set full
# summaries of the fused kernels and the unfused primitives, unfused timings.
TAG=r02zz6
mkdir -p gpurun_out
python -m paper_2407_16847_b200.build > gpurun_out/${TAG}_build.log 2>&1 || { tail gpurun_out/${TAG}_build.log; exit 1; }
timeout -s KILL 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_gpu_pytest.txt 2>&1
tail -2 gpurun_out/${TAG}_gpu_pytest.txt
timeout -s KILL 600 python bench.py > gpurun_out/${TAG}_bench_longformer.json 2> gpurun_out/${TAG}_bench_longformer.err
python -c "import json; d=json.loads(open('gpurun_out/${TAG}_bench_longformer.json').read().splitlines()[-1]); print('longformer', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks'])"
for c in bigbird sparse_transformer mistral tiny; do
  timeout -s KILL 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/${TAG}_bench_$c.json').read().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d['roofline']['frac'])"
done
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_longformer_launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for c in longformer bigbird mistral; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"mhsa_(split|tc)" -s 3 -c 1 \
      -o gpurun_out/${TAG}_prof_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"mhsa_tc" -s 6 -c 2 \
    -o gpurun_out/${TAG}_prof_sparse_transformer python bench.py --config sparse_transformer --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for k in rsddmm softmax rspmm; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
      -o gpurun_out/${TAG}_prof_unf_$k python tools/bench_unfused.py --configs longformer --iters 2 > /dev/null 2>&1
done
timeout -s KILL 600 python tools/bench_unfused.py --configs longformer,bigbird,sparse_transformer --iters 10 > gpurun_out/${TAG}_unfused.jsonl 2>&1
ls gpurun_out | grep ${TAG} | wc -l
for c in longformer bigbird sparse_transformer; do timeout -s KILL 300 python tools/shard_sim.py $c; done > gpurun_out/${TAG}_shard_sim.jsonl
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_headline_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-per-config > /dev/null 2>&1
