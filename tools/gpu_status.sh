set -x
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv
ls MEASURED_PEAKS.json
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
for c in longformer bigbird sparse_transformer mistral; do timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 > gpurun_out/bench_$c.json; cat gpurun_out/bench_$c.json | cut -c1-400; done
timeout 600 python tools/bench_unfused.py 2>&1 | tail -5 | tee gpurun_out/unfused.log
