# micro: TS/SS MMA rate with TMEM ld/st contention; new R-SpMM + tiny kernel parity + unfused timings


python -m paper_2407_16847_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "unfused or tiny or paper_grid or bf16 or residue or spmm or fp32" > gpurun_out/r02c_pytest.txt 2>&1; tail -3 gpurun_out/r02c_pytest.txt
timeout 600 python tools/bench_unfused.py --configs longformer,bigbird,sparse_transformer --iters 10 > gpurun_out/r02c_unfused.jsonl 2>&1; cat gpurun_out/r02c_unfused.jsonl | cut -c1-1500
timeout 300 python bench.py --config tiny --steps 50 --warmup 5 --no-cpu-baseline --no-per-config > gpurun_out/r02c_tiny.json 2>&1; tail -c 600 gpurun_out/r02c_tiny.json
