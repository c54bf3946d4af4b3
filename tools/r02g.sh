python -m paper_2407_16847_b200.build > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rspmm -s 2 -c 1 -o gpurun_out/r02g_rspmm python tools/bench_unfused.py --configs longformer --iters 2 > gpurun_out/r02g_rspmm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mhsa_split -s 3 -c 1 -o gpurun_out/r02g_split python bench.py --config longformer --steps 1 --warmup 3 --no-cpu-baseline --no-per-config > gpurun_out/r02g_split.log 2>&1
ls -la gpurun_out/*.ncu-rep
