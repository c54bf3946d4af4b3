python -m paper_2407_16847_b200.build > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rspmm -s 2 -c 1 -o gpurun_out/r02i_rspmm python tools/bench_unfused.py --configs longformer --iters 2 > gpurun_out/r02i_rspmm.log 2>&1
ls gpurun_out/r02i_rspmm.ncu-rep
