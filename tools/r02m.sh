python -m paper_2407_16847_b200.build > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rsddmm -s 1 -c 1 -o gpurun_out/r02m_rsddmm python tools/bench_unfused.py --configs longformer --iters 2 > gpurun_out/r02m_rsddmm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:softmax -s 1 -c 1 -o gpurun_out/r02m_softmax python tools/bench_unfused.py --configs longformer --iters 2 > gpurun_out/r02m_softmax.log 2>&1
ls gpurun_out/r02m*
