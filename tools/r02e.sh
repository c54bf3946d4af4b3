python -m paper_2407_16847_b200.build > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k "boundary or coverage" > gpurun_out/r02e_pytest_new.txt 2>&1
tail -15 gpurun_out/r02e_pytest_new.txt
timeout 600 python bench.py > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err
tail -c 3000 gpurun_out/r02e_bench.json; tail -5 gpurun_out/r02e_bench.err
