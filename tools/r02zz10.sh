#!/bin/bash
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests -m gpu -q > gpurun_out/r02zz10_gpu_pytest.txt 2>&1; tail -1 gpurun_out/r02zz10_gpu_pytest.txt
