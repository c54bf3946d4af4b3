#!/bin/bash
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests -m gpu -q -x > gpurun_out/r02zv_pytest.txt 2>&1
grep -n "Fatal\|Error\|error\|FAIL\|passed\|failed" gpurun_out/r02zv_pytest.txt | head -20
tail -40 gpurun_out/r02zv_pytest.txt | head -30
