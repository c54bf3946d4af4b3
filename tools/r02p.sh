python -m paper_2407_16847_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_layout.py -q -x > gpurun_out/r02p_pytest.txt 2>&1; tail -3 gpurun_out/r02p_pytest.txt
timeout 900 python tools/layout_grid.py --iters 10 --out gpurun_out/r02p_layout_grid.json 2>&1 | tail -22
