python -m paper_2407_16847_b200.build > /dev/null 2>&1
timeout 300 compute-sanitizer --tool memcheck --print-limit 3 python tools/spmm_case.py longformer 3 2>&1 | tail -3
timeout 300 compute-sanitizer --tool memcheck --print-limit 3 python tools/spmm_case.py bigbird 2 2>&1 | tail -2
bash tools/r02f.sh
