python -m paper_2407_16847_b200.build > /dev/null 2>&1
timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python tools/sanitize_case.py n512_d64 2>&1 | head -60
timeout 300 python -m pytest tests -m gpu -q -x -k "test_bf16_fused_and_unfused_small" 2>&1 | tail -15
