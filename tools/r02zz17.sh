#!/bin/bash
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -k "split_k" 2>&1 | tail -2
