#!/bin/bash
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout -s KILL 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-per-config 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print(round(d['value'],1), d['e2e'])"
