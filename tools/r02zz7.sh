#!/bin/bash
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 2>/dev/null | tail -1 | cut -c1-400
