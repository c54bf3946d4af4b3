#!/bin/bash
# GPU box: full build + -m gpu suite + default bench line (with per_config) + sanitizer.
TAG=${TAG:-r02a}
mkdir -p gpurun_out
python -m paper_2407_16847_b200.build > gpurun_out/${TAG}_build.log 2>&1 || { tail -20 gpurun_out/${TAG}_build.log; exit 1; }
timeout 1800 python -m pytest tests -m gpu -q -rs > gpurun_out/${TAG}_pytest.txt 2>&1
tail -8 gpurun_out/${TAG}_pytest.txt
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
tail -c 4000 gpurun_out/${TAG}_bench.json; tail -3 gpurun_out/${TAG}_bench.err
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.txt 2>&1; tail -2 gpurun_out/${TAG}_smoke.txt
