python -m paper_2407_16847_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "residue or sparse_transformer or strided" > gpurun_out/r02ac_pytest.txt 2>&1; tail -1 gpurun_out/r02ac_pytest.txt
for i in 1 2; do timeout 120 python tools/time_fused.py sparse_transformer 20; done
timeout 120 python tools/time_fused.py mistral 5
