python -m paper_2407_16847_b200.build > /dev/null 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 -k "fused or bigbird or d64 or uniform or stress or deterministic or host_path or edge or small" > gpurun_out/r02aa_pytest.txt 2>&1; tail -1 gpurun_out/r02aa_pytest.txt
for c in bigbird longformer; do timeout 120 python tools/time_fused.py $c 20; done
