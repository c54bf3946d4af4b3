python -m paper_2407_16847_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "fused or uniform or stress or deterministic or bf16 or full_config or d64" > gpurun_out/r02o_pytest.txt 2>&1; tail -2 gpurun_out/r02o_pytest.txt
for c in longformer bigbird mistral; do timeout 120 python tools/time_fused.py $c 20; done
