# d = 64 split kernel variant: parity subset + timing
python -m paper_2407_16847_b200.build > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "fused and not mistral" > gpurun_out/r02ae_pytest.txt 2>&1; tail -1 gpurun_out/r02ae_pytest.txt
for c in longformer bigbird longformer bigbird; do timeout 120 python tools/time_fused.py $c 30; done
