python -m paper_2407_16847_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "residue or sparse_transformer or strided or full_config or deterministic or host_path" > gpurun_out/r02v_pytest.txt 2>&1; tail -2 gpurun_out/r02v_pytest.txt
timeout 120 python tools/time_fused.py sparse_transformer 20
python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1
SPLAT_LIB=diag SPLAT_RESIDUE_MODE=2 TAGV=two-launch timeout 120 python tools/time_fused.py sparse_transformer 20
for p in 25 30 35 40 45; do SPLAT_LIB=diag SPLAT_RESIDUE_MODE=1 SPLAT_RESIDUE_G1_PCT=$p TAGV=g1=$p timeout 120 python tools/time_fused.py sparse_transformer 20; done
