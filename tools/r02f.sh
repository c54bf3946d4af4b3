python -m paper_2407_16847_b200.build > /dev/null 2>&1
timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_case.py n512_d64 > gpurun_out/r02f_race.txt 2>&1; grep -E "SUMMARY|Error" gpurun_out/r02f_race.txt | head -5
timeout 900 python -m pytest tests -m gpu -q -x -k "fused or boundary or smoke or uniform or deterministic" > gpurun_out/r02f_pytest.txt 2>&1; tail -2 gpurun_out/r02f_pytest.txt
VARIANTS="-DSPLAT_NEMU=0|-DSPLAT_NEMU=4|-DSPLAT_NEMU=8|-DSPLAT_NEMU=12" CONFIGS="longformer bigbird" bash tools/sweep_diag.sh
