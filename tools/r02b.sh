# sanitizer pass + NEMU sweep + split-kernel trace (Longformer)
python -m paper_2407_16847_b200.build > /dev/null 2>&1
TAG=r02b bash tools/sanitize_all.sh
VARIANTS="-DSPLAT_NEMU=4|-DSPLAT_NEMU=8|-DSPLAT_NEMU=12|-DSPLAT_NEMU=16|-DSPLAT_NEMU=20" CONFIGS="longformer bigbird" bash tools/sweep_diag.sh 2>&1 | tee gpurun_out/r02b_nemu.txt
TRACE_CONFIGS=longformer bash tools/trace_run.sh
tail -40 gpurun_out/trace_longformer_report.txt
