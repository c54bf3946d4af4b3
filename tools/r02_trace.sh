set -x
TRACE_CONFIGS=longformer bash tools/trace_run.sh
SPLAT_EXTRA_NVCC_FLAGS=-DSPLAT_FUSED_PROF python -m paper_2407_16847_b200.build --diag > /dev/null
python tools/fused_prof.py longformer > gpurun_out/r02_fprof_longformer.txt 2>&1
python -m paper_2407_16847_b200.build --diag > /dev/null
python bench.py --no-cpu-baseline > gpurun_out/r02_base_lf.json 2>gpurun_out/r02_base_lf.err
python bench.py --config bigbird --no-cpu-baseline > gpurun_out/r02_base_bb.json 2>&1
