SPLAT_EXTRA_NVCC_FLAGS=-DSPLAT_TRACE python -m paper_2407_16847_b200.build --diag > /dev/null
for c in ${TRACE_CONFIGS:-longformer mistral}; do
python tools/trace.py $c > gpurun_out/trace_$c.txt 2>&1
python tools/trace_report.py gpurun_out/trace_$c.txt > gpurun_out/trace_${c}_report.txt 2>&1; python tools/trace_tma.py gpurun_out/trace_$c.txt >> gpurun_out/trace_${c}_report.txt 2>&1
done
