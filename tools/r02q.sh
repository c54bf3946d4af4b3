python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1
SPLAT_LIB=diag timeout 900 python tools/align_ablation.py --out gpurun_out/r02q_align_ablation.json 2>&1 | tail -12
SPLAT_LIB=diag timeout 900 ncu --metrics smsp__sass_inst_executed_op_global_ld.sum,smsp__sass_thread_inst_executed_op_global_ld.sum -k regex:rspmm_cc --csv --log-file gpurun_out/r02q_align_ncu.csv python tools/align_ablation.py --iters 1 --out /tmp/x.json > /dev/null 2>&1
wc -l gpurun_out/r02q_align_ncu.csv
