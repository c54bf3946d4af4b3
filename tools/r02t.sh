python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1
for p in 37 40; do SPLAT_LIB=diag SPLAT_RESIDUE_G1_PCT=$p TAGV=g1=$p timeout 120 python tools/time_fused.py sparse_transformer 20; done
SPLAT_LIB=diag SPLAT_RESIDUE_G1_PCT=37 timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:mhsa --csv python tools/time_fused.py sparse_transformer 1 2>/dev/null | grep -v "^==" | awk -F'","' '{print $1, $(NF-2), $NF}' | tail -6
SPLAT_LIB=diag SPLAT_RESIDUE_TWO_LAUNCH=1 timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:mhsa --csv python tools/time_fused.py sparse_transformer 1 2>/dev/null | grep -v "^==" | awk -F'","' '{print $1, $(NF-2), $NF}' | tail -6
