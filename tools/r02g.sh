python -m paper_2407_16847_b200.build --diag > /dev/null 2>&1
SPLAT_LIB=diag SPLAT_TC_PAIRED64=3 timeout 600 python tools/check_fused.py
for c in longformer bigbird; do SPLAT_LIB=diag SPLAT_TC_PAIRED64=3 TAGV=halfrow2g timeout 120 python tools/time_fused.py $c 20; SPLAT_LIB=diag TAGV=split timeout 120 python tools/time_fused.py $c 20; done
