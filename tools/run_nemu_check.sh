bash tools/quick_check.sh
for n in 0 4 12; do
  SPLAT_EXTRA_NVCC_FLAGS="-DSPLAT_NEMU=$n" python -m paper_2407_16847_b200.build --force >/dev/null 2>&1
  for c in longformer bigbird; do
    r=$(timeout 60 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],4))")
    echo "NEMU=$n $c $r"
  done
done
python -m paper_2407_16847_b200.build --force >/dev/null 2>&1
