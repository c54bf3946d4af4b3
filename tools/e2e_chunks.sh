python -m paper_2407_16847_b200.build > /dev/null
for c in 4 8 12 15; do
  for cfg in longformer mistral; do
    r=$(SPLAT_HOST_CHUNKS=$c timeout 120 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['e2e']['value'],2), round(d['e2e']['ms_per_step'],3))")
    echo "chunks=$c $cfg e2e $r"
  done
done
