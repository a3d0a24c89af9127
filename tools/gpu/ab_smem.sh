for cfg in c2 c3 c4; do
for v in "" "CPDB_TTM_SMEM_EXACT=1"; do
  echo "=== $cfg $v"
  env $v python bench.py --config $cfg --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['breakdown_ms_per_step'])"
done
done
