# A/B of session switches on the bench (C2 unless CFG given)
CFG=${CFG:-c2}
for v in "$@"; do
  env $v python bench.py --config $CFG --steps 100 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],1), 'root_ovl_ms', round(d['roofline']['overlapped_avg_launch_ms'],4), d['kernel_ms_per_step'])"
done
