for v in "CPDB_TAIL_SMS=0" "CPDB_TAIL_SMS=40" "CPDB_TAIL_SMS=24" "CPDB_TAIL_SMS=64" "CPDB_TAIL_SMS=40"; do
  env $v timeout 120 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p9.json 2> gpurun_out/p9.err
  echo "$v rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p9.json')); print(round(d['value'],1))" 2>/dev/null)"
done
timeout 120 python tools/timeline.py c2 --warmup 6 --sweeps 3 > gpurun_out/tl_c2_f.txt 2>&1
