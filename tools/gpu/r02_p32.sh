for cfg in c2 c3; do for v in "CPDB_TTM_NC16=0" "CPDB_TTM_NC16=1" "CPDB_TTM_NC16=0" "CPDB_TTM_NC16=1"; do
  env $v timeout 120 python bench.py --config $cfg --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p32.json 2> gpurun_out/p32.err
  echo "$cfg $v rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p32.json')); r=d['roofline']; print(round(d['value'],1), round(r['avg_launch_ms']*1e3,1), round(r['frac'],4), round(r['overlapped_avg_launch_ms']*1e3,1))" 2>/dev/null)"
done; done
for v in "CPDB_TTM_NC16=0" "CPDB_TTM_NC16=1"; do
  env $v timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p32.json 2> gpurun_out/p32.err
  echo "c5 $v rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p32.json')); r=d['roofline']; print(round(d['value'],2), round(r['avg_launch_ms']*1e3,1), round(r['frac'],4))" 2>/dev/null)"
done
