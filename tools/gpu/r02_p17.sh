for v in "CPDB_SPEC_STREAM=aux" "CPDB_SPEC_STREAM=mid" "CPDB_SPEC_STREAM=aux" "CPDB_SPEC_STREAM=mid"; do
  env $v timeout 120 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p17.json 2> gpurun_out/p17.err
  echo "$v rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p17.json')); print(round(d['value'],1))" 2>/dev/null)"
done
for cfg in c4 c1; do for v in "CPDB_SPEC_STREAM=aux" "CPDB_SPEC_STREAM=mid"; do
  env $v timeout 120 python bench.py --config $cfg --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p17.json 2> gpurun_out/p17.err
  echo "$cfg $v rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p17.json')); print(round(d['value'],1))" 2>/dev/null)"
done; done
CPDB_SPEC_STREAM=mid timeout 120 python tools/timeline.py c2 --warmup 6 --sweeps 3 > gpurun_out/tl_c2_h.txt 2>&1
