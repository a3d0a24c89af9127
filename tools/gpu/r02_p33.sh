for cfg in c2 c4 c1; do for v in "CPDB_TTM_NC16=1" "CPDB_TTM_NC16=2" "CPDB_TTM_NC16=1" "CPDB_TTM_NC16=2"; do
  env $v timeout 120 python bench.py --config $cfg --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p33.json 2> gpurun_out/p33.err
  echo "$cfg $v rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p33.json')); r=d['roofline']; print(round(d['value'],1), round(r['frac'],4), d['kernel_ms_per_step']['branch_ttm'])" 2>/dev/null)"
done; done
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -o faulthandler_timeout=200 -k "not full_length" > gpurun_out/p33_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/p33_tests.log
