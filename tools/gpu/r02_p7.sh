timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider -o faulthandler_timeout=120 > gpurun_out/p7_tests.log 2>&1; echo tests rc=$?
tail -4 gpurun_out/p7_tests.log
for v in "CPDB_LOW_TAIL=0 CPDB_TTM_NC7=0" "CPDB_LOW_TAIL=1 CPDB_TTM_NC7=0" "CPDB_LOW_TAIL=1" "CPDB_LOW_TAIL=1 CPDB_TTM_NC7=0" "CPDB_LOW_TAIL=1"; do
  env $v timeout 120 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p7.json 2> gpurun_out/p7.err
  echo "$v rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p7.json')); print(round(d['value'],1))" 2>/dev/null)"
done
for cfg in c3 c4 c1; do for v in "CPDB_LOW_TAIL=0" "CPDB_LOW_TAIL=1"; do
  env $v timeout 120 python bench.py --config $cfg --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p7.json 2> gpurun_out/p7.err
  echo "$cfg $v rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p7.json')); print(round(d['value'],1))" 2>/dev/null)"
done; done
timeout 120 python tools/timeline.py c2 --warmup 6 --sweeps 2 > gpurun_out/tl_c2_d.txt 2>&1
