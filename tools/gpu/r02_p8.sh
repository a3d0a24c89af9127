timeout 1300 python -m pytest tests -m gpu -q -p no:cacheprovider -o faulthandler_timeout=150 --durations=5 > gpurun_out/p8_tests.log 2>&1; echo tests rc=$?
tail -12 gpurun_out/p8_tests.log
for cfg in c2 c4; do
  timeout 120 python bench.py --config $cfg --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p8.json 2> gpurun_out/p8.err
  echo "$cfg rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p8.json')); print(round(d['value'],1))" 2>/dev/null)"
done
timeout 120 python tools/timeline.py c2 --warmup 6 --sweeps 2 > gpurun_out/tl_c2_e.txt 2>&1
