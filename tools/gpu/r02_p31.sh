timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -o faulthandler_timeout=200 -k "not full_length" > gpurun_out/p31_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/p31_tests.log
for cfg in c2 c2 c2 c4 c1 c3; do
  timeout 120 python bench.py --config $cfg --steps 300 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p31.json 2> gpurun_out/p31.err
  echo "$cfg rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p31.json')); print(round(d['value'],1))" 2>/dev/null)"
done
CPDB_PHASE_TRACE=1 timeout 120 python tools/phase_trace.py c2 2> gpurun_out/phase_c2_c.txt > /dev/null; tail -2 gpurun_out/phase_c2_c.txt
timeout 600 python tools/det_probe.py c3 40 4 2>&1 | tail -1
