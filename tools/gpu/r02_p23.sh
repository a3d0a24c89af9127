timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider -o faulthandler_timeout=150 -k "not full_length" > gpurun_out/p23_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/p23_tests.log
for cfg in c5 c2 c2 c4 c3; do
  timeout 300 python bench.py --config $cfg --steps 100 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p23.json 2> gpurun_out/p23.err
  echo "$cfg rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p23.json')); print(round(d['value'],2))" 2>/dev/null)"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:vgemm --launch-skip 4 --launch-count 8 --csv python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p23_ncu.csv 2> gpurun_out/p23_ncu.err; echo ncu rc=$?
python tools/launch_summary.py gpurun_out/p23_ncu.csv 2>&1 | head -4
