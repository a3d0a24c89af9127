timeout 600 python -m pytest tests/test_gpu_solver.py -q -x -p no:cacheprovider -k "c5_proxy or tall_z or rank_edges or q0_structure or breakdown or stop_test" -o faulthandler_timeout=120 > gpurun_out/p14_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/p14_tests.log
for cfg in c5 c2; do
  timeout 300 python bench.py --config $cfg --steps 50 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p14.json 2> gpurun_out/p14.err
  echo "$cfg rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p14.json')); print(round(d['value'],2))" 2>/dev/null)"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip 150 --launch-count 120 --csv python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p14_ncu.csv 2> gpurun_out/p14_ncu.err; echo ncu rc=$?
python tools/launch_summary.py gpurun_out/p14_ncu.csv 2>&1 | head -16
