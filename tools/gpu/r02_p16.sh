for v in "CPDB_TAIL_SMS=80" "CPDB_TAIL_SMS=0" "CPDB_TAIL_SMS=40" "CPDB_TAIL_SMS=80" "CPDB_LOW_TAIL=0"; do
  env $v timeout 120 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p16.json 2> gpurun_out/p16.err
  echo "$v rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p16.json')); print(round(d['value'],1))" 2>/dev/null)"
done
timeout 120 python tools/timeline.py c2 --warmup 6 --sweeps 3 > gpurun_out/tl_c2_g.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_solver.py tests/test_gpu_determinism.py -q -x -p no:cacheprovider -o faulthandler_timeout=120 -k "not full_length" > gpurun_out/p16_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/p16_tests.log
