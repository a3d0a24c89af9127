for v in "CPDB_LOW_TAIL=0 CPDB_TTM_NC7=0" "CPDB_LOW_TAIL=0" "CPDB_LOW_TAIL=1 CPDB_TTM_NC7=0" "CPDB_LOW_TAIL=1"; do
  env $v timeout 120 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p6.json 2> gpurun_out/p6.err
  echo "$v rc=$?"; python -c "import json; d=json.load(open('gpurun_out/p6.json')); print(round(d['value'],1))" 2>/dev/null
done
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_sharded.py tests/test_gpu_determinism.py -x -v -p no:cacheprovider -o faulthandler_timeout=90 > gpurun_out/p6_tests.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/p6_tests.log
