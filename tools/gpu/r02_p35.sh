for v in 0 1 2 3; do
  CPDB_TTM_ROOTCFG=$v timeout 120 python bench.py --config c2 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p35.json 2> gpurun_out/p35.err
  echo "c2 cfg=$v rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p35.json')); r=d['roofline']; print(round(d['value'],1), round(r['avg_launch_ms']*1e3,1), round(r['frac'],4), round(r['overlapped_avg_launch_ms']*1e3,1))" 2>/dev/null)"
done
for v in 0 1; do
  CPDB_TTM_ROOTCFG=$v timeout 120 python bench.py --config c3 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p35.json 2> gpurun_out/p35.err
  echo "c3 cfg=$v rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p35.json')); r=d['roofline']; print(round(d['value'],1), round(r['avg_launch_ms']*1e3,1), round(r['frac'],4), round(r['overlapped_avg_launch_ms']*1e3,1))" 2>/dev/null)"
done
timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p35.json 2> gpurun_out/p35.err
echo "c5 rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p35.json')); r=d['roofline']; print(round(d['value'],2), round(r['avg_launch_ms']*1e3,1), round(r['frac'],4))" 2>/dev/null)"
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_prims.py tests/test_gpu_sharded.py -q -x -p no:cacheprovider -o faulthandler_timeout=200 -k "not full_length" > gpurun_out/p35_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/p35_tests.log
