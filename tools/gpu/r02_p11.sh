timeout 600 python -m pytest tests/test_gpu_solver.py -q -x -p no:cacheprovider -k "c5_proxy or tall_z or rank_edges or q0_structure" -o faulthandler_timeout=120 > gpurun_out/p11_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/p11_tests.log
for v in "CPDB_ZQR_GEMM=0" "CPDB_ZQR_GEMM=1"; do
  env $v timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p11.json 2> gpurun_out/p11.err
  echo "$v rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p11.json')); print(round(d['value'],2), d['kernel_ms_per_step'])" 2>/dev/null)"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:zqr --launch-skip 20 --launch-count 24 --csv python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p11_ncu.csv 2> gpurun_out/p11_ncu.err; echo ncu rc=$?
python tools/launch_summary.py gpurun_out/p11_ncu.csv 2>&1 | head -12
