timeout 600 python -m pytest tests/test_gpu_solver.py -q -x -p no:cacheprovider -k "c5_proxy or tall_z or rank_edges or q0_structure or ill_cond" -o faulthandler_timeout=120 > gpurun_out/p37_tests.log 2>&1; echo tests rc=$?
tail -1 gpurun_out/p37_tests.log
timeout 300 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p37.json 2> gpurun_out/p37.err
echo "c5 rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p37.json')); print(round(d['value'],2))" 2>/dev/null)"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"zqr|vgemm" --launch-skip 10 --launch-count 30 --csv python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/p37_ncu.csv 2> gpurun_out/p37_ncu.err; echo ncu rc=$?
python tools/launch_summary.py gpurun_out/p37_ncu.csv 2>&1 | head -9
