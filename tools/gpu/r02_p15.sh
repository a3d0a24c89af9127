timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -o faulthandler_timeout=150 --durations=5 -rA -k "not full_length" > gpurun_out/p15_tests.log 2>&1; echo tests rc=$?
grep -E "passed|failed|fitness gap" gpurun_out/p15_tests.log | tail -8
timeout 120 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p15.json 2> gpurun_out/p15.err; echo "c2 $(python -c "import json; d=json.load(open('gpurun_out/p15.json')); print(round(d['value'],1))")"
