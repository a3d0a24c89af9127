for i in 1 2 3; do
  timeout 120 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p24.json 2> gpurun_out/p24.err
  echo "c2 rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p24.json')); print(round(d['value'],1))" 2>/dev/null)"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:vgemm --launch-skip 40 --launch-count 20 --csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p24_ncu.csv 2> gpurun_out/p24_ncu.err
python tools/launch_summary.py gpurun_out/p24_ncu.csv 2>&1 | head -5
