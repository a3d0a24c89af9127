mkdir -p gpurun_out/ev7
for cfg in c2 c1 c3 c4; do
  timeout 600 python bench.py --config $cfg > gpurun_out/ev7/bench_$cfg.json 2> gpurun_out/ev7/bench_$cfg.err; echo "$cfg rc=$?"
done
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/ev7/bench_c2_k20.json 2> gpurun_out/ev7/bench_c2_k20.err; echo "c2 k20 rc=$?"
timeout 600 python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/ev7/bench_c5.json 2> gpurun_out/ev7/bench_c5.err; echo "c5 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ev7/launches_c2.csv 2> gpurun_out/ev7/launches_c2.err; echo "launch c2 rc=$?"
for f in gpurun_out/ev7/bench_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); print(d.get('value'), d.get('e2e',{}) and d['e2e'].get('value'), d.get('roofline',{}) and d['roofline'].get('frac'), d.get('clocks'))"; done
