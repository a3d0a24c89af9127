mkdir -p gpurun_out/ev2
for cfg in c2 c1 c3 c4; do
  timeout 600 python bench.py --config $cfg > gpurun_out/ev2/bench_$cfg.json 2> gpurun_out/ev2/bench_$cfg.err; echo "$cfg rc=$?"
done
timeout 600 python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/ev2/bench_c5.json 2> gpurun_out/ev2/bench_c5.err; echo "c5 rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev2/bench_ref_c2.json 2> gpurun_out/ev2/bench_ref_c2.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ev2/launches_c2.csv 2> gpurun_out/ev2/launches_c2.err; echo "launch c2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev2/launches_c5.csv 2> gpurun_out/ev2/launches_c5.err; echo "launch c5 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ttm_tma_kernel --launch-skip 40 --launch-count 4 -o gpurun_out/ev2/ttm_c2 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev2/ncu_ttm.log 2>&1; echo "ncu ttm rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"vgemm_wide|zqr_rows_gemm|zqr_apply_gemm" --launch-skip 4 --launch-count 4 -o gpurun_out/ev2/c5_tail -f python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev2/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
timeout 900 python tools/det_probe.py c3 90 4 > gpurun_out/ev2/det_c3.txt 2>&1; echo "det rc=$?"; tail -1 gpurun_out/ev2/det_c3.txt
for f in gpurun_out/ev2/bench_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); print(d.get('value'), d.get('e2e',{}) and d['e2e'].get('value'), d.get('roofline',{}) and d['roofline'].get('frac'), d.get('clocks'))"; done
