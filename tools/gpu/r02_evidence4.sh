python -m pytest tests -m gpu -x -q > gpurun_out/gputest_v4.log 2>&1; tail -2 gpurun_out/gputest_v4.log
mkdir -p gpurun_out/ev4
for cfg in c2 c1 c3 c4; do
  timeout 600 python bench.py --config $cfg > gpurun_out/ev4/bench_$cfg.json 2> gpurun_out/ev4/bench_$cfg.err; echo "$cfg rc=$?"
done
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/ev4/bench_c2_k20.json 2> gpurun_out/ev4/bench_c2_k20.err; echo "c2 k20 rc=$?"
timeout 600 python bench.py --config c5 --steps 20 --warmup 3 > gpurun_out/ev4/bench_c5.json 2> gpurun_out/ev4/bench_c5.err; echo "c5 rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev4/bench_ref_c2.json 2> gpurun_out/ev4/bench_ref_c2.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ev4/launches_c2.csv 2> gpurun_out/ev4/launches_c2.err; echo "launch c2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev4/launches_c5.csv 2> gpurun_out/ev4/launches_c5.err; echo "launch c5 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ttm_tma_kernel --launch-skip 40 --launch-count 4 -o gpurun_out/ev4/ttm_c2 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ev4/ncu_ttm.log 2>&1; echo "ncu ttm rc=$?"
timeout 600 python tools/wide_rank_probe.py 192x192x192 128 6 2 > gpurun_out/ev4/wide_rank.json 2> gpurun_out/ev4/wide_rank.err; echo "wide rc=$?"; cat gpurun_out/ev4/wide_rank.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:hh_coop_kernel --launch-skip 3 --launch-count 2 -o gpurun_out/ev4/hh_wide -f python tools/wide_rank_probe.py 128x128x128 96 3 0 > gpurun_out/ev4/ncu_hh.log 2>&1; echo "ncu hh rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv python tools/wide_rank_probe.py 192x192x192 128 3 0 > gpurun_out/ev4/launches_wide.csv 2> gpurun_out/ev4/launches_wide.err; echo "launch wide rc=$?"
timeout 900 python tools/det_probe.py c3 90 12 > gpurun_out/ev4/det_c3.txt 2>&1; echo "det rc=$?"; tail -1 gpurun_out/ev4/det_c3.txt
for f in gpurun_out/ev4/bench_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); print(d.get('value'), d.get('e2e',{}) and d['e2e'].get('value'), d.get('roofline',{}) and d['roofline'].get('frac'), d.get('clocks'))"; done
