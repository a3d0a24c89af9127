# round-2 baseline: GPU suite, smoke, C2 bench, launch list
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/gputest.log 2>&1; echo tests rc=$?
tail -25 gpurun_out/gputest.log
python bench.py --steps 100 --warmup 5 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench rc=$?
cat gpurun_out/bench_c2.json
