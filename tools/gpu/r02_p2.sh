python -m pytest tests/test_gpu_synth_io.py tests/test_gpu_solver.py tests/test_gpu_sharded.py -q -x -p no:cacheprovider --durations=8 2>&1 | tail -15
python tools/parity_floor.py --als-only --out gpurun_out/parity_floor_als.jsonl > /dev/null 2> gpurun_out/parity_floor_als.err; echo floor rc=$?
cat gpurun_out/parity_floor_als.jsonl
