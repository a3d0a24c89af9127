python -m pytest tests/test_gpu_synth_io.py -q -x -p no:cacheprovider 2>&1 | tail -15
python tools/parity_floor.py --out gpurun_out/parity_floor.jsonl > /dev/null 2> gpurun_out/parity_floor.err; echo floor rc=$?
cat gpurun_out/parity_floor.jsonl
nproc; lscpu | grep "Model name"
