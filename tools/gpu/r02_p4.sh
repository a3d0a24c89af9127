python -m pytest tests/test_gpu_solver.py tests/test_gpu_determinism.py tests/test_gpu_sharded.py -q -x -p no:cacheprovider 2>&1 | tail -3
bash tools/gpu/r02_ab.sh CPDB_SELF_HIST=0 CPDB_SELF_HIST=1 CPDB_TIME_TAILS=0 CPDB_SELF_HIST=0
python tools/timeline.py c2 --warmup 6 --sweeps 2 > gpurun_out/tl_c2_b.txt 2>&1
