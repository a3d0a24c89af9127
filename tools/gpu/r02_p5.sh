python -m pytest tests/test_gpu_solver.py tests/test_gpu_determinism.py tests/test_gpu_sharded.py tests/test_gpu_prims.py -q -x -p no:cacheprovider 2>&1 | tail -3
bash tools/gpu/r02_ab.sh CPDB_LOW_TAIL=0 CPDB_LOW_TAIL=1 CPDB_TTM_NC7=0 CPDB_SELF_HIST=0 CPDB_LOW_TAIL=1
CFG=c4 bash tools/gpu/r02_ab.sh CPDB_LOW_TAIL=0 CPDB_LOW_TAIL=1
CFG=c3 bash tools/gpu/r02_ab.sh CPDB_LOW_TAIL=0 CPDB_LOW_TAIL=1
python tools/timeline.py c2 --warmup 6 --sweeps 2 > gpurun_out/tl_c2_c.txt 2>&1
python tools/det_probe.py c3 20 4 2>&1 | tail -2
