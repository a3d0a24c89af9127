NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT timeout 300 python -m pytest tests/test_gpu_sharded.py -q -x -s -p no:cacheprovider -k "nccl" > gpurun_out/p30.log 2>&1; echo rc=$?
grep -E "passed|failed|NCCL INFO (Init|comm|NCCL version)" gpurun_out/p30.log | head -12
