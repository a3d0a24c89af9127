timeout 1200 python -m pytest tests/test_gpu_sharded.py -q -x -p no:cacheprovider -o faulthandler_timeout=200 > gpurun_out/p26_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/p26_tests.log
CPDB_HBCHECK=1 timeout 1200 python -m pytest tests/test_gpu_sharded.py -q -x -s -p no:cacheprovider -k "matches_unsharded and (bre or dim)" -o faulthandler_timeout=200 > gpurun_out/p26_hb.log 2>&1; echo hb rc=$?
grep -c "hbcheck" gpurun_out/p26_hb.log; grep "hbcheck" gpurun_out/p26_hb.log | grep -v " 0 violations" | head -5
tail -2 gpurun_out/p26_hb.log
CPDB_SHARD_OVERLAP=0 timeout 600 python -m pytest tests/test_gpu_sharded.py -q -x -p no:cacheprovider -k "matches_unsharded" > gpurun_out/p26_noov.log 2>&1; echo noov rc=$?; tail -1 gpurun_out/p26_noov.log
