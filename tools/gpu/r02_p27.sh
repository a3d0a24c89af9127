timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -o faulthandler_timeout=200 --durations=8 > gpurun_out/p27_tests.log 2>&1; echo tests rc=$?
tail -14 gpurun_out/p27_tests.log
