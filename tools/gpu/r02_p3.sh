timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=12 > gpurun_out/gputest_p3.log 2>&1; echo tests rc=$?
tail -22 gpurun_out/gputest_p3.log
CPDB_PHASE_TRACE=1 python tools/phase_trace.py c2 2> gpurun_out/phase_c2.txt > /dev/null; echo phase rc=$?
tail -12 gpurun_out/phase_c2.txt
