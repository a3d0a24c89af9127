timeout 900 python -m pytest tests/test_gpu_sharded.py -q -x -p no:cacheprovider -k "c5_proxy" -o faulthandler_timeout=300 > gpurun_out/p25_tests.log 2>&1; echo tests rc=$?
tail -2 gpurun_out/p25_tests.log
free -g | head -2
for k in 4 12; do
  timeout 1500 python tools/teacher_forced.py c5 $k --out gpurun_out/r02_parity_c5_tf_k${k}_v2.json 2> gpurun_out/c5full_k$k.err > /dev/null
  echo "k=$k rc=$?"; tail -3 gpurun_out/c5full_k$k.err
done
