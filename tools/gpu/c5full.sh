free -g | head -2
for k in 4 12; do
  python tools/teacher_forced.py c5 $k --out gpurun_out/r02_parity_c5_tf_k$k.json 2> gpurun_out/c5full_k$k.err > /dev/null
  echo "k=$k rc=$?"; tail -5 gpurun_out/c5full_k$k.err
done
