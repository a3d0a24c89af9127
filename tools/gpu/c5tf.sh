python -m pytest tests/test_gpu_solver.py -q -x -k c5_proxy 2>&1 | tail -5
python tools/teacher_forced.py c5 4 --dims 64x64x64x64 --out gpurun_out/tf_c5proxy_k4.json > /dev/null
python tools/teacher_forced.py c5 12 --dims 64x64x64x64 --out gpurun_out/tf_c5proxy_k12.json > /dev/null
