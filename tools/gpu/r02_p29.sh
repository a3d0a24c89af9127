timeout 120 python tools/timeline.py c3 --warmup 6 --sweeps 4 > gpurun_out/tl_c3.txt 2>&1
