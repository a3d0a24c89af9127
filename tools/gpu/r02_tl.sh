python tools/timeline.py c2 --warmup 6 --sweeps 3 > gpurun_out/tl_c2.txt 2>&1; echo tl rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ttm_tma_kernel --launch-skip 30 --launch-count 8 -o gpurun_out/ttm_c2_r02 -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_ttm.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_ttm.log
