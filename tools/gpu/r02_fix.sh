cd $GRAFT_REPO_ROOT
bash tools/gpu/coresid.sh > gpurun_out/coresid.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_suite2.log 2>&1; echo suite_rc=$? >> gpurun_out/gpu_suite2.log
for C in c2 c3 c4; do python bench.py --config $C --steps 100 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fix_$C.json 2>/dev/null; done
python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fix_c5.json 2>/dev/null
for C in c2 c3; do CPDB_TTM_SMEM_WHOLE=1 python bench.py --config $C --steps 100 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fixwhole_$C.json 2>/dev/null; done
