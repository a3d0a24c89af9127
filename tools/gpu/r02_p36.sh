for v in 0 1 2 0 1 2; do
  CPDB_TTM_BRANCHCFG=$v timeout 120 python bench.py --config c2 --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p36.json 2> gpurun_out/p36.err
  echo "c2 bcfg=$v rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p36.json')); r=d['roofline']; print(round(d['value'],1), round(d['kernel_ms_per_step']['branch_ttm'],4))" 2>/dev/null)"
done
