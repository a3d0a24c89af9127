for v in "X=1" "CPDB_VSPLIT_MAX=8" "CPDB_VSPLIT_MAX=24" "CPDB_OVERLAP_FRAC=0.3" "CPDB_OVERLAP_FRAC=0.5" "CPDB_PREFETCH_TPC=1" "CPDB_PREFETCH_TPC=3" "CPDB_TAIL_SMS=64" "CPDB_TAIL_SMS=100" "X=1"; do
  env $v timeout 120 python bench.py --steps 300 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p20.json 2> gpurun_out/p20.err
  echo "$v rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p20.json')); print(round(d['value'],1))" 2>/dev/null)"
done
