set -x
nproc; free -g; lscpu | head -20; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for v in "" "CPDB_NO_PDL=1" "CPDB_ROOT_PREFETCH=0" "CPDB_EARLY_FRONT=0" "CPDB_CHAIN_EVENTS=0" "CPDB_SPECULATE=0" "CPDB_CHAIN_SIDE=0"; do
  echo "=== exact $v"
  env CPDB_TTM_SMEM_EXACT=1 $v timeout 300 python tools/det_probe.py c3 40 4 2>&1 | tail -4
done
echo "=== baseline (227KB)"
timeout 300 python tools/det_probe.py c3 40 4 2>&1 | tail -3
