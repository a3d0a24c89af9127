B="CPDB_TTM_SMEM_EXACT=1 CPDB_NO_PDL=1"
for round in 1 2; do
for v in "" "CPDB_TTM=1" "CPDB_VSPLIT_MAX=0" "CPDB_EARLY_CHAIN_RELAXED=0" "CPDB_CHAIN_EVENTS=0" "CPDB_ZQR_AUX=1"; do
  echo "=== $B $v"
  env $B $v timeout 300 python tools/det_probe.py c3 40 4 2>&1 | tail -1
done
done
echo "=== CPDB_TTM=1 only"
CPDB_TTM=1 CPDB_NO_PDL=1 timeout 300 python tools/det_probe.py c3 40 4 2>&1 | tail -1
