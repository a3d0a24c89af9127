for v in "CPDB_TTM_SMEM_EXACT=1 CPDB_NO_PDL=1" "CPDB_TTM_SMEM_EXACT=1 CPDB_NO_PDL=1 CPDB_PROXY_FENCE=1"; do
  echo "=== $v"
  env $v timeout 300 python tools/det_probe.py c3 40 4 2>&1 | tail -2
done
