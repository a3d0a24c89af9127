for v in "" "CPDB_TTM_NC7=1" "CPDB_OVERLAP_FRAC=0.3" "CPDB_OVERLAP_FRAC=0.5" "CPDB_LOW_TAIL=0" "CPDB_TAIL_SMS=40" "CPDB_TAIL_SMS=120" "CPDB_ZQR_AUX=0" "CPDB_SPEC_STREAM=aux" "CPDB_VSPLIT_MAX=8" "CPDB_PREFETCH_TPC=1"; do
  echo "=== $v"
  for rep in 1 2; do env $v python tools/run_boundary_probe.py c2 5 100 | grep whole | cut -c1-30; done
done
