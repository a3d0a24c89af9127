for v in "CPDB_OVERLAP_FRAC=0.5" "CPDB_OVERLAP_FRAC=0.6" "CPDB_OVERLAP_FRAC=0.75" "CPDB_OVERLAP_FRAC=1.0" "CPDB_OVERLAP_FRAC=0.5 CPDB_ZQR_AUX=0" "CPDB_OVERLAP_FRAC=0.5 CPDB_ZQR_AUX=0 CPDB_TAIL_SMS=40" "CPDB_OVERLAP_FRAC=0.6 CPDB_TAIL_SMS=40"; do
  echo "=== $v"
  for rep in 1 2; do env $v python tools/run_boundary_probe.py c2 5 100 | grep whole | cut -c1-30; done
done
for v in "" "CPDB_OVERLAP_FRAC=0.5" "CPDB_OVERLAP_FRAC=0.75"; do
  echo "=== c3 $v"
  for rep in 1 2; do env $v python tools/run_boundary_probe.py c3 5 60 | grep whole | cut -c1-30; done
done
for v in "" "CPDB_ZQR_AUX=0"; do
  echo "=== c4 $v"
  for rep in 1 2; do env $v python tools/run_boundary_probe.py c4 5 200 | grep whole | cut -c1-30; done
  echo "=== c1 $v"
  for rep in 1 2; do env $v python tools/run_boundary_probe.py c1 5 200 | grep whole | cut -c1-30; done
done
