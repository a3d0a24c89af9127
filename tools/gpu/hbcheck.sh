# happens-before check of the multi-stream sweep on every BASELINE config
for cfg in c1 c2 c3 c4 c5; do
  echo "=== $cfg"
  CPDB_HBCHECK=1 timeout 600 python tools/det_probe.py $cfg 2 8 2>&1 | sort | uniq -c | sort -rn | head -30
done
for v in "CPDB_ROOT_PREFETCH=0" "CPDB_EARLY_FRONT=0" "CPDB_CHAIN_SIDE=0" "CPDB_SPECULATE=0"; do
  echo "=== c3 $v"
  env CPDB_HBCHECK=1 $v timeout 600 python tools/det_probe.py c3 2 8 2>&1 | sort | uniq -c | sort -rn | head -20
done
