for cfg in c2 c3; do
  echo "=== $cfg"
  CPDB_HBCHECK=1 timeout 600 python tools/det_probe.py $cfg 1 8 2>&1 | head -30
done
