CS=/usr/local/cuda/bin/compute-sanitizer
for shape in "24x20x18x16:8" "40x36x32:16" "64x48x40:32"; do
  echo "=== racecheck $shape"
  timeout 900 $CS --tool racecheck --racecheck-report hazard --print-limit 20 python tools/det_probe.py $shape 1 4 2>&1 | grep -v "^$" | head -60
done
echo "=== synccheck"
timeout 600 $CS --tool synccheck --print-limit 20 python tools/det_probe.py 24x20x18x16:8 1 4 2>&1 | tail -20
