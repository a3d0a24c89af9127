# TMA TTM beside DSMEM cluster grids: the round-1 build (tools/probes/ctl/, arrive
# before the stage's shared loads returned) vs the current build (data-dependent arrive)
P=./tools/probes/ttm_coresid
C=./tools/probes/ttm_coresid_ctl
echo "# TMA TTM (ttm_tma.cu) beside other grids: outputs vs an isolated run (bitwise)"
echo "# layout 0 = contract last mode (kRows, 262144x128 -> R16), 1 = contract first (kGroups)"
for L in 0 1; do
 if [ -x $C ]; then
  echo "--- layout $L, previous build (arrive could overtake in-flight LDS), ring-sized smem"
  CPDB_TTM_SMEM_EXACT=1 $C $L 40 0 64 cluster | tail -1
  CPDB_TTM_SMEM_EXACT=1 HOG_WRITE=1 $C $L 40 0 296 cluster | tail -1
 fi
 echo "--- layout $L, current build (arrive after the stage's loads returned), ring-sized smem (default)"
 $P $L 40 0 64 cluster | tail -1
 $P $L 40 0 296 cluster | tail -1
 HOG_WRITE=1 $P $L 40 0 64 cluster | tail -1
 HOG_WRITE=1 $P $L 40 0 296 cluster | tail -1
 HOG_NO_DSMEM=1 $P $L 40 0 64 cluster | tail -1
 $P $L 40 32768 296 hog | tail -1
done
echo "# repeated C3 solves (tools/det_probe.py c3 90 4): mismatching runs, co-residency allowed"
python tools/det_probe.py c3 90 4 2>&1 | tail -1
echo "(CPDB_NO_PDL=1)"; CPDB_NO_PDL=1 python tools/det_probe.py c3 90 4 2>&1 | tail -1
