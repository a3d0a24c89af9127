P=./tools/probes/ttm_coresid
echo "# TMA TTM (ttm_tma.cu) beside other grids: outputs vs an isolated run (bitwise)"
echo "# layout 0 = contract last mode (kRows, 262144x128 -> R16), 1 = contract first (kGroups)"
for L in 0 1; do
 echo "--- layout $L, exclusive SMs (default: 227 KB per TTM CTA)"
 $P $L 40 0 64 cluster | tail -1
 $P $L 40 0 296 cluster | tail -1
 HOG_WRITE=1 $P $L 40 0 64 cluster | tail -1
 echo "--- layout $L, ring-sized smem (CPDB_TTM_SMEM_EXACT=1: co-residency allowed)"
 CPDB_TTM_SMEM_EXACT=1 $P $L 40 0 64 cluster | tail -1
 CPDB_TTM_SMEM_EXACT=1 $P $L 40 0 296 cluster | tail -1
 CPDB_TTM_SMEM_EXACT=1 HOG_WRITE=1 $P $L 40 0 64 cluster | tail -1
 CPDB_TTM_SMEM_EXACT=1 HOG_NO_DSMEM=1 $P $L 40 0 64 cluster | tail -1
 CPDB_TTM_SMEM_EXACT=1 $P $L 40 32768 296 hog | tail -1
 CPDB_TTM_SMEM_EXACT=1 CPDB_TTM=1 $P $L 40 0 64 cluster | tail -1
done
echo "# repeated C3 solves (tools/det_probe.py c3 90 4): mismatching runs"
python tools/det_probe.py c3 90 4 2>&1 | tail -1
CPDB_NO_PDL=1 python tools/det_probe.py c3 90 4 2>&1 | tail -1
echo "(CPDB_TTM_SMEM_EXACT=1 CPDB_NO_PDL=1)"; CPDB_TTM_SMEM_EXACT=1 CPDB_NO_PDL=1 python tools/det_probe.py c3 90 4 2>&1 | tail -1
