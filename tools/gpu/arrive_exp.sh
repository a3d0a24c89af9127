cd $GRAFT_REPO_ROOT
for L in 0 1; do
 echo "== layout $L control (HEAD build), exact smem"
 CPDB_TTM_SMEM_EXACT=1 ./tools/probes/ttm_coresid_ctl $L 20 0 64 cluster | tail -3
 for M in 0 1 2; do
  echo "== layout $L new build arrive_mode $M, exact smem"
  CPDB_TTM_ARRIVE=$M CPDB_TTM_SMEM_EXACT=1 ./tools/probes/ttm_coresid $L 20 0 64 cluster | tail -3
  CPDB_TTM_ARRIVE=$M CPDB_TTM_SMEM_EXACT=1 HOG_WRITE=1 ./tools/probes/ttm_coresid $L 20 0 296 cluster | tail -1
 done
done
