cd $GRAFT_REPO_ROOT
for M in 0 1 5; do
 for C in c2 c5; do
  S=100; [ $C = c5 ] && S=10
  CPDB_TTM_ARRIVE=$M python bench.py --config $C --steps $S --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('mode $M $C', round(d['value'],2), 'root frac', round(d['roofline']['frac'],4), round(d['roofline']['frac_in_timed_run'],4))"
 done
done
echo "== exact smem (co-residency allowed), mode 5"
for C in c2 c3 c4; do
  CPDB_TTM_SMEM_EXACT=1 CPDB_TTM_ARRIVE=5 python bench.py --config $C --steps 100 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('exact mode 5 $C', round(d['value'],2))"
  CPDB_TTM_ARRIVE=5 python bench.py --config $C --steps 100 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('227K mode 5 $C', round(d['value'],2))"
done
echo "== det probe c3, exact smem, no pdl, mode 5"
CPDB_TTM_ARRIVE=5 CPDB_TTM_SMEM_EXACT=1 CPDB_NO_PDL=1 python tools/det_probe.py c3 60 4 2>&1 | tail -1
CPDB_TTM_ARRIVE=5 CPDB_TTM_SMEM_EXACT=1 python tools/det_probe.py c3 60 4 2>&1 | tail -1
echo "== probe mode 5 exact smem"
for L in 0 1; do CPDB_TTM_ARRIVE=5 CPDB_TTM_SMEM_EXACT=1 ./tools/probes/ttm_coresid $L 20 0 64 cluster | tail -1; CPDB_TTM_ARRIVE=5 CPDB_TTM_SMEM_EXACT=1 HOG_WRITE=1 ./tools/probes/ttm_coresid $L 20 0 296 cluster | tail -1; done
