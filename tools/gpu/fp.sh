rm -f gpurun_out/fp_c3*.txt
CPDB_FINGERPRINT=gpurun_out/fp_c3.txt CPDB_FINGERPRINT_LIGHT=1 CPDB_TTM_SMEM_EXACT=1 CPDB_NO_PDL=1 timeout 600 python tools/det_probe.py c3 20 4 2>&1 | tail -3
python tools/fp_compare.py gpurun_out/fp_c3.txt
