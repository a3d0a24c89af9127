python -c "
import ctypes
cr=ctypes.CDLL('libcudart.so.12') if False else None
" 2>/dev/null
python - <<'PY'
import torch
print("torch prio range", torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream,'priority_range') else None)
import ctypes, glob
for p in glob.glob('/usr/local/cuda/lib64/libcudart.so*'):
    try:
        lib = ctypes.CDLL(p); break
    except OSError: pass
lo, hi = ctypes.c_int(), ctypes.c_int()
print("cudart", p, lib.cudaDeviceGetStreamPriorityRange(ctypes.byref(lo), ctypes.byref(hi)), lo.value, hi.value)
PY
for v in "CPDB_TAIL_SMS=0" "CPDB_TAIL_SMS=64" "CPDB_TAIL_SMS=96" "CPDB_TAIL_SMS=128" "CPDB_TAIL_SMS=0" "CPDB_TAIL_SMS=64"; do
  env $v timeout 120 python bench.py --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/p10.json 2> gpurun_out/p10.err
  echo "$v rc=$? $(python -c "import json; d=json.load(open('gpurun_out/p10.json')); print(round(d['value'],1))" 2>/dev/null)"
done
timeout 300 python tools/strategy_bench.py --out gpurun_out/strategies.json > /dev/null 2> gpurun_out/strategies.err; echo strat rc=$?
python -c "
import json
for c in json.load(open('gpurun_out/strategies.json')):
    print(c['case'], c['c12_order_holds'], round(c['br_over_naive'],3), {k: round(v,3) for k,v in c['time_ratio_vs_naive'].items()}, {k: round(v['steady_sweeps_per_s'],1) for k,v in c['results'].items()})
"
