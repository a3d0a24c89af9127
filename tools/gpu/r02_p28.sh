for st in 20 100; do
timeout 300 python bench.py --steps $st --warmup 5 --no-cpu-baseline > gpurun_out/p28.json 2> gpurun_out/p28.err
python -c "import json; d=json.load(open('gpurun_out/p28.json')); print($st, round(d['value'],1), {k:(round(v,2) if isinstance(v,float) else v) for k,v in d['e2e'].items() if k!='note'})"
done
