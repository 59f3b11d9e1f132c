# full GPU suite + the default bench line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json;d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]);print(round(d['value'],1), d['config'].get('backward'), d['roofline']['frac'], {k:round(v*1e3,1) for k,v in d['roofline']['per_kind_ms'].items()}); ex=d.get('extra',{}); print({k:(round(v.get('value',0),1), v.get('bwd')) for k,v in ex.get('c2_variants',{}).items()})"
