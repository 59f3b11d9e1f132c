# GPU validation of a round: full -m gpu suite, smoke(), the default bench line with extras, C3 at 65 536 tokens
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json;d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]);print(round(d['value'],1), d['roofline']['frac'], {k:round(v*1e3,1) for k,v in d['roofline']['per_kind_ms'].items()}, d['dense_cublas']['tflops']); ex=d.get('extra',{}); print({k:(round(v.get('value',0),1), v.get('bwd')) for k,v in ex.get('c2_variants',{}).items()}); print(json.dumps(ex.get('c3_bert_step')))"
timeout 600 python bench.py --workload c3 --steps 10 --warmup 3 > gpurun_out/c3.json 2> gpurun_out/c3.err
python -c "
import json;d=json.loads(open('gpurun_out/c3.json').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['breakdown']['ms'], d['e2e'])"
