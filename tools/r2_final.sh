# round-2 refresh: full GPU suite, smoke, default bench line, C3 (encoder, whole BERT; ROAST vs dense)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "
import json;d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1]);print(round(d['value'],1), d['config'].get('backward'), d['roofline']['frac'], {k:round(v*1e3,1) for k,v in d['roofline']['per_kind_ms'].items()}, d['dense_cublas']['tflops']); ex=d.get('extra',{}); print({k:(round(v.get('value',0),1), v.get('bwd')) for k,v in ex.get('c2_variants',{}).items()}); print(ex.get('c4_embeddings'))"
for a in "" "--dense" "--full" "--full --dense"; do timeout 300 python tools/bert_step.py $a --steps 10 2>/dev/null | tail -1; done > gpurun_out/bert_steps.jsonl; cat gpurun_out/bert_steps.jsonl
