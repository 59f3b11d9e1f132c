mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/clocks.csv &
SMI=$!
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
kill $SMI
python - <<'PY'
import json
d=json.load(open('gpurun_out/bench.json'))
for k in ['value','ms_per_step','roofline','dense_cublas','sustained','clocks','e2e']: print(k, json.dumps(d.get(k))[:700])
e=d.get('extra') or {}
print('per_gemm', json.dumps({k:(round(v['roast_us'],1),round(v['cublas_us'],1)) for k,v in e.get('per_gemm',{}).get('gemms',{}).items()}))
print('variants', json.dumps({k:round(v.get('value',0),1) for k,v in e.get('c2_variants',{}).items()}))
print('c4', json.dumps(e.get('c4_embeddings'))[:500])
PY
