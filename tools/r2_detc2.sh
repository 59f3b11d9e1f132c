mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "bwd_chain" > gpurun_out/detc2_tests.log 2>&1; tail -2 gpurun_out/detc2_tests.log
for c in 0 11 40; do
ROAST_VERBOSE=1 ROAST_DET_SPLIT_COST=$c ROAST_BENCH_KEEP_BWD=1 timeout 300 python bench.py --deterministic --bwd fused --steps 20 --warmup 5 --no-cpu --sustained-seconds 0 --extras 0 > gpurun_out/detc2_$c.json 2> gpurun_out/detc2_$c.err
grep "bwd chain plan" gpurun_out/detc2_$c.err | head -2
python -c "
import json;d=json.loads(open('gpurun_out/detc2_$c.json').read().strip().splitlines()[-1]);print('cost $c', round(d['value'],1), d['config'].get('backward'), {k:round(v*1e3,1) for k,v in d['roofline']['per_kind_ms'].items()}, d['dense_cublas']['tflops'])"
done
timeout 300 python bench.py --deterministic --steps 20 --warmup 5 --no-cpu --sustained-seconds 0 --extras 0 > gpurun_out/detc2_auto.json 2> gpurun_out/detc2_auto.err
python -c "
import json;d=json.loads(open('gpurun_out/detc2_auto.json').read().strip().splitlines()[-1]);print('auto', round(d['value'],1), d['config'].get('backward'), {k:round(v*1e3,1) for k,v in d['roofline']['per_kind_ms'].items()}, d['dense_cublas']['tflops'])"
