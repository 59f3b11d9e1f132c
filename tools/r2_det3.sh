mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "determin or embedding or bwd_chain or c2_block or lms or autotune" > gpurun_out/det_tests.log 2>&1; tail -3 gpurun_out/det_tests.log
for b in fused streams; do
timeout 300 python bench.py --deterministic --bwd $b --steps 20 --warmup 5 --no-cpu --sustained-seconds 0 --extras 0 > gpurun_out/det_c2_$b.json 2> gpurun_out/det_c2_$b.err
python -c "
import json;d=json.loads(open('gpurun_out/det_c2_$b.json').read().strip().splitlines()[-1]);print(round(d['value'],1), d['config'].get('backward'), d['roofline']['frac'], {k:round(v*1e3,1) for k,v in d['roofline']['per_kind_ms'].items()}, d['dense_cublas']['tflops'])"
done
