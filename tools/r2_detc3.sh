mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_exchange.py -m gpu -q -x -k "determin or bwd_chain or c2_block or lms or autotune or poison or workspace" > gpurun_out/detc3_tests.log 2>&1; tail -2 gpurun_out/detc3_tests.log
for i in 1 2; do
timeout 300 python bench.py --deterministic --steps 20 --warmup 5 --no-cpu --sustained-seconds 0 --extras 0 > gpurun_out/detc3.json 2> gpurun_out/detc3.err
python -c "
import json;d=json.loads(open('gpurun_out/detc3.json').read().strip().splitlines()[-1]);print('auto', round(d['value'],1), d['config'].get('backward'), {k:round(v*1e3,1) for k,v in d['roofline']['per_kind_ms'].items()}, d['dense_cublas']['tflops'], d['value']/d['dense_cublas']['tflops'])"
done
ROAST_BENCH_KEEP_BWD=1 timeout 600 ncu --nvtx --nvtx-include "roast_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/det_launches.csv python bench.py --deterministic --steps 3 --warmup 3 --no-cpu --extras 0 --sustained-seconds 0 --nvtx-step > /dev/null 2>&1
python - <<'PY'
import csv
for f in ("gpurun_out/det_launches.csv",):
    rows=[r for r in csv.reader(open(f)) if len(r)>10]
    h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
    for r in rows[1:]: print("  ", r[ki][:90], r[vi])
PY
