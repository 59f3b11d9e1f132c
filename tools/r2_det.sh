# deterministic-mode breakdown: C2 step (per kind + ncu launch list), C4 backward launch list
mkdir -p gpurun_out
timeout 300 python bench.py --deterministic --steps 20 --warmup 5 --no-cpu --sustained-seconds 0 --extras 0 > gpurun_out/det_c2.json 2> gpurun_out/det_c2.err
python -c "
import json;d=json.loads(open('gpurun_out/det_c2.json').read().strip().splitlines()[-1]);print(round(d['value'],1), d['config'].get('backward'), d['roofline']['frac'], {k:round(v*1e3,1) for k,v in d['roofline']['per_kind_ms'].items()}, d['dense_cublas']['tflops'])"
timeout 300 python bench.py --deterministic --bwd streams --steps 20 --warmup 5 --no-cpu --sustained-seconds 0 --extras 0 > gpurun_out/det_c2s.json 2> gpurun_out/det_c2s.err
python -c "
import json;d=json.loads(open('gpurun_out/det_c2s.json').read().strip().splitlines()[-1]);print(round(d['value'],1), d['config'].get('backward'), d['roofline']['frac'], {k:round(v*1e3,1) for k,v in d['roofline']['per_kind_ms'].items()})"
timeout 600 ncu --nvtx --nvtx-include "roast_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/det_launches.csv python bench.py --deterministic --steps 3 --warmup 3 --no-cpu --extras 0 --sustained-seconds 0 --nvtx-step > /dev/null 2>&1
python tools/emb_bench.py --deterministic --steps 10 > gpurun_out/emb_det.json 2>&1; tail -3 gpurun_out/emb_det.json
timeout 600 ncu --nvtx --nvtx-include "emb_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/emb_det_launches.csv python tools/emb_bench.py --deterministic --nvtx --steps 2 > /dev/null 2>&1
python - <<'PY'
import csv
for f in ("gpurun_out/det_launches.csv","gpurun_out/emb_det_launches.csv"):
    rows=[r for r in csv.reader(open(f)) if len(r)>10]
    h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
    print(f)
    for r in rows[1:]: print("  ", r[ki][:90], r[vi])
PY
