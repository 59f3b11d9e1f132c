mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "embedding or c4" > gpurun_out/emb_tests.log 2>&1; tail -3 gpurun_out/emb_tests.log
for d in uniform zipf; do for a in 32 8; do python tools/emb_bench.py --deterministic --steps 10 --dist $d --align $a > gpurun_out/emb_det_${d}_$a.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/emb_det_${d}_$a.json').read().strip().splitlines()[-1]); print('$d A=$a bwd_multi', d['bwd_multi'])"; done; done
timeout 600 ncu --nvtx --nvtx-include "emb_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/emb_det_launches.csv python tools/emb_bench.py --deterministic --nvtx --steps 2 > /dev/null 2>&1
python - <<'PY'
import csv
for f in ("gpurun_out/emb_det_launches.csv",):
    rows=[r for r in csv.reader(open(f)) if len(r)>10]
    h=rows[0]; ki=h.index("Kernel Name"); vi=h.index("Metric Value")
    print(f)
    for r in rows[1:]: print("  ", r[ki][:90], r[vi])
PY
