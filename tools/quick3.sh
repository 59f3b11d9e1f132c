timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "bwd_chain or determin or poison or lms" 2>&1 | tail -2
timeout 300 python tools/det_dm_bench.py 2>&1 | tail -4
timeout 600 python bench.py --deterministic --steps 10 --warmup 3 --extras 0 --no-cpu --sustained-seconds 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['config']['backward'], d['dense_cublas']['roast_over_dense'], d['roofline']['per_kind_ms'])"
