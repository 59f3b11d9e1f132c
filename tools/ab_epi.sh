for e in 0 1; do echo "ROAST_EPI=$e"; ROAST_EPI=$e timeout 120 python tools/prof_step.py 2>&1 | tail -6; done
ROAST_EPI=1 timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for e in 0 1; do ROAST_EPI=$e timeout 200 python bench.py --steps 20 --warmup 5 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('EPI', $e, round(d['value'],1), d['roofline']['per_kind_ms'], round(d['dense_cublas']['roast_over_dense'],3))"; done
