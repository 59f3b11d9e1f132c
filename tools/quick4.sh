timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "emb or c4 or determin or bias" 2>&1 | tail -2
for A in 32 8; do
timeout 300 python tools/emb_bench.py --deterministic --align $A 2>&1 | tail -1
ROAST_EMB_DET_WARP=1 timeout 300 python tools/emb_bench.py --deterministic --align $A 2>&1 | tail -1
done
