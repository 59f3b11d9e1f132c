timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "chain or 192 or fuzz or c2_full or bit_exact or parity" 2>&1 | tail -2
timeout 300 python tools/prof_shapes.py --exps 0 --wm 2 2>&1 | grep -v "^\[" | head -8
timeout 300 python tools/bwd_fused_probe.py 8192 2>&1 | tail -1
