mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -k "determin or embedding or bwd_chain or c2_block" > gpurun_out/det_tests.log 2>&1; tail -3 gpurun_out/det_tests.log
bash tools/r2_det.sh
