# quick GPU iteration: parity suite (tcgen05 parts), kernel shape timings, one bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -5 gpurun_out/gpu_tests.log
timeout 300 python tools/prof_shapes.py --exps 0 > gpurun_out/shapes.log 2>&1; cat gpurun_out/shapes.log | grep -v "^\[roast"
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
