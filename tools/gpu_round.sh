# one GPU round: parity tests, bench, launch list, one full ncu capture of the GEMM kernels
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
if [ "${NCU:-1}" = "1" ]; then
# launch list of one bench step (all kernels inside the NVTX range of the extra eager step)
timeout 300 ncu --nvtx --nvtx-include "roast_step/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu --nvtx-step --tuned-file gpurun_out/bench.json > /dev/null 2>&1
timeout 900 ncu --nvtx --nvtx-include "roast_step/" --set full --clock-control none --import-source on -k regex:roast_mm_sm100 -o gpurun_out/prof_mm -f python bench.py --steps 3 --warmup 3 --no-cpu --nvtx-step --tuned-file gpurun_out/bench.json > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
timeout 300 ncu --nvtx --nvtx-include "emb_step/" --set full --clock-control none --import-source on -k regex:embed_kernel -o gpurun_out/prof_emb -f python tools/emb_bench.py --nvtx --steps 2 > gpurun_out/ncu_emb.log 2>&1; tail -1 gpurun_out/ncu_emb.log
fi
timeout 300 python tools/emb_bench.py > gpurun_out/emb.json 2>&1; tail -1 gpurun_out/emb.json
timeout 300 python tools/emb_bench.py --dist zipf > gpurun_out/emb_zipf.json 2>&1; tail -1 gpurun_out/emb_zipf.json
