# one GPU round: parity tests, bench, launch list, one full ncu capture of the GEMM kernels
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
if [ "${NCU:-1}" = "1" ]; then
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --graph 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:roast_mm_sm100 -s 6 -c 6 -o gpurun_out/prof_mm -f python bench.py --steps 1 --warmup 1 --no-cpu --graph 0 > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
timeout 300 ncu --set full --clock-control none -k regex:embed_kernel -c 2 -o gpurun_out/prof_emb -f python tools/emb_bench.py --quick > gpurun_out/ncu_emb.log 2>&1; tail -1 gpurun_out/ncu_emb.log
fi
timeout 300 python tools/emb_bench.py > gpurun_out/emb.json 2>&1; tail -1 gpurun_out/emb.json
timeout 300 python tools/emb_bench.py --dist zipf > gpurun_out/emb_zipf.json 2>&1; tail -1 gpurun_out/emb_zipf.json
