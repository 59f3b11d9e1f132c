# 1000x diagnosis: per-GEMM ROAST vs cuBLAS at |M| = 4720, both backward schedules
mkdir -p gpurun_out
for b in fused streams; do
timeout 600 python bench.py --ratio 1000 --bwd $b --steps 20 --warmup 5 --no-cpu --sustained-seconds 0 > gpurun_out/b1000_$b.json 2> gpurun_out/b1000_$b.err; tail -2 gpurun_out/b1000_$b.err
done
timeout 300 python bench.py --ratio 100 --steps 20 --warmup 5 --no-cpu --sustained-seconds 0 --extras 0 > gpurun_out/b100.json 2> gpurun_out/b100.err
