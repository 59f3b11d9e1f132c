# shadow replicas A/B at 1000x and 100x (default policy vs ROAST_SHADOW_REPS=1), parity of the GEMM suite first
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
for r in 1000 100; do for reps in 1 def; do
if [ $reps = def ]; then unset ROAST_SHADOW_REPS; else export ROAST_SHADOW_REPS=$reps; fi
timeout 300 python bench.py --ratio $r --steps 20 --warmup 5 --no-cpu --sustained-seconds 0 --extras 0 > gpurun_out/reps_${r}_${reps}.json 2> gpurun_out/reps_${r}_${reps}.err
python -c "
import json;d=json.loads(open('gpurun_out/reps_${r}_${reps}.json').read().strip().splitlines()[-1]);print('$r $reps', round(d['value'],1), d['config'].get('backward'), {k:round(v*1e3,1) for k,v in d['roofline']['per_kind_ms'].items()})"
done; done
unset ROAST_SHADOW_REPS
timeout 300 python tools/prof_shapes.py --exps 0 --wm 2 --mem 4720 > gpurun_out/shapes1000.log 2>&1; grep -v "^\[roast" gpurun_out/shapes1000.log | tail -20
