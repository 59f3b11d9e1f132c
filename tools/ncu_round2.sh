# ncu evidence for the round-2 step: launch list of one bench step + --set full of its GEMM kernels
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-cpu --extras 0 --sustained-seconds 0 --nvtx-step"
timeout 600 ncu --nvtx --nvtx-include "roast_step/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_r2.csv $B > gpurun_out/ncu_launch.log 2>&1; tail -2 gpurun_out/ncu_launch.log
timeout 900 ncu --nvtx --nvtx-include "roast_step/" --set full --clock-control none --import-source on \
  -k regex:"roast_m" -o gpurun_out/prof_r2 -f $B > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
ls -la gpurun_out/
