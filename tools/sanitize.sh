#!/bin/bash
# compute-sanitizer passes over the GPU parity suite (round-1 evidence: profiles/round1/sanitizer_*.txt).
# PYTORCH_NO_CUDA_MEMORY_CACHING=1 so every torch tensor is its own allocation and memcheck sees
# out-of-bounds accesses that the caching allocator's pooled blocks would hide.
set -u
mkdir -p gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
SEL=${SEL:-"not fullsize and not fuzz"}
for tool in ${TOOLS:-memcheck synccheck initcheck racecheck}; do
  timeout ${TMO:-1200} compute-sanitizer --tool $tool --error-exitcode 99 --print-limit 20 \
    python -m pytest tests/test_gpu_parity.py tests/test_gpu_exchange.py tests/test_gpu_model.py \
    -q -x -p no:cacheprovider -k "$SEL" > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer_rc.txt
done
