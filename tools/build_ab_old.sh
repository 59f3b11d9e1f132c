#!/bin/bash
# Build libroast_old.so = the working tree's library with gemm_sm100.cu taken from git REV (default HEAD),
# for A/B timing with tools/ab_bench.sh.
set -e
REV=${1:-HEAD}
cd "$(dirname "$0")/.."
python -c "import sys; sys.path.insert(0,'.'); from paper_2207_10702_b200 import build; build.build()"
git show $REV:paper_2207_10702_b200/csrc/gemm_sm100.cu > paper_2207_10702_b200/csrc/zz_old.cu.txt
(cd paper_2207_10702_b200/csrc && /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
  -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -I../../include -x cu -c zz_old.cu.txt -o /tmp/gemm_old.o)
rm paper_2207_10702_b200/csrc/zz_old.cu.txt
objs=""
for f in paper_2207_10702_b200/csrc/*.cu; do b=$(basename $f); [ $b = gemm_sm100.cu ] && continue; objs="$objs paper_2207_10702_b200/build/$b.o"; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o libroast_old.so $objs /tmp/gemm_old.o -ldl
echo built libroast_old.so from $REV
