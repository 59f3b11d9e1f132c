# A/B: bench with two library builds, interleaved
for i in 1 2 3; do
  for lib in libroast_old.so paper_2207_10702_b200/libroast.so; do
    ROAST_LIB=$PWD/$lib timeout 300 python bench.py --no-cpu --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['value'],1), d['ms_per_step'], d['roofline']['per_kind_ms'], round(d['dense_cublas']['roast_over_dense'],3))"
  done
done
