"""paper_2207_10702_b200 — B200-native hot path of ROAST hashing (arXiv 2207.10702).

The product is libroast.so (C ABI, include/roast.h) built from csrc/ for
sm_100a; `roast` is its thin ctypes binding.  Build with
`python -m paper_2207_10702_b200.build`.
"""
