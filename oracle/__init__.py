"""ROAST CPU oracle — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct fp64 implementation of what the ROAST hot
path computes, written from PAPER.md (arXiv 2207.10702) with the readings of
SURVEY.md §8(c) / DESIGN.md "Readings".  It shares no code with the CUDA
library (paper_2207_10702_b200/); neither imports the other.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference`
legs may import it.  The product path never routes through it.

Modules
  hashing    Appendix A mapping: h1 / h2 offsets, sign g, lambda
  roast_mm   materialise W, Y = X W, dX = dY W^T, dM scatter
  embedding  L lookup forward and gradient scatter
  estimator  GMS / LMS feature-hashing estimators, Theorem 1

Parity status of each function is stated in its docstring ("pinned by" /
"parity unpinned").
"""
