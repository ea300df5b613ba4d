"""B200-native BM25 hot path of AgentIR (arxiv/paper_2605_25092).

Batched BM25 term-at-a-time scoring over a resident CSR inverted index, exact
per-query top-k and the cascade-trigger margin, on hand-written sm_100a
kernels behind a C ABI (include/hm_b200.h).  This package is the Python host
mirror of the reference's C++ search API (proj/include/hybrid/*.hpp).
"""
__all__ = ["synth", "search"]
