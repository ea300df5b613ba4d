"""TEST INFRASTRUCTURE ONLY -- the checkers for the B200 BM25 path.

restate: plain-C restatement of the reference hot path (oracle/bm25_oracle.c)
ref:     the unmodified reference library built from /root/reference sources
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this package; the product path (paper_2605_25092_b200) never does.
"""
