"""Dense escalate channel: GPU exact inner-product top-k vs the reference CPU
(dense_topk, src/dense.cpp:86-101).

Workload (synthetic, seed 11): --docs random unit vectors of --dim floats
(the reference's EmbeddingMatrix layout), --queries unit query vectors (the
escalated share of a batch: 20% of 10K by default), k = 10.  Work per query =
docs x dim fp64 multiply-adds, exactly the reference's.

    python tools/dense_bench.py [--docs 8841823] [--dim 64] [--queries 2000]

Prints one JSON line: kernel / host-API throughput, the fp64 rate achieved,
the reference's multi-threaded CPU throughput on a bounded sample and a parity
check of that sample (ids and score bits).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_25092_b200 import search  # noqa: E402


def unit_rows(rng, n, dim, chunk=1 << 20):
    out = np.empty((n, dim), np.float32)
    for s in range(0, n, chunk):
        x = rng.standard_normal((min(chunk, n - s), dim), dtype=np.float32)
        out[s:s + len(x)] = x / np.linalg.norm(x, axis=1, keepdims=True)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--docs", type=int, default=8_841_823)
    ap.add_argument("--dim", type=int, default=64)
    ap.add_argument("--queries", type=int, default=2000)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--ref-queries", type=int, default=32)
    ap.add_argument("--exact", action="store_true", help="force the fp64 path")
    args = ap.parse_args()
    rng = np.random.default_rng(11)
    t0 = time.time()
    E = unit_rows(rng, args.docs, args.dim)
    ids = np.arange(args.docs, dtype=np.uint64)
    Q = unit_rows(rng, args.queries, args.dim)
    gen_s = time.time() - t0
    dev = search.DenseIndex(E, ids)
    dev.search_batch(Q[:64], args.k)  # warm-up
    kms, wall = [], []
    for _ in range(args.reps):
        a = time.perf_counter()
        r = dev.search_batch(Q, args.k, flags=search.HM_FLAG_TIMING | (search.HM_FLAG_FORCE_EXACT if args.exact else 0))
        wall.append(time.perf_counter() - a)
        t = search.C.c_float()
        search.lib().hm_dense_last_timing(search.C.byref(t))
        kms.append(t.value)
    k_ms = float(np.median(kms))
    path, overflow, cands = search.DenseIndex.last_stats()
    fma = float(args.docs) * args.dim * args.queries
    out = dict(workload="dense", docs=args.docs, dim=args.dim, queries=args.queries, k=args.k,
               gen_s=round(gen_s, 1), kernel_ms=round(k_ms, 3), kernel_qps=round(args.queries / (k_ms / 1e3), 1),
               api_qps=round(args.queries / float(np.median(wall)), 1),
               path={1: "tcgen05-tf32+fp64-rescore", 2: "fp64", 3: "fp64+sort"}.get(path, path),
               candidates_per_query=round(cands / args.queries, 1), overflowed=overflow,
               effective_tflops=round(2 * fma / (k_ms / 1e3) / 1e12, 2),
               matrix_gb=round(E.nbytes / 1e9, 2))
    try:
        from oracle import ref
        if ref.available():
            R = min(args.ref_queries, args.queries)
            cores = os.cpu_count() or 1
            want = ref.dense_topk_batch(E, ids, Q[:R], args.k, workers=cores)
            ok = bool((want["n"] == r["n"][:R]).all() and (want["ids"] == r["ids"][:R]).all() and
                      (want["scores"].view(np.uint64) == r["scores"][:R].view(np.uint64)).all())
            out["cpu_reference"] = dict(qps=round(R / (want["wall_ms"] / 1e3), 2), cores=cores,
                                        sample=f"first {R} queries, dense_topk, {cores} threads",
                                        parity_bit_identical=ok)
    except Exception as e:
        out["cpu_reference"] = dict(unavailable=str(e))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
