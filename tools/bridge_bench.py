"""Learned-sparse bridge path: GPU throughput vs the reference CPU
(bridge_topk, src/bridge.cpp:112-137) on a SPLADE-shaped synthetic index.

Workload (synthetic, fixed seed): --docs documents, each with ~--nnz distinct
terms drawn Zipf(1.0) over a --vocab vocabulary (BERT's 30,522 by default),
weights 0.05 + 3u as test_bridge.cpp:15-28; queries take --qnnz terms of a
random document plus a few random terms, weights 0.1 + u.  Algorithmic bytes
per query = sum of the query terms' df x 12 B (u32 row + f64 weight, the
reference layout the kernel streams).

    python tools/bridge_bench.py [--docs 1000000] [--queries 4000] [--ref-queries 200]

Prints one JSON line: GPU kernel / host-API throughput, achieved GB/s against
MEASURED_PEAKS.json, the reference's multi-threaded CPU throughput on a bounded
sample, and a parity check of that sample (ids and score bits).
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


def make_workload(n_docs, vocab, nnz, n_q, qnnz, seed=7):
    rng = np.random.default_rng(seed)
    ranks = np.arange(1, vocab + 1, dtype=np.float64)
    cdf = np.cumsum(1.0 / ranks)
    cdf /= cdf[-1]
    per = int(nnz * 1.15)  # draws per doc (duplicates collapse)
    row = np.repeat(np.arange(n_docs, dtype=np.int64), per)
    tid = np.searchsorted(cdf, rng.random(len(row))).astype(np.int64)
    key = np.unique(row * vocab + tid)  # distinct terms per doc, doc-major sorted
    rows = (key // vocab).astype(np.uint32)
    tids = (key % vocab).astype(np.uint32)
    w = 0.05 + rng.random(len(key)) * 3.0
    order = np.argsort(tids, kind="stable")  # term-major, rows ascending per term
    off = np.zeros(vocab + 1, np.uint64)
    off[1:] = np.cumsum(np.bincount(tids, minlength=vocab))
    doc_lens = np.bincount(rows, minlength=n_docs).astype(np.uint32)
    doc_ids = np.arange(n_docs, dtype=np.uint64)
    avgdl = float(doc_lens.sum()) / n_docs
    dstart = np.concatenate([[0], np.cumsum(doc_lens.astype(np.int64))])
    queries = []
    for _ in range(n_q):
        d = int(rng.integers(0, n_docs))
        own = tids[dstart[d]:dstart[d + 1]]
        pick = rng.choice(own, size=min(qnnz, len(own)), replace=False) if len(own) else own
        extra = rng.integers(0, vocab, size=3)
        idx = np.unique(np.concatenate([pick, extra]).astype(np.uint32))
        queries.append((idx, 0.1 + rng.random(len(idx))))
    return dict(off=off, rows=rows[order], w=w[order], doc_ids=doc_ids, doc_lens=doc_lens, avgdl=avgdl,
                queries=queries)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        for key in ("hbm_gbs", "hbm_gbps"):
            if key in p:
                return float(p[key]), key
    except Exception:
        pass
    return 7672.0, "B200_PROFILING.md fallback"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--docs", type=int, default=1_000_000)
    ap.add_argument("--vocab", type=int, default=30522)
    ap.add_argument("--nnz", type=int, default=100)
    ap.add_argument("--queries", type=int, default=4000)
    ap.add_argument("--qnnz", type=int, default=30)
    ap.add_argument("--k", type=int, default=10)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--ref-queries", type=int, default=200)
    args = ap.parse_args()

    t0 = time.time()
    W = make_workload(args.docs, args.vocab, args.nnz, args.queries, args.qnnz)
    gen_s = time.time() - t0
    df = np.diff(W["off"].astype(np.int64))
    q_post = np.array([int(df[i].sum()) for i, _ in W["queries"]], np.int64)
    off = np.zeros(len(W["queries"]) + 1, np.uint64)
    off[1:] = np.cumsum([len(i) for i, _ in W["queries"]])
    qi = np.concatenate([i for i, _ in W["queries"]]).astype(np.uint32)
    qv = np.concatenate([v for _, v in W["queries"]])

    dev = search.DeviceBridge(W["off"], W["rows"], W["w"], W["doc_ids"])
    for _ in range(2):  # warm-up
        dev.search_arrays(off, qi, qv, args.k, flags=search.HM_FLAG_TIMING)
    kms, wall = [], []
    for _ in range(args.reps):
        a = time.perf_counter()
        r = dev.search_arrays(off, qi, qv, args.k, flags=search.HM_FLAG_TIMING)
        wall.append(time.perf_counter() - a)
        t = search.C.c_float()
        search.lib().hm_bridge_last_timing(search.C.byref(t))
        kms.append(t.value)
    nq = len(W["queries"])
    k_ms = float(np.median(kms))
    bytes_algo = float(q_post.sum()) * 12.0
    peak, peak_src = peaks()
    out = dict(workload="bridge", docs=args.docs, vocab=args.vocab, postings=int(len(W["rows"])),
               queries=nq, k=args.k, mean_query_postings=float(q_post.mean()), gen_s=round(gen_s, 1),
               kernel_ms=round(k_ms, 3), kernel_qps=round(nq / (k_ms / 1e3), 1),
               api_qps=round(nq / float(np.median(wall)), 1),
               roofline=dict(bound="hbm", achieved=round(bytes_algo / (k_ms / 1e3) / 1e9, 1), peak=peak,
                             unit="GB/s", frac=round(bytes_algo / (k_ms / 1e3) / 1e9 / peak, 3),
                             peak_source=peak_src, bytes_per_posting=12))
    try:
        from oracle import ref
        if ref.available():
            R = min(args.ref_queries, nq)
            rb = ref.RefBridge.from_csr(W["off"], W["rows"], W["w"], W["doc_ids"], W["doc_lens"], W["avgdl"])
            cores = os.cpu_count() or 1
            want = rb.topk_batch(W["queries"][:R], args.k, workers=cores)
            ok = bool((want["n"] == r["n"][:R]).all() and (want["ids"] == r["ids"][:R]).all() and
                      (want["scores"].view(np.uint64) == r["scores"][:R].view(np.uint64)).all() and
                      (want["postings"] == r["postings"][:R]).all())
            out["cpu_reference"] = dict(qps=round(R / (want["wall_ms"] / 1e3), 1), cores=cores,
                                        sample=f"first {R} queries, bridge_topk, {cores} threads",
                                        parity_bit_identical=ok)
    except Exception as e:  # the reference library is test infrastructure
        out["cpu_reference"] = dict(unavailable=str(e))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
