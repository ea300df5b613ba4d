"""Randomised parity fuzzing of every GPU channel against the reference
(oracle/_ref) -- test infrastructure, run on the GPU box:

    python tools/fuzz.py [seconds]

BM25 (random corpora, k1/b, k, row windows, duplicate/unknown terms),
learned-sparse bridge (random vectors, quantised weights for ties), dense
(tensor-core and fp64 paths, duplicated rows), doc-sharded search (2-8 shards,
the bound exchange, windows).  Stops at the first mismatch
with the failing case printed."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle import ref, restate  # noqa: E402
from paper_2605_25092_b200 import search  # noqa: E402


def same(a_ids, a_sc, a_n, b_ids, b_sc, b_n, what):
    assert (np.asarray(a_n) == np.asarray(b_n)).all(), what
    for q in range(len(b_n)):
        m = int(b_n[q])
        assert np.asarray(a_ids)[q, :m].tolist() == np.asarray(b_ids)[q, :m].tolist(), (what, q)
        assert (np.asarray(a_sc)[q, :m].view(np.uint64) == np.asarray(b_sc)[q, :m].view(np.uint64)).all(), (what, q)


def fuzz_bm25(rng):
    n = int(rng.integers(5, 3000)) if rng.random() < 0.8 else int(rng.integers(20000, 120000))
    V = int(rng.integers(3, 400)) if n < 5000 else int(rng.integers(500, 5000))
    docs = [(int(d), " ".join("t%d" % rng.integers(0, V) for _ in range(rng.integers(1, 25))))
            for d in rng.permutation(n * 3)[:n]]
    ri = ref.RefIndex.from_texts(docs, ref.TOK_MINIMAL)
    e = ri.export()
    csr = search.CsrIndex(e["terms"], e["term_offsets"], e["posting_rows"], e["posting_weights"], e["idf"],
                          e["order_key"], e["doc_lens"], e["doc_ids"], e["avgdl"])
    k1 = float(rng.choice([1.2, 0.5, 2.0, 0.9]))
    b = float(rng.choice([0.75, 0.0, 1.0, 0.3]))
    k = int(rng.integers(1, 40))
    qs = [["t%d" % rng.integers(0, V + 5) for _ in range(rng.integers(1, 8))] for _ in range(int(rng.integers(1, 60)))]
    flags = int(rng.choice([0, search.HM_FLAG_SEED_ALL, search.HM_FLAG_NE_ALL, search.HM_FLAG_NE_ALL,
                               search.HM_FLAG_EXHAUSTIVE, search.HM_FLAG_FORCE_EXACT]))
    lo = hi = 0
    if rng.random() < 0.3:  # a row window (temporal recency / doc shard)
        lo = int(rng.integers(0, n))
        hi = int(rng.integers(lo, n + 1))
    got = csr.search_batch(qs, k, search.Bm25Params(k1, b), flags=flags, row_lo=lo, row_hi=hi)
    if lo or hi:
        orc = restate.OracleIndex(e["term_offsets"], e["posting_rows"], e["posting_weights"], e["idf"],
                                  e["order_key"], e["doc_lens"], e["doc_ids"], e["avgdl"])
        w = orc.topk([csr.resolve(q) for q in qs], k, k1=k1, b=b, row_lo=lo, row_hi=hi if hi else n)
        same(got["ids"], got["scores"], got["n"], w[0], w[1], w[2], ("bm25 window", n, V, k1, b, k, lo, hi, flags))
        assert (got["postings"] == w[3]).all(), ("bm25 window postings", lo, hi)
        return
    for i, q in enumerate(qs):
        w_ids, w_sc, w_post = ri.search(q, k, k1=k1, b=b)
        same(got["ids"][i:i + 1], got["scores"][i:i + 1], got["n"][i:i + 1], [w_ids], [w_sc], [len(w_ids)],
             ("bm25", n, V, k1, b, k, q, flags))
        assert int(got["postings"][i]) == w_post, ("bm25 postings", q)
        assert got["conf"][i] == ref.confidence(w_sc), ("bm25 conf", q)


def fuzz_bridge(rng):
    n = int(rng.integers(1, 20000))
    V = int(rng.integers(2, 600))
    dens = float(rng.choice([0.002, 0.01, 0.05]))
    vecs = []
    for _ in range(n):
        idx = np.nonzero(rng.random(V) < dens)[0].astype(np.uint32)
        w = 0.05 + rng.random(len(idx)) * 3.0
        if rng.random() < 0.5:
            w = np.round(w * 2) / 2 + 0.5  # ties
        vecs.append((idx, w))
    ids = rng.permutation(n * 2)[:n].astype(np.uint64)
    rb = ref.RefBridge.from_vectors(ids, vecs)
    bi = search.bridge_ingest([(int(d), search.SparseVector(i, v)) for d, (i, v) in zip(ids, vecs)])
    qs = []
    for _ in range(int(rng.integers(1, 50))):
        idx = np.nonzero(rng.random(V + 10) < float(rng.choice([0.01, 0.1, 0.5])))[0].astype(np.uint32)
        qs.append((idx, 0.1 + np.round(rng.random(len(idx)) * 4) / 4))
    k = int(rng.integers(0, 513))
    want = rb.topk_batch(qs, k)
    got = bi.search_batch([search.SparseVector(i, v) for i, v in qs], k)
    if k:
        same(got["ids"], got["scores"], got["n"], want["ids"], want["scores"], want["n"], ("bridge", n, V, k))
    assert (got["postings"] == want["postings"]).all(), "bridge postings"


def fuzz_dense(rng):
    n = int(rng.integers(1, 60000))
    dim = int(rng.choice([8, 24, 32, 64, 96, 128, 30]))
    m = rng.standard_normal((n, dim)).astype(np.float32)
    if rng.random() < 0.5:
        m = np.round(m * 2) / 2  # many exact ties
    if rng.random() < 0.3 and n > 10:
        m[rng.integers(0, n, n // 3)] = m[0]
    ids = rng.permutation(n * 2)[:n].astype(np.uint64)
    dev = search.DenseIndex(m, ids)
    nq = int(rng.integers(1, 300))
    q = rng.standard_normal((nq, dim)).astype(np.float32)
    k = int(min(n, rng.choice([1, 5, 10, 32, 100, 300])))
    flags = int(rng.choice([0, search.HM_FLAG_FORCE_EXACT]))
    want = ref.dense_topk_batch(m, ids, q, k, workers=16)
    got = dev.search_batch(q, k, flags=flags)
    same(got["ids"], got["scores"], got["n"], want["ids"], want["scores"], want["n"],
         ("dense", n, dim, k, flags, search.DenseIndex.last_stats()))


def fuzz_sharded(rng):
    """Doc-sharded search behind the C ABI (hm_sharded_*): 2-8 shards of a
    random corpus on cuda:0, batches large enough for the shards' bound
    exchange (and small ones without it), the seeded pass forced or not,
    row windows -- against the reference library query by query."""
    n = int(rng.integers(2000, 60000))
    V = int(rng.integers(50, 3000))
    docs = [(int(d), " ".join("t%d" % min(V - 1, int(rng.zipf(1.3)) - 1) for _ in range(rng.integers(1, 30))))
            for d in rng.permutation(n * 3)[:n]]
    ri = ref.RefIndex.from_texts(docs, ref.TOK_MINIMAL)
    e = ri.export()
    G = int(rng.integers(2, 9))
    sh = search.ShardedDeviceIndex(e["term_offsets"], e["posting_rows"], e["idf"], e["order_key"], e["doc_lens"],
                                   e["doc_ids"], e["avgdl"], [0] * G, posting_weights=e["posting_weights"])
    vocab = {t: i for i, t in enumerate(e["terms"])}
    nq = int(rng.choice([int(rng.integers(1, 40)), int(rng.integers(256, 600))]))
    qs = [["t%d" % min(V + 3, int(rng.zipf(1.3)) - 1) for _ in range(rng.integers(1, 7))] for _ in range(nq)]
    tids = [[vocab.get(t, 0xFFFFFFFF) for t in q] for q in qs]
    off = np.zeros(nq + 1, np.uint32)
    off[1:] = np.cumsum([len(t) for t in tids])
    flat = np.array([x for t in tids for x in t], np.uint32)
    k = int(rng.choice([1, 3, 10, 50, 100]))
    flags = int(rng.choice([0, search.HM_FLAG_SEED_ALL]))
    lo = hi = 0
    if rng.random() < 0.3:
        lo = int(rng.integers(0, n))
        hi = int(rng.integers(lo, n + 1))
    got = sh.search_batch(off, flat, k, flags=flags, row_lo=lo, row_hi=hi)
    if lo or hi:
        orc = restate.OracleIndex(e["term_offsets"], e["posting_rows"], e["posting_weights"], e["idf"],
                                  e["order_key"], e["doc_lens"], e["doc_ids"], e["avgdl"])
        w = orc.topk(tids, k, row_lo=lo, row_hi=hi if hi else n)
        same(got["ids"], got["scores"], got["n"], w[0], w[1], w[2], ("sharded window", n, V, G, k, lo, hi, flags))
        return
    for i, q in enumerate(qs):
        w_ids, w_sc, w_post = ri.search(q, k)
        same(got["ids"][i:i + 1], got["scores"][i:i + 1], got["n"][i:i + 1], [w_ids], [w_sc], [len(w_ids)],
             ("sharded", n, V, G, k, q, flags))
        assert int(got["postings"][i]) == w_post, ("sharded postings", q)


def main():
    budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
    rng = np.random.default_rng(int(time.time()))
    t0 = time.time()
    counts = dict(bm25=0, bridge=0, dense=0, sharded=0)
    while time.time() - t0 < budget:
        which = rng.choice(["bm25", "bridge", "dense", "sharded"])
        {"bm25": fuzz_bm25, "bridge": fuzz_bridge, "dense": fuzz_dense, "sharded": fuzz_sharded}[which](rng)
        counts[which] += 1
    print("fuzz ok:", counts)


if __name__ == "__main__":
    main()
