"""The cascade's escalate channel: dense brute-force
top-k (proj/src/dense.cpp:86-101) on the GPU, bit-identical to the reference,
and the fusion / cascade callers around it (fusion.cpp:8-50,
cascade.cpp:44-101) in the Python mirror.

Shapes follow test_dense.cpp (hash_embed matrices with many exact score ties,
1,000 x 32 / 20 x 16 / 50 x 24) plus large random unit-vector matrices; the
cascade test replays acceptance.cpp's criterion-9 structure (BM25 list,
Margin skip, dense list, agent_rrf) against the reference's own functions.
"""
import numpy as np
import pytest

from oracle import ref, restate
from paper_2605_25092_b200 import search


def unit_rows(rng, n, dim):
    x = rng.standard_normal((n, dim)).astype(np.float32)
    return (x / np.linalg.norm(x, axis=1, keepdims=True)).astype(np.float32)


def hash_matrix(n, dim, seed, fmt="doc %d"):
    return np.stack([ref.hash_embed(fmt % d, dim, seed) for d in range(n)])


def assert_dense(got, want, what=""):
    assert (got["n"] == want["n"]).all(), what
    for q in range(len(want["n"])):
        m = int(want["n"][q])
        assert got["ids"][q, :m].tolist() == want["ids"][q, :m].tolist(), (what, q)
        assert (got["scores"][q, :m].view(np.uint64) == want["scores"][q, :m].view(np.uint64)).all(), (what, q)


# ---------------------------------------------------------------- CPU
def test_dense_restatement_matches_reference():
    rng = np.random.default_rng(1)
    for n, dim, seed in ((1000, 32, 7), (20, 16, 1), (50, 24, 5)):
        m = hash_matrix(n, dim, seed)
        ids = rng.permutation(10 * n)[:n].astype(np.uint64)
        q = np.stack([ref.hash_embed(t, dim, seed) for t in ("doc 123 probe", "item 7", "", "doc 5 doc 6")])
        for k in (1, 10, n + 5):
            w = ref.dense_topk_batch(m, ids, q, k)
            i, s, nn = restate.dense_topk(m, ids, q, k)
            assert_dense(dict(ids=i, scores=s, n=nn), w, f"restate {n}x{dim} k={k}")


def test_fusion_mirror_matches_reference():
    rng = np.random.default_rng(2)

    class Rec:
        def __init__(self, ts, w):
            self.ts_ms, self.weight = ts, w

    for trial in range(30):
        pool = rng.permutation(40)[:25]
        sparse = [(int(d), float(s)) for d, s in zip(pool[:10], np.sort(rng.random(10))[::-1])]
        dense = [(int(d), float(s)) for d, s in zip(pool[5:17], np.sort(rng.random(12))[::-1])]
        recs = {int(d): (int(rng.integers(0, 10 ** 7)), float(rng.random())) for d in pool}
        beta = [0.0, 0.3][trial % 2]
        want = ref.agent_rrf(sparse, dense, recs, 5 * 10 ** 6, beta=beta)
        p = search.FusionParams(beta=beta)
        got = search.agent_rrf(sparse, dense, lambda d: Rec(*recs[d]) if d in recs else None, 5 * 10 ** 6, None, p)
        assert [d for d, _ in got] == [d for d, _ in want]
        assert np.array([s for _, s in got]).view(np.uint64).tolist() == \
            np.array([s for _, s in want]).view(np.uint64).tolist()
    with pytest.raises(RuntimeError, match="record missing from lookup: 3"):
        search.agent_rrf([(3, 1.0)], [], lambda d: None, 0, None, search.FusionParams())


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_dense_gpu_bit_identical_on_tied_hash_embeddings(gpu):
    rng = np.random.default_rng(3)
    for n, dim, seed in ((1000, 32, 7), (20, 16, 1), (50, 24, 5), (5000, 30, 9), (3000, 64, 42)):
        m = hash_matrix(n, dim, seed)
        ids = rng.permutation(10 * n)[:n].astype(np.uint64)
        dev = search.DenseIndex(m, ids)
        texts = ["doc %d probe" % int(rng.integers(0, n)) for _ in range(37)] + ["", "doc 1 doc 2 doc 3"]
        q = np.stack([ref.hash_embed(t, dim, seed) for t in texts])
        for k in (1, 3, 10, 100, 256):
            kk = min(k, n)
            want = ref.dense_topk_batch(m, ids, q, kk)
            assert_dense(dev.search_batch(q, kk), want, f"{n}x{dim} k={kk}")
    # a stored vector retrieves itself at score ~1 (test_dense.cpp:88-100)
    m = hash_matrix(20, 16, 1, "item %d")
    r = search.DenseIndex(m, np.arange(20, dtype=np.uint64)).dense_topk(ref.hash_embed("item 7", 16, 1), 1)
    assert r[0][0] == 7 and abs(r[0][1] - 1.0) < 1e-6


@pytest.mark.gpu
def test_dense_tensor_core_path_selects_exactly(gpu):
    """The tcgen05 TF32 candidate path (dim % 32 == 0, k <= 32) against the
    reference and against the fp64 path, with the candidate statistics:
    the selection must be tight (few candidates, no overflow) on random data
    and must still be exact on heavily tied hash embeddings."""
    rng = np.random.default_rng(12)
    for n, dim, nq in ((100_000, 64, 300), (30_001, 128, 77), (5_000, 32, 129), (300, 64, 5)):
        m = unit_rows(rng, n, dim)
        ids = rng.permutation(n).astype(np.uint64) * 3
        dev = search.DenseIndex(m, ids)
        q = unit_rows(rng, nq, dim)
        for k in (1, 10, 32):
            want = ref.dense_topk_batch(m, ids, q, min(k, n), workers=16)
            got = dev.search_batch(q, min(k, n), flags=search.HM_FLAG_TIMING)
            path, overflow, cands = search.DenseIndex.last_stats()
            assert path == 1, path
            assert_dense(got, want, f"tc {n}x{dim} k={k}")
            # each row slab starts its own bound: at most ~k per slab plus the band
            assert overflow == 0 and cands < nq * (160 * k + 512), (overflow, cands)
            exact = dev.search_batch(q, min(k, n), flags=search.HM_FLAG_FORCE_EXACT)
            assert search.DenseIndex.last_stats()[0] == 2
            assert_dense(exact, want, f"fp64 {n}x{dim} k={k}")
    # ties: duplicate-heavy hash embeddings (overflowing lists fall back to a full rescoring)
    m = np.concatenate([hash_matrix(2000, 32, 3, "w%d")] * 6)
    m[1000:11000] = m[7]
    ids = np.arange(len(m), dtype=np.uint64)
    dev = search.DenseIndex(m, ids)
    q = np.stack([m[7], m[8], ref.hash_embed("w7 w8", 32, 3)])
    want = ref.dense_topk_batch(m, ids, q, 10)
    assert_dense(dev.search_batch(q, 10, flags=search.HM_FLAG_TIMING), want, "tc ties")
    assert search.DenseIndex.last_stats()[1] >= 1  # 10,001 exact ties overflow the candidate list


@pytest.mark.gpu
def test_dense_gpu_large_random_and_errors(gpu):
    rng = np.random.default_rng(4)
    for n, dim in ((200_003, 64), (50_000, 384)):
        m = unit_rows(rng, n, dim)
        m[100:110] = m[5]  # exact duplicates: ties broken by DocId
        ids = rng.permutation(n).astype(np.uint64) + 1000
        dev = search.DenseIndex(m, ids)
        q = unit_rows(rng, 300, dim)
        q[0] = m[5]
        want = ref.dense_topk_batch(m, ids, q, 10, workers=16)
        assert_dense(dev.search_batch(q, 10), want, f"random {n}x{dim}")
    with pytest.raises(ValueError, match="query dimension mismatch"):
        dev.search_batch(np.zeros((1, 32), np.float32), 5)
    # k beyond the shared-memory lists: the sort path, same bits
    want = ref.dense_topk_batch(m, ids, q[:3], 1000, workers=16)
    assert_dense(dev.search_batch(q[:3], 1000), want, "large k")


@pytest.mark.gpu
def test_cascade_batch_equals_reference_cascade(gpu):
    """Per query: reference bm25_topk_maxscore -> Margin -> skip at tau, else
    reference dense_topk + agent_rrf, truncated to k (cascade.cpp:44-101);
    ours: one GPU BM25 batch, one GPU dense batch over the escalated queries."""
    from _util import export_to_csr
    corpus = ref.RefCorpus(20000, vocab_size=2000)
    ri = ref.RefIndex.from_corpus(corpus, tok_mode=ref.TOK_MINIMAL)
    csr = export_to_csr(ri)
    queries = ref.RefQueries(corpus, n_queries=300)
    ids, ts, texts = corpus.export()
    dim = 64
    emb = np.stack([ref.hash_embed(t, dim, 42) for t in texts])
    dense = search.DenseIndex(emb, ids)
    qv = np.stack([ref.hash_embed(" ".join(t), dim, 42) for t in queries.terms])
    qts = queries.ts

    class Rec:
        def __init__(self, ts_ms):
            self.ts_ms, self.weight = ts_ms, 0.0

    by_id = {int(i): Rec(int(t)) for i, t in zip(ids, ts)}
    got = search.cascade_batch(csr, dense, queries.terms, qv, 10, by_id.get, qts)
    recs = {int(i): (int(t), 0.0) for i, t in zip(ids, ts)}
    n_esc = 0
    for i, q in enumerate(queries.terms):
        w_ids, w_sc, _ = ri.search(q, 10, maxscore=True)
        sparse = list(zip(w_ids.tolist(), w_sc.tolist()))
        conf = ref.confidence(w_sc)
        assert got[i].confidence == conf
        if conf >= 0.10:
            assert not got[i].escalated and got[i].results == sparse
            continue
        n_esc += 1
        d = ref.dense_topk_batch(emb, ids, qv[i:i + 1], 10)
        dl = list(zip(d["ids"][0, :d["n"][0]].tolist(), d["scores"][0, :d["n"][0]].tolist()))
        want = ref.agent_rrf(sparse, dl, recs, int(qts[i]))[:10]
        assert got[i].escalated and got[i].results == want, i
    assert n_esc > 10


@pytest.mark.gpu
def test_dense_gpu_degenerate_matrices(gpu):
    """Single row, fewer rows than k, zero query, all-equal rows (every score
    tied: DocId order), on both the tensor-core and fp64 paths."""
    for dim in (32, 24):
        one = search.DenseIndex(np.ones((1, dim), np.float32) / np.sqrt(dim), np.array([42], np.uint64))
        assert [d for d, _ in one.dense_topk(np.ones(dim, np.float32), 10)] == [42]
        m = np.tile(np.linspace(-1, 1, dim, dtype=np.float32), (700, 1))
        ids = (np.arange(700, dtype=np.uint64) * 7919) % 1009
        dev = search.DenseIndex(m, ids)
        q = np.stack([np.zeros(dim, np.float32), m[0]])
        for flags in (0, search.HM_FLAG_FORCE_EXACT):
            got = dev.search_batch(q, 10, flags=flags)
            want = ref.dense_topk_batch(m, ids, q, 10)
            assert_dense(got, want, f"ties dim={dim} flags={flags}")


@pytest.mark.gpu
def test_dense_tensor_core_batches_larger_than_a_launch(gpu):
    """More queries than one tensor-core launch takes (16,384): chunked."""
    rng = np.random.default_rng(21)
    m = unit_rows(rng, 1500, 32)
    ids = rng.permutation(1500).astype(np.uint64)
    q = unit_rows(rng, 16_500, 32)
    dev = search.DenseIndex(m, ids)
    got = dev.search_batch(q, 5, flags=search.HM_FLAG_TIMING)
    assert search.DenseIndex.last_stats()[:2] == (1, 0)
    assert_dense(got, ref.dense_topk_batch(m, ids, q, 5, workers=16), "chunked")
