"""Learned-sparse bridge scoring (proj/src/bridge.cpp).

The contract (bridge.hpp:28-33): S[doc] += w_q * W_t accumulated per document
in ascending query term-id order, so exact floating-point equality with the
brute-force dot is required (test_bridge.cpp:87-111, acceptance criterion 5 at
acceptance.cpp:232-278), and bridge_topk_maxscore returns the same list.
CPU tests pin the oracle restatement and the host-side ingest/export/validate
mirror against the UNMODIFIED reference (oracle/_ref); GPU tests compare the
device path (kernels/bridge.cu through hm_bridge_*) with the reference bit for
bit.
"""
import threading

import numpy as np
import pytest

from oracle import ref, restate
from paper_2605_25092_b200 import search


def random_vectors(rng, ndocs, vocab, density):
    """Per-doc sparse vectors as test_bridge.cpp:15-28 (0.05 + 3u weights)."""
    out = []
    for _ in range(ndocs):
        idx = np.nonzero(rng.random(vocab) < density)[0].astype(np.uint32)
        out.append((idx, 0.05 + rng.random(len(idx)) * 3.0))
    return out


def random_queries(rng, n, vocab, density, extra_unknown=0):
    qs = []
    for _ in range(n):
        idx = np.nonzero(rng.random(vocab + extra_unknown) < density)[0].astype(np.uint32)
        qs.append((idx, 0.1 + rng.random(len(idx))))
    return qs


def to_sv(qs):
    return [search.SparseVector(i, v) for i, v in qs]


def assert_same(got, want, what=""):
    n = want["n"]
    assert (got["n"] == n).all(), what
    for q in range(len(n)):
        m = int(n[q])
        assert got["ids"][q, :m].tolist() == want["ids"][q, :m].tolist(), (what, q)
        assert (got["scores"][q, :m].view(np.uint64) == want["scores"][q, :m].view(np.uint64)).all(), (what, q)
    assert (got["postings"] == want["postings"]).all(), what


# ---------------------------------------------------------------- CPU
def test_oracle_restatement_matches_reference_bridge():
    rng = np.random.default_rng(21)
    for ndocs, vocab, dens in ((10, 200, 0.05), (1000, 200, 0.05), (3000, 1000, 0.005)):
        docs = random_vectors(rng, ndocs, vocab, dens)
        ids = np.arange(ndocs, dtype=np.uint64) * 3 + 7
        rb = ref.RefBridge.from_vectors(ids, docs)
        ob = restate.OracleBridge.ingest(ids, docs)
        qs = random_queries(rng, 40, vocab, 0.03, extra_unknown=20) + [(np.zeros(0), np.zeros(0))]
        for k in (1, 10, 57):
            want = rb.topk_batch(qs, k)
            pruned = rb.topk_batch(qs, k, maxscore=True)
            i, s, n, p = ob.topk(qs, k)
            assert_same(dict(ids=i, scores=s, n=n, postings=p), want, f"oracle {ndocs} k={k}")
            assert (pruned["n"] == want["n"]).all() and (pruned["ids"] == want["ids"]).all()


def test_ingest_and_export_mirror_the_reference():
    rng = np.random.default_rng(11)
    for ndocs, vocab, dens in ((40, 120, 0.08), (100, 500, 0.02), (7, 30, 0.0)):
        docs = random_vectors(rng, ndocs, vocab, dens)
        ids = rng.permutation(10 * ndocs)[:ndocs].astype(np.uint64)
        want = ref.RefBridge.from_vectors(ids, docs).export()
        got = search.bridge_ingest([(int(d), search.SparseVector(i, v)) for d, (i, v) in zip(ids, docs)])
        assert (got.term_offsets == want["term_offsets"]).all()
        assert (got.posting_rows == want["posting_rows"]).all()
        assert (got.posting_weights.view(np.uint64) == want["posting_weights"].view(np.uint64)).all()
        assert (got.term_maxscores.view(np.uint64) == want["maxscore"].view(np.uint64)).all()
        assert (got.doc_lens == want["doc_lens"]).all() and (got.doc_ids == want["doc_ids"]).all()
        assert np.float64(got.avgdl).view(np.uint64) == np.float64(want["avgdl"]).view(np.uint64)
        back = search.bridge_export(got)  # exact round trip (test_bridge.cpp:69-80)
        for (d, (i, v)), (bd, bv) in zip(zip(ids, docs), back):
            assert bd == int(d) and bv.indices.tolist() == i.tolist() and (bv.values == v).all()


def test_sparse_vector_validation_messages_match_reference():
    cases = [([3, 1], [1.0, 1.0]), ([1, 1], [1.0, 1.0]), ([1, 2], [1.0, 0.0]), ([1, 2], [1.0]),
             ([1, 2], [1.0, float("nan")]), ([1, 2], [0.5, 1.0]), ([], [])]
    for idx, val in cases:
        try:
            ref.sparse_validate(idx, val)
            want = None
        except RuntimeError as e:
            want = str(e)
        try:
            search.SparseVector(idx, val).validate()
            got = None
        except ValueError as e:
            got = str(e)
        assert got == want, (idx, val, got, want)


def test_duplicate_doc_ids_rejected_like_reference():
    docs = [(np.array([1], np.uint32), np.array([1.0])), (np.array([2], np.uint32), np.array([1.0]))]
    with pytest.raises(RuntimeError) as e_ref:
        ref.RefBridge.from_vectors(np.array([3, 3], np.uint64), docs)
    with pytest.raises(RuntimeError) as e_our:
        search.bridge_ingest([(3, search.SparseVector([1], [1.0])), (3, search.SparseVector([2], [1.0]))])
    assert str(e_our.value) == str(e_ref.value) == "duplicate doc id: 3"


def test_reference_refuses_bm25_on_bridge_index():
    rb = ref.RefBridge.from_vectors(np.array([1], np.uint64), [(np.array([0], np.uint32), np.array([1.0]))])
    assert rb.bm25_error() == "BM25 scoring requires a BM25-mode index"


# ---------------------------------------------------------------- GPU
def _dev(ids, docs):
    return search.bridge_ingest([(int(d), search.SparseVector(i, v)) for d, (i, v) in zip(ids, docs)])


@pytest.mark.gpu
def test_bridge_gpu_bit_identical_to_reference(gpu):
    """acceptance criterion 5 (10 / 1,000 / 100,000 docs, vocab 1,000, density
    0.005, queries at 0.01) plus test_bridge.cpp's 200-term shape."""
    rng = np.random.default_rng(5005)
    shapes = [(10, 1000, 0.005, 0.01), (1000, 1000, 0.005, 0.01), (100000, 1000, 0.005, 0.01),
              (10, 200, 0.05, 0.03), (1000, 200, 0.05, 0.03)]
    for ndocs, vocab, dens, qd in shapes:
        docs = random_vectors(rng, ndocs, vocab, dens)
        ids = np.arange(ndocs, dtype=np.uint64)
        rb = ref.RefBridge.from_vectors(ids, docs)
        bi = _dev(ids, docs)
        qs = random_queries(rng, 50, vocab, qd, extra_unknown=10)
        for k in (1, 10, 100, 512):
            want = rb.topk_batch(qs, k)
            got = bi.search_batch(to_sv(qs), k)
            assert_same(got, want, f"{ndocs} docs k={k}")
            pruned = rb.topk_batch(qs, k, maxscore=True)
            assert (pruned["ids"] == want["ids"]).all()


@pytest.mark.gpu
def test_bridge_gpu_edge_cases(gpu):
    # single posting scores w_q * W_t (test_bridge.cpp:55-64)
    bi = search.bridge_ingest([(7, search.SparseVector([3], [1.5]))])
    assert bi.bridge_topk(search.SparseVector([3], [2.0]), 5) == [(7, 2.0 * 1.5)]
    # one-hot query ranks docs by that term's weight (:120-131)
    bi = search.bridge_ingest([(1, search.SparseVector([4], [0.2])), (2, search.SparseVector([4], [0.9])),
                               (3, search.SparseVector([5], [5.0]))])
    assert [d for d, _ in bi.bridge_topk(search.SparseVector([4], [1.0]), 10)] == [2, 1]
    # empty query, only-unknown terms, k = 0 (stats still count), k > n_docs
    st = search.SearchStats()
    assert bi.bridge_topk(search.SparseVector(), 5) == []
    assert bi.bridge_topk(search.SparseVector([9, 100], [1.0, 2.0]), 5, st) == [] and st.postings_touched == 0
    r = bi.search_batch([search.SparseVector([4, 5], [1.0, 1.0])], 0)
    assert r["n"][0] == 0 and r["postings"][0] == 3
    assert len(bi.bridge_topk(search.SparseVector([4, 5], [1.0, 1.0]), 1000)) == 3
    # ties: equal scores rank by DocId ascending
    bi = search.bridge_ingest([(d, search.SparseVector([0], [1.0])) for d in (9, 4, 6, 1, 8)])
    assert [d for d, _ in bi.bridge_topk(search.SparseVector([0], [0.5]), 3)] == [1, 4, 6]
    # invalid query vectors and oversize k
    with pytest.raises(ValueError, match="strictly increasing"):
        bi.search_batch([search.SparseVector([2, 1], [1.0, 1.0])], 5)
    with pytest.raises(ValueError, match="must be > 0"):
        bi.search_batch([search.SparseVector([1], [-1.0])], 5)
    with pytest.raises(ValueError, match="supported maximum"):
        bi.search_batch([search.SparseVector([0], [1.0])], 513)


@pytest.mark.gpu
def test_bridge_gpu_long_queries_windows_and_ties(gpu):
    """Queries longer than the 128 register-resident cursors (the global cursor
    path), row windows against the restatement, quantised weights (many
    exact ties) and DocIds in reverse row order."""
    rng = np.random.default_rng(77)
    ndocs, vocab = 20000, 2000
    docs = random_vectors(rng, ndocs, vocab, 0.01)
    docs = [(i, np.round(v * 4) / 4 + 0.25) for i, v in docs]  # quantised: ties
    ids = (10 ** 6 - np.arange(ndocs)).astype(np.uint64)
    rb = ref.RefBridge.from_vectors(ids, docs)
    ob = restate.OracleBridge.ingest(ids, docs)
    bi = _dev(ids, docs)
    qs = random_queries(rng, 30, vocab, 0.15)  # ~300 terms per query
    qs = [(i, np.round(v * 4) / 4 + 0.25) for i, v in qs]
    assert max(len(i) for i, _ in qs) > 200
    for k in (10, 200):
        assert_same(bi.search_batch(to_sv(qs), k), rb.topk_batch(qs, k), f"long k={k}")
    for lo, hi in ((0, 5000), (4999, 15001), (12345, ndocs), (100, 101)):
        i, s, n, p = ob.topk(qs, 10, row_lo=lo, row_hi=hi)
        assert_same(bi.search_batch(to_sv(qs), 10, row_lo=lo, row_hi=hi),
                    dict(ids=i, scores=s, n=n, postings=p), f"window {lo}:{hi}")


@pytest.mark.gpu
def test_bridge_hidx_file_and_device_batch(gpu, tmp_path):
    """A Bridge-mode HIDX file written by the reference (save_index) uploads
    straight to the device; the device-buffer entry point gives the same bits;
    BM25 on it is refused with the reference's message."""
    import torch
    rng = np.random.default_rng(3)
    docs = random_vectors(rng, 5000, 500, 0.02)
    ids = np.arange(5000, dtype=np.uint64) + 100
    rb = ref.RefBridge.from_vectors(ids, docs)
    p = tmp_path / "b.hidx"
    rb.save(p)
    h = search.Hidx(p)
    assert h.mode == 1
    with pytest.raises(RuntimeError, match="BM25 scoring requires a BM25-mode index"):
        h.device_index()
    dev = h.bridge_index()
    qs = random_queries(rng, 64, 500, 0.02)
    want = rb.topk_batch(qs, 10)
    off, idx, val = ref.sparse_pack(qs)
    assert_same(dev.search_arrays(off, idx, val, 10), want, "hidx")
    nq = len(qs)
    out = dict(ids=torch.zeros((nq, 10), dtype=torch.int64, device="cuda"),
               scores=torch.zeros((nq, 10), dtype=torch.float64, device="cuda"),
               n=torch.zeros(nq, dtype=torch.int32, device="cuda"),
               postings=torch.zeros(nq, dtype=torch.int64, device="cuda"))
    dev.search_batch_device(torch.from_numpy(off.astype(np.int64)).cuda(),
                            torch.from_numpy(idx.astype(np.int32)).cuda(),
                            torch.from_numpy(val).cuda(), out, 10, max_nnz=int(np.diff(off).max()))
    torch.cuda.synchronize()
    got = dict(ids=out["ids"].cpu().numpy().view(np.uint64), scores=out["scores"].cpu().numpy(),
               n=out["n"].cpu().numpy().astype(np.uint32), postings=out["postings"].cpu().numpy().view(np.uint64))
    assert_same(got, want, "device batch")


@pytest.mark.gpu
def test_bridge_concurrent_batches(gpu):
    rng = np.random.default_rng(9)
    docs = random_vectors(rng, 30000, 800, 0.01)
    ids = np.arange(30000, dtype=np.uint64)
    rb = ref.RefBridge.from_vectors(ids, docs)
    bi = _dev(ids, docs)
    qs = random_queries(rng, 100, 800, 0.02)
    want = rb.topk_batch(qs, 10)
    errs = []

    def run():
        try:
            for _ in range(3):
                assert_same(bi.search_batch(to_sv(qs), 10), want, "concurrent")
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=run) for _ in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs[0]


@pytest.mark.gpu
def test_bridge_gpu_degenerate_indexes(gpu):
    """Empty index, no postings, all-unknown queries, k larger than the index."""
    empty = search.bridge_ingest([])
    assert empty.num_docs() == 0
    r = empty.dev.search_batch([search.SparseVector([0], [1.0])], 5)
    assert r["n"][0] == 0 and r["postings"][0] == 0
    nopost = search.bridge_ingest([(5, search.SparseVector()), (6, search.SparseVector())])
    assert nopost.bridge_topk(search.SparseVector([0, 1], [1.0, 2.0]), 3) == []
    one = search.bridge_ingest([(9, search.SparseVector([2], [0.25]))])
    assert one.bridge_topk(search.SparseVector([0, 1, 2, 7], [1.0, 1.0, 4.0, 1.0]), 100) == [(9, 1.0)]


@pytest.mark.gpu
@pytest.mark.parametrize("nq,k", [(1, 10), (7, 3), (40, 50)])
def test_bridge_small_batches_split_into_row_slabs(gpu, nq, k):
    """Small bridge batches run as row-slab queries merged like doc shards:
    identical to the unsplit run and to the reference (ids, bits, postings)."""
    rng = np.random.default_rng(nq * 100 + k)
    docs = random_vectors(rng, 80000, 800, 0.01)
    ids = rng.permutation(200000)[:80000].astype(np.uint64)
    rb = ref.RefBridge.from_vectors(ids, docs)
    bi = _dev(ids, docs)
    qs = random_queries(rng, nq, 800, 0.05)
    want = rb.topk_batch(qs, k)
    got = bi.search_batch(to_sv(qs), k)
    assert_same(got, want, f"split nq={nq} k={k}")
    one = bi.dev.search_batch(to_sv(qs), k, flags=search.HM_FLAG_NO_SPLIT)
    for key in ("ids", "scores", "n", "postings"):
        assert (np.asarray(got[key]).view(np.uint8) == np.asarray(one[key]).view(np.uint8)).all(), key
