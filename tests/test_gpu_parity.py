"""GPU parity: the CUDA path through the C ABI vs the oracle / the reference.

Bar: bit-identical ids, score bits, counts, Margin confidence, skip decision
and postings_touched (stricter than north_star's 1e-5 relative tolerance).
Mirrors proj/tests/test_csr.cpp, test_cascade.cpp and acceptance.cpp:144-208.
"""
import threading

import numpy as np
import pytest

from _util import (assert_same, check_batch, export_to_csr, random_instance, ref, restate,
                   search, synth_setup, toy_docs)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1(gpu):
    """BASELINE config 1: 100K Zipf docs (V=5000, 5-30 tokens), 1K queries, k=10."""
    corpus, queries, hx, tids = synth_setup(100000, 5000, 5, 30, 1000)
    dev = search.DeviceIndex.from_host(hx)
    orc = restate.OracleIndex.from_host(hx)
    return dict(corpus=corpus, queries=queries, hx=hx, tids=tids, dev=dev, orc=orc)


def test_c1_bit_identical_to_oracle(c1):
    got = c1["dev"].search_lists(c1["tids"], 10)
    ids, sc, n, post = c1["orc"].topk(c1["tids"], 10)
    check_batch(got, ids, sc, n, post, what="C1")
    # nDCG@10 (exponential gain, qrels = gold) identical -> within 0.0002
    q = c1["queries"]
    d_got = np.mean([restate.ndcg(got["ids"][i, :got["n"][i]], {int(q.gold[i]): 1}, 10)
                     for i in range(len(q))])
    d_orc = np.mean([restate.ndcg(ids[i, :n[i]], {int(q.gold[i]): 1}, 10) for i in range(len(q))])
    assert abs(d_got - d_orc) <= 2e-4


def test_c1_matches_reference_library(c1):
    """Against the reference's own bm25_topk and bm25_topk_maxscore on the same index."""
    hx, q = c1["hx"], c1["queries"]
    ri = ref.RefIndex.from_arrays(hx.term_strings(), hx.term_offsets, hx.posting_rows,
                                  hx.posting_tf.astype(np.float64), hx.idf, hx.maxscore,
                                  hx.order_key, hx.doc_lens, hx.doc_ids, hx.avgdl)
    sub = list(range(0, len(q), 7))
    got = c1["dev"].search_lists([c1["tids"][i] for i in sub], 10)
    for j, i in enumerate(sub):
        for ms in (False, True):
            ids, sc, post = ri.search(q.terms(i), 10, maxscore=ms)
            m = got["n"][j]
            assert_same(got["ids"][j, :m], got["scores"][j, :m], ids, sc, f"ref q{i} ms={ms}")
            if not ms:
                assert got["postings"][j] == post


@pytest.mark.parametrize("k", [1, 3, 100, 256])
def test_c1_other_k(c1, k):
    tids = c1["tids"][:300]
    got = c1["dev"].search_lists(tids, k)
    ids, sc, n, post = c1["orc"].topk(tids, k)
    check_batch(got, ids, sc, n, post, what=f"k={k}")


@pytest.mark.parametrize("k1,b", [(0.9, 0.4), (2.0, 1.0), (1.2, 0.0), (0.0, 0.75)])
def test_c1_other_params(c1, k1, b):
    tids = c1["tids"][:200]
    got = c1["dev"].search_lists(tids, 10, k1=k1, b=b)
    ids, sc, n, post = c1["orc"].topk(tids, 10, k1=k1, b=b)
    check_batch(got, ids, sc, n, post, what=f"k1={k1} b={b}")


@pytest.mark.parametrize("k1,b", [(1.2, 1.5), (1.2, -0.5)])
def test_params_outside_unit_b_use_exact_kernel(c1, k1, b):
    tids = c1["tids"][:64]
    got = c1["dev"].search_lists(tids, 10, k1=k1, b=b)
    assert got["n_exact"] == len(tids)
    ids, sc, n, post = c1["orc"].topk(tids, 10, k1=k1, b=b)
    check_batch(got, ids, sc, n, post, what=f"exact k1={k1} b={b}")


def test_forced_exact_kernel_identical(c1):
    tids = c1["tids"][:300]
    fast = c1["dev"].search_lists(tids, 10)
    exact = c1["dev"].search_lists(tids, 10, flags=search.HM_FLAG_FORCE_EXACT)
    assert exact["n_exact"] == len(tids)
    for key in ("ids", "scores", "n", "conf", "skip", "postings"):
        assert (fast[key] == exact[key]).all(), key


def test_duplicate_and_unknown_terms(c1):
    base = c1["tids"][:100]
    tids = [np.concatenate([t, t[:1], [search.NO_TERM], t[-1:]]) for t in base]
    got = c1["dev"].search_lists(tids, 10)
    ids, sc, n, post = c1["orc"].topk(tids, 10)
    check_batch(got, ids, sc, n, post, what="mult")


def test_per_query_tau(c1):
    tids = c1["tids"][:128]
    tau = np.linspace(0.0, 0.5, len(tids))
    got = c1["dev"].search_lists(tids, 10, tau=tau)
    ids, sc, n, _ = c1["orc"].topk(tids, 10)
    for i in range(len(tids)):
        conf = restate.margin(sc[i, :n[i]])
        assert bool(got["skip"][i]) == (conf >= tau[i])


def test_empty_and_k0(c1):
    got = c1["dev"].search_lists([[], [search.NO_TERM]], 10)
    assert (got["n"] == 0).all() and (got["conf"] == 0).all() and (got["skip"] == 0).all()
    got = c1["dev"].search_lists(c1["tids"][:5], 0)
    assert (got["n"] == 0).all()
    got = c1["dev"].search_lists(c1["tids"][:5], 10, tau_default=0.0)
    assert (got["skip"] == 1).all()  # tau = 0 => always skip (test_cascade.cpp:93-115)


def test_batch_composition_and_concurrency(c1):
    tids = c1["tids"][:200]
    full = c1["dev"].search_lists(tids, 10)
    single = [c1["dev"].search_lists([t], 10) for t in tids[:20]]
    for i, s in enumerate(single):
        for key in ("ids", "scores", "n", "conf"):
            assert (s[key][0] == full[key][i]).all()
    outs = [None] * 4

    def run(j):
        outs[j] = c1["dev"].search_lists(tids, 10)

    th = [threading.Thread(target=run, args=(j,)) for j in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for o in outs:
        for key in ("ids", "scores", "n", "conf", "skip"):
            assert (o[key] == full[key]).all()


def test_concurrent_batches_with_different_params(c1):
    """Batches with different Bm25Params from concurrent threads: each (k1, b)
    needs its own baked postings (bake.cu); the index re-bakes under an
    exclusive lock while same-parameter batches share it.  Every result must
    still be the oracle's for its own parameters."""
    tids = c1["tids"][:150]
    params = [(1.2, 0.75), (0.9, 0.4), (1.2, 0.75), (2.0, 1.0)]
    want = {p: c1["orc"].topk(tids, 10, k1=p[0], b=p[1]) for p in set(params)}
    errs = []

    def run(p):
        try:
            for _ in range(3):
                got = c1["dev"].search_lists(tids, 10, k1=p[0], b=p[1])
                ids, sc, n, post = want[p]
                check_batch(got, ids, sc, n, post, what=f"concurrent k1={p[0]} b={p[1]}")
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=run, args=(p,)) for p in params]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs[0]


@pytest.mark.parametrize("k", [1, 10, 100])
def test_c1_seeded_everything_identical(c1, k):
    """HM_FLAG_SEED_ALL: the seeded MaxScore pre-pass (search_seed.cu) serves
    every query that has a short term -- seeds, essential candidates and the
    hand-over to the exhaustive kernel must not change a single bit."""
    got = c1["dev"].search_lists(c1["tids"], k, flags=search.HM_FLAG_SEED_ALL)
    ids, sc, n, post = c1["orc"].topk(c1["tids"], k)
    check_batch(got, ids, sc, n, post, what=f"C1 seeded k={k}")


@pytest.mark.parametrize("k1,b", [(0.9, 0.4), (2.0, 1.0)])
def test_c1_seeded_other_params(c1, k1, b):
    tids = c1["tids"][:300]
    got = c1["dev"].search_lists(tids, 10, k1=k1, b=b, flags=search.HM_FLAG_SEED_ALL)
    ids, sc, n, post = c1["orc"].topk(tids, 10, k1=k1, b=b)
    check_batch(got, ids, sc, n, post, what=f"seeded k1={k1} b={b}")


def test_c1_exhaustive_only_identical(c1):
    got = c1["dev"].search_lists(c1["tids"], 10, flags=search.HM_FLAG_EXHAUSTIVE)
    ids, sc, n, post = c1["orc"].topk(c1["tids"], 10)
    check_batch(got, ids, sc, n, post, what="C1 exhaustive only")


def test_sentinel_reset_is_load_bearing(c1):
    """Pitfall 3 (test_twophase.cpp:66-83): without the
    per-query reset of the candidate state, stale entries of the previous query
    contaminate the next one."""
    heavy = max(range(len(c1["tids"])), key=lambda i: len(c1["tids"][i]))
    tids = [c1["tids"][heavy] if i % 2 == 0 else c1["tids"][i % len(c1["tids"])] for i in range(2000)]
    ids, sc, n, _ = c1["orc"].topk(tids, 10)
    good = c1["dev"].search_lists(tids, 10)
    check_batch(good, ids, sc, n, what="reset on")
    bad = c1["dev"].search_lists(tids, 10, flags=search.HM_FLAG_DEBUG_NO_RESET | search.HM_FLAG_EXHAUSTIVE)
    differs = any(bad["n"][i] != n[i] or (bad["ids"][i, :n[i]] != ids[i, :n[i]]).any()
                  for i in range(len(tids)))
    assert differs, "disabling the reset should contaminate results"


def test_random_instances_vs_reference(gpu):
    """test_csr.cpp:162-176 shape: random tiny corpora, reference build_index +
    reference bm25_topk as the oracle."""
    rng = np.random.default_rng(1234)
    for trial in range(150):
        docs, q = random_instance(rng)
        ri = ref.RefIndex.from_texts(docs, ref.TOK_MINIMAL)
        idx = export_to_csr(ri)
        k = 1 + int(rng.integers(0, 10))
        want_ids, want_sc, want_post = ri.search(q, k)
        stats = search.SearchStats()
        got = idx.bm25_topk(q, k, stats=stats)
        assert_same([g[0] for g in got], [g[1] for g in got], want_ids, want_sc, f"trial {trial}")
        assert stats.postings_touched == want_post
        got = idx.bm25_topk(q, k, flags=search.HM_FLAG_SEED_ALL)
        assert_same([g[0] for g in got], [g[1] for g in got], want_ids, want_sc, f"trial {trial} seeded")


def test_toy_corpus_known_answers(gpu):
    ri = ref.RefIndex.from_texts(toy_docs(), ref.TOK_MINIMAL)
    idx = export_to_csr(ri)
    assert idx.bm25_topk(["unicorn"], 5) == []
    allc = idx.bm25_topk(["cat"], 100)
    assert len(allc) == 4 and all(s > 0 for _, s in allc)
    assert len(idx.bm25_topk(["cat", "dog"], 5)) == 5
    for q in (["cat"], ["cat", "dog"], ["fish", "cat", "cat"], ["dog", "z00"]):
        want_ids, want_sc, _ = ri.search(q, 5)
        got = idx.bm25_topk(q, 5)
        assert_same([g[0] for g in got], [g[1] for g in got], want_ids, want_sc, str(q))


def test_empty_index(gpu):
    ri = ref.RefIndex.from_texts([], ref.TOK_MINIMAL)
    idx = export_to_csr(ri)
    assert idx.bm25_topk(["cat"], 5) == []


def test_repeated_batches_replay_a_cuda_graph(c1):
    """A batch repeated on a workspace is captured into a CUDA graph on its
    second run and replayed afterwards; results stay the oracle's, and a
    changed argument (k, parameters, window) falls back to a fresh sequence."""
    tids = c1["tids"][:300]
    ids, sc, n, post = c1["orc"].topk(tids, 10)
    modes = []
    for _ in range(4):
        got = c1["dev"].search_lists(tids, 10)
        modes.append(search.last_graph())
        check_batch(got, ids, sc, n, post, what="graph replay")
    assert modes[-2:] == [2, 2] and 1 in modes, modes
    i5, s5, n5, p5 = c1["orc"].topk(tids, 5)
    got = c1["dev"].search_lists(tids, 5)
    assert search.last_graph() == 0
    check_batch(got, i5, s5, n5, p5, what="new k after replay")
    for _ in range(3):
        got = c1["dev"].search_lists(tids, 10, k1=0.9, b=0.4)
    w = c1["orc"].topk(tids, 10, k1=0.9, b=0.4)
    check_batch(got, *w, what="other params, replayed")


@pytest.mark.parametrize("nq,k", [(1, 10), (3, 1), (17, 10), (60, 100), (140, 5)])
def test_small_batches_split_into_row_slabs(c1, nq, k):
    """Small batches run each query as row-slab queries (intra-query
    parallelism) merged like doc shards: ids, score bits, conf, skip and
    postings equal the oracle and the unsplit run, with and without a row
    window and for other BM25 parameters."""
    tids = c1["tids"][5:5 + nq]
    n_docs = len(c1["hx"].doc_ids)
    for (lo, hi), (k1, b) in [((0, 0), (1.2, 0.75)), ((1234, n_docs - 777), (1.2, 0.75)), ((0, 0), (0.9, 0.4))]:
        w = c1["orc"].topk(tids, k, k1=k1, b=b, row_lo=lo, row_hi=hi if hi else n_docs)
        got = c1["dev"].search_lists(tids, k, k1=k1, b=b, row_lo=lo, row_hi=hi)
        check_batch(got, *w, what=f"split nq={nq} k={k} window=({lo},{hi})")
        ref_run = c1["dev"].search_lists(tids, k, k1=k1, b=b, row_lo=lo, row_hi=hi, flags=search.HM_FLAG_NO_SPLIT)
        for key in ("ids", "scores", "n", "conf", "skip", "postings"):
            assert (np.asarray(got[key]).view(np.uint8) == np.asarray(ref_run[key]).view(np.uint8)).all(), key


def test_seed_term_tied_with_another_term(gpu):
    """Two terms that always appear together (same df, same max impact) tie on
    the MaxScore bound.  The seeded pass picks the first as its seed t*; the
    bound-ascending prefix may then cover t* but not its twin, and the seed
    rows reached again through the twin's postings must still be recognised
    as seen (duplicates in the top-k otherwise).  The reference's
    bm25_topk / bm25_topk_maxscore on its own build are the oracle."""
    rng = np.random.default_rng(99)
    docs = []
    for d in range(3000):
        words = ["f%d" % int(rng.integers(0, 400)) for _ in range(5)]
        if d % 50 == 7:
            words[:2] = ["qa", "qb"]          # 60 docs: the twins, always together
        if d % 3 == 0:
            words[4] = "cc"                   # a frequent third term, lower bound
        docs.append((d, " ".join(words)))
    ri = ref.RefIndex.from_texts(docs, ref.TOK_MINIMAL)
    idx = export_to_csr(ri)
    for q in (["qa", "qb", "cc"], ["qb", "qa"], ["cc", "qa", "qb", "f3"]):
        for k in (1, 10, 50):
            want_ids, want_sc, _ = ri.search(q, k)
            for flags in (0, search.HM_FLAG_SEED_ALL):
                got = idx.bm25_topk(q, k, flags=flags)
                ids = [g[0] for g in got]
                assert len(set(ids)) == len(ids), f"{q} k={k}: duplicate DocIds {ids}"
                assert_same(ids, [g[1] for g in got], want_ids, want_sc, f"{q} k={k} flags={flags}")


@pytest.mark.parametrize("k", [257, 1000, 5000])
def test_k_above_256_wide_path(c1, k):
    """The reference's bm25_topk takes any k (csr_index.hpp:72-79; collect_topk
    has no cap, csr_index.cpp:50-59): k > 256 runs on the wide path
    (kernels/wide.cu) -- bit-identical ids, scores, counts, conf, skip and
    postings, including queries with fewer than k positive documents and a
    row window."""
    tids = c1["tids"][:40]
    got = c1["dev"].search_lists(tids, k)
    assert search.last_wide() == len(tids)
    ids, sc, n, post = c1["orc"].topk(tids, k)
    check_batch(got, ids, sc, n, post, what=f"wide k={k}")
    n_docs = len(c1["hx"].doc_ids)
    got = c1["dev"].search_lists(tids, k, row_lo=777, row_hi=n_docs - 12345, k1=0.9, b=0.4)
    w = c1["orc"].topk(tids, k, row_lo=777, row_hi=n_docs - 12345, k1=0.9, b=0.4)
    check_batch(got, *w, what=f"wide k={k} window")


def test_more_than_256_distinct_terms(c1):
    """make_plan accepts any query length (csr_index.cpp:31-48): plans of more
    than 256 distinct terms are served by the wide path inside an ordinary
    batch; the other queries of the batch keep the fast kernels."""
    rng = np.random.default_rng(5)
    V = len(c1["hx"].idf)
    longq = [rng.choice(V, size=n, replace=False).astype(np.uint32) for n in (257, 300, 1000)]
    longq.append(np.concatenate([longq[0], longq[0][:50], [search.NO_TERM] * 3]).astype(np.uint32))
    tids = list(c1["tids"][:30]) + longq + list(c1["tids"][30:60])
    for k in (10, 100):
        got = c1["dev"].search_lists(tids, k)
        assert search.last_wide() == 4
        ids, sc, n, post = c1["orc"].topk(tids, k)
        check_batch(got, ids, sc, n, post, what=f"long plans k={k}")
    got = c1["dev"].search_lists(longq, 10, tau=np.full(len(longq), 0.0))
    assert (got["skip"] == 1).all()


def test_many_ties_at_the_kth_score(gpu):
    """A single-term query over documents with equal (tf, len) ties on its
    score everywhere: the k-th document is decided by DocId alone
    (types.hpp:21-25).  DocIds run against the row order."""
    docs = [(10_000 - d, " ".join(["aa"] + ["z%d" % (d % 7)] * 4)) for d in range(3000)]
    ri = ref.RefIndex.from_texts(docs, ref.TOK_MINIMAL)
    idx = export_to_csr(ri)
    for k in (5, 256, 300, 2999, 3000, 4000):
        want_ids, want_sc, _ = ri.search(["aa"], k)
        got = idx.bm25_topk(["aa"], k)
        assert_same([g[0] for g in got], [g[1] for g in got], want_ids, want_sc, f"ties k={k}")


@pytest.mark.parametrize("k", [10, 300])
def test_search_parts_equal_per_window_search(c1, k):
    """hm_search_batch_parts: each (query, part) list equals the oracle's search
    restricted to that row range -- including an empty part, a part inside
    one tile, and parts cut mid-tile (the temporal drop-in's partitions)."""
    tids = c1["tids"][:150]
    N = len(c1["hx"].doc_ids)
    parts = np.array([0, 1000, 1000, 1500, 30000, 77777, N], np.uint32)
    off = np.zeros(len(tids) + 1, np.uint32)
    off[1:] = np.cumsum([len(t) for t in tids])
    got = c1["dev"].search_parts(off, np.concatenate(tids).astype(np.uint32), k, parts)
    for p in range(len(parts) - 1):
        ids, sc, n, post = c1["orc"].topk(tids, k, row_lo=int(parts[p]), row_hi=int(parts[p + 1]))
        assert (got["n"][p] == n).all(), p
        assert (got["postings"][p] == post).all(), p
        for i in range(len(tids)):
            m = int(n[i])
            assert_same(got["ids"][p, i, :m], got["scores"][p, i, :m], ids[i, :m], sc[i, :m], f"part {p} q{i}")
