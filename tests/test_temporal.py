"""GPU parity of the time-partitioned path (proj/src/temporal_index.cpp:72-169).

Rows are laid out partition by partition; the newest min(k*, kmax, K)
partitions are a row suffix scored by the flat kernel with a row window.
Results must equal the reference's TemporalIndex::topk (greedy most-recent-
first merge of per-partition MaxScore top-k lists) bit for bit.
"""
import json
import os

import numpy as np
import pytest

from _util import assert_same, check_batch, ref, restate, search, synth

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
DAY = 24 * 3600 * 1000


def partition_rows(ts, window_ms):
    """Bucketing of build_temporal_index (temporal_index.cpp:144-157)."""
    ts = np.asarray(ts, np.int64)
    t0 = int(ts.min())
    K = int((ts.max() - t0) // window_ms + 1)
    j = (ts - t0) // window_ms
    order = np.argsort(j, kind="stable").astype(np.uint32)
    part = np.zeros(K + 1, np.uint32)
    part[1:] = np.cumsum(np.bincount(j, minlength=K))
    return order, part


def test_golden_temporal_cases(gpu):
    with open(os.path.join(GOLD, "temporal.json")) as f:
        g = json.load(f)
    ids, ts, texts = g["ids"], g["ts"], g["texts"]
    order, part = partition_rows(ts, 7 * DAY)
    docs = [(ids[r], texts[r]) for r in order]
    ri = ref.RefIndex.from_texts(docs, ref.TOK_MINIMAL)
    e = ri.export()
    idx = search.CsrIndex(e["terms"], e["term_offsets"], e["posting_rows"], e["posting_weights"],
                          e["idf"], e["order_key"], e["doc_lens"], e["doc_ids"], e["avgdl"])
    for case in g["cases"]:
        assert case["partitions"] == len(part) - 1
        assert (np.diff(part) == case["part_docs"]).all()
        params = search.TemporalParams(7 * DAY, case["epsilon"], case["lambda_hat"], case["k_max"])
        tix = search.TemporalIndex(idx.dev(), part, params)
        for qd in case["queries"]:
            tid = idx.resolve(qd["terms"])
            r = tix.topk_batch(np.array([0, len(tid)], np.uint32), np.array(tid, np.uint32), qd["k"])
            n = int(r["n"][0])
            want = np.array([float.fromhex(x) for x in qd["scores"]])
            assert_same(r["ids"][0, :n], r["scores"][0, :n], qd["ids"], want, str(qd))


@pytest.fixture(scope="module")
def c3_small(gpu):
    n = 200000
    span = int(28 * DAY * n / 4052)  # constant arrival rate (acceptance.cpp:101-104)
    corpus = synth.Corpus(n_records=n, time_span_ms=span)
    queries = synth.Queries(corpus, n_queries=1000)
    K, order, part, _ = corpus.partition(7 * DAY)
    hx = synth.HostIndex(corpus, row_order=order)
    dev = search.DeviceIndex.from_host(hx)
    tids = [hx.resolve(queries.term_ranks[queries.offsets[i]:queries.offsets[i + 1]])
            for i in range(len(queries))]
    return dict(corpus=corpus, queries=queries, hx=hx, dev=dev, part=part, tids=tids, span=span)


def test_c3_shape_matches_reference_temporal_index(c3_small):
    c = c3_small
    tix = search.TemporalIndex(c["dev"], c["part"])
    assert tix.budget() == 3
    off = np.zeros(len(c["tids"]) + 1, np.uint32)
    off[1:] = np.cumsum([len(t) for t in c["tids"]])
    got = tix.topk_batch(off, np.concatenate(c["tids"]), 10)
    rc = ref.RefCorpus(200000, time_span_ms=c["span"])
    rt = ref.RefTemporal.from_corpus(rc, tok_mode=ref.TOK_STOPWORD)
    assert rt.partitions()[0].shape[0] == tix.num_partitions()
    for i in range(0, len(c["tids"]), 3):
        ids, sc, searched, _ = rt.topk(c["queries"].terms(i), 10)
        n = int(got["n"][i])
        assert_same(got["ids"][i, :n], got["scores"][i, :n], ids, sc, f"q{i}")
        conf = restate.margin(sc)
        assert got["conf"][i] == conf and bool(got["skip"][i]) == (conf >= 0.10)


def test_c3_window_equals_restricted_oracle_and_full_budget_equals_flat(c3_small):
    c = c3_small
    orc = restate.OracleIndex.from_host(c["hx"])
    tix = search.TemporalIndex(c["dev"], c["part"])
    lo, hi = tix.window()
    tids = c["tids"][:300]
    off = np.zeros(len(tids) + 1, np.uint32)
    off[1:] = np.cumsum([len(t) for t in tids])
    got = tix.topk_batch(off, np.concatenate(tids), 10)
    ids, sc, n, post = orc.topk(tids, 10, row_lo=lo, row_hi=hi)
    check_batch(got, ids, sc, n, post, what="window")
    # epsilon -> 0, kmax large: the whole index (flat equivalence, acceptance.cpp:173-208)
    full = search.TemporalIndex(c["dev"], c["part"], search.TemporalParams(
        epsilon=1e-9, lambda_hat=0.01, k_max_partitions=1 << 20))  # k* = 2073 >= K
    assert full.window() == (0, c["hx"].n_docs)
    got = full.topk_batch(off, np.concatenate(tids), 7)
    ids, sc, n, post = orc.topk(tids, 7)
    check_batch(got, ids, sc, n, post, what="full budget")


def test_window_edges_not_tile_aligned(c3_small):
    """Arbitrary row windows (partial first/last tiles) through the C ABI."""
    c = c3_small
    orc = restate.OracleIndex.from_host(c["hx"])
    rng = np.random.default_rng(5)
    tids = c["tids"][:40]
    for _ in range(6):
        lo = int(rng.integers(0, c["hx"].n_docs - 1))
        hi = int(rng.integers(lo + 1, c["hx"].n_docs + 1))
        got = c["dev"].search_lists(tids, 10, row_lo=lo, row_hi=hi)
        ids, sc, n, post = orc.topk(tids, 10, row_lo=lo, row_hi=hi)
        check_batch(got, ids, sc, n, post, what=f"[{lo},{hi})")
        ex = c["dev"].search_lists(tids, 10, row_lo=lo, row_hi=hi, flags=search.HM_FLAG_FORCE_EXACT)
        check_batch(ex, ids, sc, n, post, what=f"exact [{lo},{hi})")
        sd = c["dev"].search_lists(tids, 10, row_lo=lo, row_hi=hi, flags=search.HM_FLAG_SEED_ALL)
        check_batch(sd, ids, sc, n, post, what=f"seeded [{lo},{hi})")
