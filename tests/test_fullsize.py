"""Full-size parity on BASELINE configs C2, C3 and C4 against the reference
itself (tests/golden/fullsize_*.{json,npz}, made by
oracle/make_fullsize_golden.py from the unmodified reference library).

* Builder: the native generator + builder (libhm_synth) regenerates each
  config at full size and must reproduce the SHA-256 of every array of the
  reference's gen_corpus + build_index (src/workload.cpp:47-135,
  src/csr_index.cpp:232-324) -- C2 and C4 at 8,841,823 docs, V = 1M -- so the
  reference's answers on its own index are answers on ours.
* Search: the GPU batch over every query of the config, compared on the
  sampled queries with the reference's bm25_topk_maxscore (C2: 1,000 queries,
  C4: 256 at k = 100) or TemporalIndex::topk (C3: 1,000 queries at 5M
  records): ids and score bits identical, Margin confidence and skip equal to
  the reference's rule on the reference's scores, nDCG@10 identical, C2
  postings_touched equal to the reference's exhaustive count, C3
  partitions_searched equal to the reference's.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from _util import restate, search, synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
DAY = 24 * 3600 * 1000


def golden(name):
    with open(os.path.join(GOLD, f"fullsize_{name}.json")) as f:
        meta = json.load(f)
    return meta, dict(np.load(os.path.join(GOLD, f"fullsize_{name}.npz")))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def queries_digest(q):
    return hashlib.sha256("\n".join(" ".join(q.terms(i)) for i in range(len(q))).encode()).hexdigest()


def build(c, row_order_window=None):
    corpus = synth.Corpus(n_records=c["n_records"], vocab_size=c["vocab_size"], min_doc_tokens=c["min_tok"],
                          max_doc_tokens=c["max_tok"], **({"time_span_ms": c["time_span_ms"]}
                                                         if "time_span_ms" in c else {}))
    queries = synth.Queries(corpus, n_queries=c["n_queries"], min_terms=c["min_terms"], max_terms=c["max_terms"])
    part = None
    if row_order_window:
        K, order, part, _ = corpus.partition(row_order_window)
        hx = synth.HostIndex(corpus, row_order=order)
    else:
        hx = synth.HostIndex(corpus)
    return corpus, queries, hx, part


def check_sample(got, g, name, sample, k, gold_docs):
    ids, sc, n = g[f"{name}_ids"], g[f"{name}_scores"].view(np.float64), g[f"{name}_n"]
    nd_got, nd_ref = [], []
    for j, i in enumerate(sample):
        m = int(n[j])
        assert int(got["n"][i]) == m, f"{name} query {i}: count"
        assert (got["ids"][i, :m] == ids[j, :m]).all(), f"{name} query {i}: ids"
        assert (got["scores"][i, :m].view(np.uint64) == sc[j, :m].view(np.uint64)).all(), f"{name} query {i}: scores"
        conf = restate.margin(sc[j, :m])
        assert got["conf"][i] == conf and bool(got["skip"][i]) == (conf >= 0.10), f"{name} query {i}: decision"
        nd_got.append(restate.ndcg(got["ids"][i, :m], {gold_docs[j]: 1}, 10))
        nd_ref.append(restate.ndcg(ids[j, :m], {gold_docs[j]: 1}, 10))
    assert abs(np.mean(nd_got) - np.mean(nd_ref)) <= 2e-4
    return float(np.mean(nd_got))


@pytest.mark.parametrize("name", ["c2", "c4"])
def test_flat_configs_match_reference(gpu, name):
    meta, g = golden(name)
    c = meta["config"]
    _, queries, hx, _ = build(c)
    # the native builder == the reference's build_index, every array, full size
    d = meta["index"]
    assert len(hx.term_rank) == d["n_terms"] and len(hx.posting_rows) == d["n_postings"]
    assert hashlib.sha256("\n".join(hx.term_strings()).encode()).hexdigest() == d["terms"]
    for key, arr in (("term_offsets", hx.term_offsets), ("posting_rows", hx.posting_rows),
                     ("posting_weights", hx.posting_tf.astype(np.float64)), ("idf", hx.idf),
                     ("maxscore", hx.maxscore), ("order_key", hx.order_key), ("doc_lens", hx.doc_lens),
                     ("doc_ids", hx.doc_ids)):
        assert sha(arr) == d[key], f"{name}: {key} differs from the reference's build_index"
    assert float(hx.avgdl).hex() == d["avgdl"]
    assert queries_digest(queries) == meta["queries"], f"{name}: queries differ from gen_queries"
    # every query of the config in one GPU batch (the bench's batch)
    dev = search.DeviceIndex.from_host(hx)
    tids = hx.resolve(queries.term_ranks)
    got = dev.search_batch(queries.offsets.astype(np.uint32), tids, c["k"])
    sample = [int(x) for x in g[f"{name}_sample"]]
    check_sample(got, g, name, sample, c["k"], meta["gold"])
    if name == "c2":
        assert (got["postings"][sample[:64]] == g["c2_postings64"]).all()
    # every query's list is ranked, positive and postings = sum of df (all queries)
    df = np.diff(hx.term_offsets.astype(np.int64))
    off = queries.offsets
    for i in range(0, len(queries), 97):
        m = int(got["n"][i])
        s = got["scores"][i, :m]
        assert (s > 0).all() and (np.diff(s) <= 0).all()
        assert got["postings"][i] == df[np.unique(tids[off[i]:off[i + 1]])].sum()


def test_c3_temporal_matches_reference(gpu):
    meta, g = golden("c3")
    c = meta["config"]
    corpus, queries, hx, part = build(c, row_order_window=7 * DAY)
    assert len(part) - 1 == meta["partitions"]
    assert sha(np.diff(part).astype(np.uint32)) == meta["part_docs"]
    assert queries_digest(queries) == meta["queries"]
    host = search.CsrIndex.from_host(hx)
    tix = search.TemporalIndex(host.dev(), part, host=host)
    sample = [int(x) for x in g["c3_sample"]]
    # the bench path: the newest budget partitions as one row window, every query
    got = tix.topk_batch(queries.offsets.astype(np.uint32), hx.resolve(queries.term_ranks), c["k"])
    check_sample(got, g, "c3", sample, c["k"], meta["gold"])
    # the reference-shaped path: per-partition lists merged newest first with
    # the upper-bound stop (partitions_searched as the reference)
    lists, stats = tix.topk_many([queries.terms(i) for i in sample], c["k"])
    for j, i in enumerate(sample):
        m = int(g["c3_n"][j])
        assert [e[0] for e in lists[j]] == g["c3_ids"][j, :m].tolist()
        assert stats[j].partitions_searched == int(g["c3_searched"][j]), f"query {i}"
