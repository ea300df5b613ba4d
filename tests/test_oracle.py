"""Pin the oracle: the C restatement (oracle/bm25_oracle.c) against the golden
vectors generated from the reference library (tests/golden/, made by
oracle/make_golden.py) and, where oracle/_ref exists, against the reference
library itself.  CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import ref, restate

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLD, name + ".json")) as f:
        return json.load(f)


def unhex(xs):
    return np.array([float.fromhex(x) for x in xs], np.float64)


def bits_equal(a, b):
    return np.asarray(a, np.float64).view(np.uint64).tolist() == np.asarray(b, np.float64).view(np.uint64).tolist()


def oracle_from_texts(docs, k1=1.2, b=0.75):
    """Index of tiny texts built by a minimal Python restatement of build_index
    (csr_index.cpp:232-324, Minimal tokenizer on 't<n>'/'z<n>' words)."""
    rows = {}
    lens = []
    for row, (_, text) in enumerate(docs):
        toks = text.lower().split()
        lens.append(len(toks))
        counts = {}
        for t in toks:
            counts[t] = counts.get(t, 0) + 1
        for t, c in counts.items():
            rows.setdefault(t, []).append((row, c))
    terms = sorted(rows)
    off = [0]
    pr, pw = [], []
    for t in terms:
        for r, c in rows[t]:
            pr.append(r)
            pw.append(float(c))
        off.append(len(pr))
    N = len(docs)
    idf = [restate.lib().or_idf_from_df(len(rows[t]), N) for t in terms]
    avgdl = (sum(float(l) for l in lens) / N) if N else 0.0
    ms = []
    for ti, t in enumerate(terms):
        ms.append(max(restate.bm25_score(c, idf[ti], lens[r], avgdl, k1, b) for r, c in rows[t]))
    orc = restate.OracleIndex(off, pr, pw, idf, ms, lens, [d for d, _ in docs], avgdl)
    return orc, {t: i for i, t in enumerate(terms)}, terms


def test_toy_layout_and_known_answers():
    g = load("toy")
    orc, vocab, terms = oracle_from_texts(g["docs"])
    assert terms == g["terms"]
    assert orc.term_offsets.tolist() == g["term_offsets"]
    assert orc.posting_rows.tolist() == g["posting_rows"]
    assert orc.posting_weights.tolist() == g["posting_tf"]
    assert bits_equal(orc.idf, unhex(g["idf"]))
    assert bits_equal(orc.order_key, unhex(g["maxscore"]))
    assert orc.doc_lens.tolist() == g["doc_lens"] == [10, 8, 12, 7, 9]
    assert orc.avgdl == float.fromhex(g["avgdl"])
    assert terms[:3] == ["cat", "dog", "fish"]
    assert g["term_offsets"][:4] == [0, 4, 7, 9]
    for q in g["queries"]:
        tids = [vocab.get(t, 0xFFFFFFFF) for t in q["terms"]]
        ids, sc, n, post = orc.topk([tids], q["k"])
        assert ids[0, :n[0]].tolist() == q["ids"], q
        assert bits_equal(sc[0, :n[0]], unhex(q["scores"])), q
        assert post[0] == q["postings"]


def test_random_instances_golden():
    for c in load("random_instances"):
        orc, vocab, _ = oracle_from_texts(c["docs"])
        tids = [vocab.get(t, 0xFFFFFFFF) for t in c["query"]]
        ids, sc, n, post = orc.topk([tids], c["k"], k1=c["k1"], b=c["b"])
        assert ids[0, :n[0]].tolist() == c["ids"]
        assert bits_equal(sc[0, :n[0]], unhex(c["scores"]))
        assert post[0] == c["postings"]


def test_known_answers():
    g = load("knowns")
    for e in g["bm25"]:
        assert restate.bm25_score(*e["args"]).hex() == e["value"], e
    # test_csr.cpp:92-100 anchors
    assert abs(restate.bm25_score(1.0, 1.2, 12.0, 9.2) - 1.0672) <= 1.0672e-3
    both = restate.bm25_score(1.0, 1.2, 12.0, 9.2) + restate.bm25_score(2.0, 0.8, 12.0, 9.2)
    assert abs(both - 2.0805) <= 2.0805e-3
    for c in g["confidence"]:
        assert restate.confidence(c["scores"], 0).hex() == c["margin"]
        assert restate.confidence(c["scores"], 1).hex() == c["top1"]
        assert restate.confidence(c["scores"], 2).hex() == c["entropy"]
    assert abs(restate.margin([8.74, 2.13, 1.40, 0.91, 0.83]) - 0.756) <= 1e-3
    assert abs(restate.margin([4.21, 3.97, 3.48, 3.11, 2.96]) - 0.057) <= 1e-3
    for c in g["k_star"]:
        assert restate.k_star(c["eps"], c["lam"]) == c["value"]
    assert restate.k_star(0.0, 1.0) == 0 and restate.k_star(0.05, 0.0) == 0  # domain errors
    for c in g["ndcg"]:
        rels = {int(a): b for a, b in c["rels"].items()}
        assert restate.ndcg(c["ids"], rels, c["k"]).hex() == c["exp"]
        assert restate.ndcg(c["ids"], rels, c["k"], linear=True).hex() == c["lin"]


def test_twophase_golden_and_sentinel():
    g = load("knowns")
    for c in g["twophase"]:
        sel = restate.TwoPhase(c["cap"])
        ids, sc = sel.select(unhex(c["row"]), c["k"])
        assert ids.tolist() == c["ids"] and bits_equal(sc, unhex(c["scores"]))
    big = [100.0 + i for i in range(40)]
    small = [float(i) for i in range(1, 9)]
    for reset in (False, True):
        sel = restate.TwoPhase(32, reset_sentinel=reset)
        sel.select(big, 2)
        ids, sc = sel.select(small, 2)
        want = g["twophase_reset_%d" % reset]
        assert ids.tolist() == want["ids"] and bits_equal(sc, unhex(want["scores"]))
    assert g["twophase_reset_1"]["ids"] == [7, 6]          # sort oracle
    assert g["twophase_reset_0"]["ids"] != [7, 6]          # contamination reproduced
    with pytest.raises(ValueError):
        restate.TwoPhase(8).select([1.0, 2.0], 9)


def test_c1_golden_sample_with_native_builder():
    """The native generator + builder + restatement reproduce the reference
    at BASELINE config 1 (hashes of every CSR array, first 40 queries' top-10)."""
    from paper_2605_25092_b200 import synth
    import hashlib

    g = load("c1_sample")
    sp = g["spec"]
    c = synth.Corpus(n_records=sp["n_records"], vocab_size=sp["vocab_size"],
                     min_doc_tokens=sp["min_tok"], max_doc_tokens=sp["max_tok"])
    q = synth.Queries(c, n_queries=1000)
    hx = synth.HostIndex(c)
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
    _, _, ts = c.arrays()
    assert sha(ts) == g["ts_sha"]
    assert hx.n_terms == g["n_terms"] and len(hx.posting_rows) == g["n_postings"]
    assert sha(hx.posting_rows) == g["rows_sha"] and sha(hx.posting_tf) == g["tf_sha"]
    assert sha(hx.idf) == g["idf_sha"] and sha(hx.order_key) == g["order_key_sha"]
    assert sha(hx.doc_lens) == g["doc_lens_sha"] and hx.avgdl == float.fromhex(g["avgdl"])
    orc = restate.OracleIndex.from_host(hx)
    for i, e in enumerate(g["queries"]):
        assert q.terms(i) == e["terms"] and q.gold[i] == e["gold"] and q.ts[i] == e["ts"]
        tids = hx.resolve(q.term_ranks[q.offsets[i]:q.offsets[i + 1]])
        ids, sc, n, post = orc.topk([tids], 10)
        assert ids[0, :n[0]].tolist() == e["ids"]
        assert bits_equal(sc[0, :n[0]], unhex(e["scores"]))
        assert post[0] == e["postings"]
        assert restate.margin(sc[0, :n[0]]).hex() == e["margin"]


@pytest.mark.skipif(not ref.available(), reason="reference library not built here")
def test_restatement_vs_reference_library_random():
    rng = np.random.default_rng(7)
    for trial in range(200):
        nd = 5 + int(rng.integers(0, 61))
        V = 8 + int(rng.integers(0, 26))
        docs = [(d, " ".join("t%d" % int(rng.integers(0, V)) for _ in range(2 + int(rng.integers(0, 16)))))
                for d in range(nd)]
        q = ["t%d" % int(rng.integers(0, V)) for _ in range(1 + int(rng.integers(0, 5)))]
        k = 1 + int(rng.integers(0, 12))
        ri = ref.RefIndex.from_texts(docs, ref.TOK_MINIMAL)
        e = ri.export()
        orc = restate.OracleIndex(e["term_offsets"], e["posting_rows"], e["posting_weights"],
                                  e["idf"], e["order_key"], e["doc_lens"], e["doc_ids"], e["avgdl"])
        vocab = {t: i for i, t in enumerate(e["terms"])}
        ids, sc, n, post = orc.topk([[vocab.get(t, 0xFFFFFFFF) for t in q]], k)
        w_ids, w_sc, w_post = ri.search(q, k)
        assert ids[0, :n[0]].tolist() == w_ids.tolist(), trial
        assert bits_equal(sc[0, :n[0]], w_sc) and post[0] == w_post


def test_temporal_budget_restatement():
    g = load("temporal")
    for c in g["cases"]:
        b = restate.temporal_budget(c["epsilon"], c["lambda_hat"], c["k_max"], c["partitions"])
        assert max(q["searched"] for q in c["queries"]) <= b


def test_reference_temporal_from_flat_equals_its_own_build():
    """ref_temporal_from_flat (the bench's C3 CPU baseline object: partitions
    cut from a partition-ordered flat index) == the reference's own
    build_temporal_index on the same corpus: results and partitions searched."""
    import numpy as np
    from paper_2605_25092_b200 import synth
    day = 24 * 3600 * 1000
    n = 20000
    span = int(28 * day * n / 4052)
    corpus = synth.Corpus(n_records=n, time_span_ms=span)
    queries = synth.Queries(corpus, n_queries=200)
    K, order, part, t0 = corpus.partition(7 * day)
    hx = synth.HostIndex(corpus, row_order=order)
    rf = ref.RefTemporal.from_flat(hx.term_strings(), hx.term_offsets, hx.posting_rows,
                                   hx.posting_tf.astype(np.float64), hx.idf, hx.order_key, hx.doc_lens,
                                   hx.doc_ids, hx.avgdl, part, t0)
    rt = ref.RefTemporal.from_corpus(ref.RefCorpus(n, time_span_ms=span))
    assert len(rf.partitions()[2]) == len(rt.partitions()[2]) == K
    assert (rf.partitions()[2] == rt.partitions()[2]).all() and (rf.partitions()[0] == rt.partitions()[0]).all()
    for i in range(len(queries)):
        a = rf.topk(queries.terms(i), 10)
        b = rt.topk(queries.terms(i), 10)
        assert a[0].tolist() == b[0].tolist() and a[1].view(np.uint64).tolist() == b[1].view(np.uint64).tolist()
        assert a[2] == b[2] and a[3] == b[3]
