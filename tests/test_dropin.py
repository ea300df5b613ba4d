"""The C++ drop-in (csrc/dropin/hybrid_b200.cpp compiled against the
reference's own headers, linked in place of csr_index.o/temporal_index.o)
against the unmodified reference library, call for call: the reference's
test_csr.cpp / test_temporal.cpp shapes through hybrid::CsrIndex and
hybrid::TemporalIndex.  Driver: tests/cpp/dropin_driver.cpp."""
import os
import subprocess

import numpy as np
import pytest

from _util import random_instance, ref, toy_docs

DRIVER = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "bin", "dropin_driver")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(DRIVER), reason="drop-in driver not built")]


class Driver:
    def __init__(self):
        self.p = subprocess.Popen([DRIVER], stdin=subprocess.PIPE, stdout=subprocess.PIPE, text=True)

    def send(self, lines, expect=1):
        self.p.stdin.write("".join(l + "\n" for l in lines))
        self.p.stdin.flush()
        return [self.p.stdout.readline().strip() for _ in range(expect)]

    def close(self):
        self.p.stdin.close()
        self.p.wait(timeout=30)


def parse(line):
    parts = line.split()
    assert parts[0] == "R", line
    n, extra = int(parts[1]), int(parts[2])
    ids = [int(x.split(":")[0]) for x in parts[3:3 + n]]
    sc = [float.fromhex(x.split(":")[1]) for x in parts[3:3 + n]]
    return ids, sc, extra


def parse_ext(line, n_extra):
    """R n x1 .. x_{n_extra} id:score ... -> (ids, scores, [x1 ..])"""
    parts = line.split()
    assert parts[0] == "R", line
    n = int(parts[1])
    extra = parts[2:2 + n_extra]
    ent = parts[2 + n_extra:2 + n_extra + n]
    return [int(x.split(":")[0]) for x in ent], [float.fromhex(x.split(":")[1]) for x in ent], extra


def bits(xs):
    return np.asarray(xs, np.float64).view(np.uint64).tolist()


def test_csr_dropin_matches_reference(gpu):
    d = Driver()
    rng = np.random.default_rng(77)
    cases = [(toy_docs(), [(["cat"], 100), (["cat", "dog"], 5), (["unicorn"], 5), (["fish", "cat", "cat"], 3)])]
    for _ in range(60):
        docs, q = random_instance(rng)
        cases.append((docs, [(q, 1 + int(rng.integers(0, 10)))]))
    for docs, queries in cases:
        d.send([f"DOCS {len(docs)}"] + [f"{i}\t{t}" for i, t in docs], expect=0)
        assert d.send(["INDEX 0 1.2 0.75"])[0].startswith("OK")
        ri = ref.RefIndex.from_texts(docs, ref.TOK_MINIMAL)
        for q, k in queries:
            for ms in (0, 1):
                ids, sc, post = parse(d.send([f"QUERY {k} 1.2 0.75 {ms} " + " ".join(q)])[0])
                w_ids, w_sc, w_post = ri.search(q, k, maxscore=bool(ms))
                assert ids == w_ids.tolist() and bits(sc) == bits(w_sc), (docs, q, k)
                if not ms:
                    assert post == w_post
    # error mapping: bm25_term_score range check (test_csr.cpp:125-130)
    d.send([f"DOCS {len(toy_docs())}"] + [f"{i}\t{t}" for i, t in toy_docs()], expect=0)
    d.send(["INDEX 0 1.2 0.75"])
    assert d.send(["TERMSCORE 0 3"])[0].startswith("V ")
    assert d.send(["TERMSCORE 0 4"])[0].startswith("THROW out_of_range")
    assert d.send(["KSTAR 0.05 1.4"])[0] == "V 3"
    assert d.send(["KSTAR 0 1"])[0].startswith("THROW invalid_argument")
    d.close()


def test_temporal_dropin_matches_reference(gpu):
    day = 24 * 3600 * 1000
    rng = np.random.default_rng(17)
    n = 300
    ts = [int(rng.integers(0, 60 * day)) for _ in range(n)]
    texts = [" ".join("t%d" % int(rng.integers(0, 40)) for _ in range(3 + int(rng.integers(0, 12))))
             for _ in range(n)]
    d = Driver()
    d.send([f"RECORDS {n}"] + [f"{i} {ts[i]} {texts[i]}" for i in range(n)], expect=0)
    for eps, kmax in [(0.05, 4), (1e-9, 64)]:
        assert d.send([f"TEMPORAL {7 * day} {eps} 1.4 {kmax} 0"])[0].startswith("OK")
        rt = ref.RefTemporal.from_records(list(range(n)), ts, texts, epsilon=eps, k_max=kmax,
                                          tok_mode=ref.TOK_MINIMAL)
        for _ in range(40):
            q = ["t%d" % int(rng.integers(0, 40)) for _ in range(1 + int(rng.integers(0, 4)))]
            k = 1 + int(rng.integers(0, 10))
            for ub in (1, 0):
                ids, sc, searched = parse(d.send([f"TQUERY {k} {ub} " + " ".join(q)])[0])
                w_ids, w_sc, w_searched, _ = rt.topk(q, k, use_ub_stop=bool(ub))
                assert ids == w_ids.tolist() and bits(sc) == bits(w_sc)
                assert searched == w_searched
    d.close()


def _vec_str(idx, val):
    return f"{len(idx)} " + " ".join(f"{int(i)}:{float(v).hex()}" for i, v in zip(idx, val))


def test_bridge_dropin_matches_reference(gpu):
    """hybrid::bridge_ingest / bridge_export / bridge_topk(_maxscore) /
    SparseVector::validate through the drop-in (csrc/dropin/bridge_b200.cpp)
    against the reference's bridge.cpp, call for call."""
    rng = np.random.default_rng(5)
    d = Driver()
    for ndocs, vocab, dens in ((10, 200, 0.05), (1000, 200, 0.05), (4000, 1000, 0.005)):
        docs = []
        for _ in range(ndocs):
            idx = np.nonzero(rng.random(vocab) < dens)[0]
            docs.append((idx, 0.05 + rng.random(len(idx)) * 3.0))
        ids = rng.permutation(5 * ndocs)[:ndocs]
        d.send([f"BDOCS {ndocs}"] + [f"{int(i)} " + _vec_str(*v) for i, v in zip(ids, docs)], expect=0)
        ok = d.send(["BINGEST"])[0].split()
        rb = ref.RefBridge.from_vectors(ids.astype(np.uint64), docs)
        x = rb.export()
        assert ok[0] == "OK" and int(ok[1]) == ndocs and int(ok[2]) == len(x["posting_rows"])
        assert float.fromhex(ok[3]) == x["avgdl"]
        # export round trip, exact
        e = d.send(["BEXPORT"])[0].split()
        w_ids, w_off, w_idx, w_val = rb.export_vectors()
        assert int(e[1]) == ndocs
        for r, tok in enumerate(e[2:]):
            head, *rest = tok.split(",")
            assert head == f"{int(w_ids[r])}:{int(w_off[r + 1] - w_off[r])}"
            for j, kv in enumerate(rest):
                t, v = kv.split("=")
                assert int(t) == int(w_idx[w_off[r] + j]) and float.fromhex(v) == w_val[w_off[r] + j]
        for _ in range(30):
            qi = np.nonzero(rng.random(vocab + 5) < 0.03)[0]
            qv = 0.1 + rng.random(len(qi))
            k = int(rng.choice([1, 5, 10, 100]))
            want = rb.topk_batch([(qi, qv)], k)
            for ms in (0, 1):
                got_ids, got_sc, post = parse(d.send([f"BQUERY {k} {ms} " + _vec_str(qi, qv)])[0])
                n = int(want["n"][0])
                assert got_ids == want["ids"][0, :n].tolist() and bits(got_sc) == bits(want["scores"][0, :n])
                assert post == int(want["postings"][0])
    # validation messages and mode checks (test_bridge.cpp:141-167)
    for idx, val in (([3, 1], [1.0, 1.0]), ([1, 1], [1.0, 1.0]), ([1, 2], [1.0, 0.0]), ([1, 2], [0.5, 1.0])):
        try:
            ref.sparse_validate(idx, val)
            want = "OK"
        except RuntimeError as ex:
            want = "THROW invalid_argument " + str(ex)
        assert d.send(["BVALIDATE " + _vec_str(idx, val)])[0] == want
    assert d.send(["BM25ONBRIDGE"])[0] == "THROW runtime_error BM25 scoring requires a BM25-mode index"
    d.send([f"DOCS {len(toy_docs())}"] + [f"{i}\t{t}" for i, t in toy_docs()], expect=0)
    d.send(["INDEX 0 1.2 0.75"])
    assert d.send(["BONBM25"])[0] == "THROW runtime_error bridge scoring requires a bridge-mode index"
    d.send(["BDOCS 2", "3 1 1:0x1p+0", "3 1 2:0x1p+0"], expect=0)
    assert d.send(["BINGEST"])[0] == "THROW runtime_error duplicate doc id: 3"
    d.close()


def test_dense_and_cascade_dropin_match_reference(gpu):
    """hybrid::dense_topk through the drop-in (csrc/dropin/dense_b200.cpp; the
    reference's dense.o keeps hash_embed with its dense_topk weakened), and
    the reference's own cascade_retrieve driving both GPU channels."""
    rng = np.random.default_rng(8)
    docs, _ = random_instance(rng)
    docs = [(i, "t%d t%d t%d z%d" % (i % 7, i % 11, i % 5, i)) for i in range(300)]
    d = Driver()
    d.send([f"DOCS {len(docs)}"] + [f"{i}\t{t}" for i, t in docs], expect=0)
    assert d.send(["INDEX 0 1.2 0.75"])[0].startswith("OK")
    assert d.send(["EMBDOCS 32 42"])[0] == "OK 300"
    emb = np.stack([ref.hash_embed(t, 32, 42) for _, t in docs])
    ids = np.array([i for i, _ in docs], np.uint64)
    ri = ref.RefIndex.from_texts(docs, ref.TOK_MINIMAL)
    recs = {i: (i * 1000, 0.0) for i, _ in docs}
    n_esc = 0
    for trial in range(40):
        q = ["t%d" % int(rng.integers(0, 12)) for _ in range(1 + int(rng.integers(0, 3)))]
        k = int(rng.choice([1, 3, 10, 400]))
        text = " ".join(q)
        got_ids, got_sc, _ = parse(d.send([f"DQUERY {k} {text}"])[0])
        w = ref.dense_topk_batch(emb, ids, ref.hash_embed(text, 32, 42)[None, :], min(k, 300))
        n = int(w["n"][0])
        assert got_ids == w["ids"][0, :n].tolist() and bits(got_sc) == bits(w["scores"][0, :n])
        # cascade_retrieve (cascade.cpp:44-101) with both channels on the GPU
        tau = float(rng.choice([0.0, 0.1, 0.5, 1e300]))  # 1e300: always escalate (istream has no "inf")
        kk = min(k, 50)
        c_ids, c_sc, esc = parse(d.send([f"CASCADE {kk} {tau} 500000 {text}"])[0])
        s_ids, s_sc, _ = ri.search(q, kk, maxscore=True)
        sparse = list(zip(s_ids.tolist(), s_sc.tolist()))
        if ref.confidence(s_sc) >= tau:
            assert esc == 0 and c_ids == s_ids.tolist() and bits(c_sc) == bits(s_sc)
        else:
            n_esc += 1
            dl = ref.dense_topk_batch(emb, ids, ref.hash_embed(text, 32, 42)[None, :], kk)
            dense = list(zip(dl["ids"][0, :dl["n"][0]].tolist(), dl["scores"][0, :dl["n"][0]].tolist()))
            want = ref.agent_rrf(sparse, dense, recs, 500000)[:kk]
            assert esc == 1 and c_ids == [x for x, _ in want] and bits(c_sc) == bits([s for _, s in want])
    assert n_esc > 5
    assert d.send(["DBADDIM"])[0] == "THROW invalid_argument query dimension mismatch"
    d.close()


def test_batch_entries_match_reference_and_cache_is_bounded(gpu):
    """hybrid_b200::bm25_topk_batch / temporal_topk_batch (include/hybrid_b200.hpp):
    one GPU batch per call, result i == the reference's per-query call on
    query i (ids, score bits, postings, Margin/skip, partitions searched); the
    drop-in's device cache stays bounded (LRU) however many indexes are built."""
    rng = np.random.default_rng(41)
    d = Driver()
    for trial in range(12):
        docs, _ = random_instance(rng)
        d.send([f"DOCS {len(docs)}"] + [f"{i}\t{t}" for i, t in docs], expect=0)
        assert d.send(["INDEX 0 1.2 0.75"])[0].startswith("OK")
        ri = ref.RefIndex.from_texts(docs, ref.TOK_MINIMAL)
        qs = [random_instance(rng)[1] for _ in range(25)] + [[], ["zz_unknown"]]
        k = 1 + int(rng.integers(0, 12))
        lines = d.send([f"QBATCH {k} 1 {len(qs)}"] + [" ".join(q) for q in qs], expect=len(qs))
        for q, line in zip(qs, lines):
            ids, sc, (post, conf, skip) = parse_ext(line, 3)
            post, conf, skip = int(post), float.fromhex(conf), int(skip)
            w_ids, w_sc, w_post = ri.search(q, k)
            assert ids == w_ids.tolist() and bits(sc) == bits(w_sc) and post == w_post, (q, k)
            assert conf == ref.confidence(w_sc) and skip == int(conf >= 0.10)
    n_cached = int(d.send(["NCACHED"])[0].split()[1])
    assert 1 <= n_cached <= 6
    # temporal batches
    day = 24 * 3600 * 1000
    n = 400
    ts = [int(rng.integers(0, 50 * day)) for _ in range(n)]
    texts = [" ".join("t%d" % int(rng.integers(0, 30)) for _ in range(2 + int(rng.integers(0, 10))))
             for _ in range(n)]
    d.send([f"RECORDS {n}"] + [f"{i} {ts[i]} {texts[i]}" for i in range(n)], expect=0)
    for eps, kmax in [(0.05, 4), (1e-9, 64)]:
        assert d.send([f"TEMPORAL {7 * day} {eps} 1.4 {kmax} 0"])[0].startswith("OK")
        rt = ref.RefTemporal.from_records(list(range(n)), ts, texts, epsilon=eps, k_max=kmax,
                                          tok_mode=ref.TOK_MINIMAL)
        budget = min(ref.k_star(eps, 1.4), kmax, len(rt.partitions()[0]))
        qs = [["t%d" % int(rng.integers(0, 30)) for _ in range(1 + int(rng.integers(0, 4)))] for _ in range(60)]
        for k in (1, 5, 50):
            for ub in (1, 0):
                lines = d.send([f"TBATCH {k} {ub} {len(qs)}"] + [" ".join(q) for q in qs], expect=len(qs))
                for q, line in zip(qs, lines):
                    ids, sc, (searched, stopped) = parse_ext(line, 2)
                    searched, stopped = int(searched), int(stopped)
                    w_ids, w_sc, w_searched, _ = rt.topk(q, k, use_ub_stop=bool(ub))
                    assert ids == w_ids.tolist() and bits(sc) == bits(w_sc), (q, k, ub)
                    assert searched == w_searched
                    assert stopped == int(w_searched < budget)
    d.close()
