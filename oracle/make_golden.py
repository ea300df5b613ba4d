"""Generate tests/golden/*.json from the UNMODIFIED reference library.

TEST INFRASTRUCTURE ONLY.  Run in a container that has /root/reference (the
reference library is built by `make -C oracle ref`):

    python oracle/make_golden.py

The fixtures pin the C restatement (oracle/bm25_oracle.c) and the native
generator/builder where the reference itself is absent (the GPU box).  Inputs
are stored in the fixtures, so they do not depend on this script's RNG.
Scores are stored as float.hex() strings (bit-exact).
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
DAY = 24 * 3600 * 1000


def hx(a):
    return [float(x).hex() for x in a]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def toy():
    docs = [(0, "cat cat fish z00 z01 z02 z03 z04 z05 z06"),
            (1, "dog z10 z11 z12 z13 z14 z15 z16"),
            (2, "cat dog dog z20 z21 z22 z23 z24 z25 z26 z27 z28"),
            (3, "cat fish z30 z31 z32 z33 z34"),
            (4, "cat cat cat dog z40 z41 z42 z43 z44")]
    ri = ref.RefIndex.from_texts(docs, ref.TOK_MINIMAL)
    e = ri.export()
    out = dict(docs=docs, terms=e["terms"], term_offsets=e["term_offsets"].tolist(),
               posting_rows=e["posting_rows"].tolist(), posting_tf=e["posting_weights"].tolist(),
               idf=hx(e["idf"]), maxscore=hx(e["maxscore"]), doc_lens=e["doc_lens"].tolist(),
               avgdl=float(e["avgdl"]).hex(), queries=[])
    for q, k in [(["cat"], 100), (["cat", "dog"], 5), (["unicorn"], 5), (["fish", "cat", "cat"], 3),
                 (["dog", "z00", "nope"], 4), (["cat"], 2)]:
        ids, sc, post = ri.search(q, k)
        out["queries"].append(dict(terms=q, k=k, ids=ids.tolist(), scores=hx(sc), postings=post))
    return out


def random_instances(n=60, seed=1234):
    rng = np.random.default_rng(seed)
    cases = []
    for _ in range(n):
        nd = 5 + int(rng.integers(0, 61))
        V = 8 + int(rng.integers(0, 26))
        docs = [(d, " ".join("t%d" % int(rng.integers(0, V)) for _ in range(2 + int(rng.integers(0, 16)))))
                for d in range(nd)]
        q = ["t%d" % int(rng.integers(0, V)) for _ in range(1 + int(rng.integers(0, 5)))]
        k = 1 + int(rng.integers(0, 10))
        k1, b = (1.2, 0.75) if rng.random() < 0.7 else (float(rng.uniform(0.3, 2.0)), float(rng.uniform(0, 1)))
        ri = ref.RefIndex.from_texts(docs, ref.TOK_MINIMAL, k1=1.2, b=0.75)
        ids, sc, post = ri.search(q, k, k1=k1, b=b)
        ids2, sc2, _ = ri.search(q, k, k1=k1, b=b, maxscore=True)
        assert (ids == ids2).all() and (sc == sc2).all()
        cases.append(dict(docs=docs, query=q, k=k, k1=k1, b=b, ids=ids.tolist(), scores=hx(sc),
                          postings=post))
    return cases


def knowns():
    out = {}
    out["bm25"] = [dict(args=list(a), value=ref.bm25_score(*a).hex()) for a in
                   [(1.0, 1.2, 12.0, 9.2, 1.2, 0.75), (2.0, 0.8, 12.0, 9.2, 1.2, 0.75),
                    (1e9, 2.0, 50.0, 10.0, 1.2, 0.75), (3.0, 1.0, 5.0, 10.0, 1.2, 0.0),
                    (3.0, 1.0, 500.0, 10.0, 1.2, 0.0), (1.0, 1.0, 2.0, 3.0, 1.2, 0.75),
                    (3.0, 1.0, 4.0, 3.0, 1.2, 0.75), (2.0, 1.5, 7.0, 0.0, 1.2, 0.75)]]
    conf = []
    for s in [[8.74, 2.13, 1.40, 0.91, 0.83], [4.21, 3.97, 3.48, 3.11, 2.96], [], [0.0, 0.0],
              [5.0], [3.0, 1.0], [2.0, 2.0, 2.0, 2.0], [7.0, 0.0, 0.0], [1e-12, 5e-13]]:
        conf.append(dict(scores=s, margin=ref.confidence(s, 0).hex(),
                         top1=ref.confidence(s, 1).hex(), entropy=ref.confidence(s, 2).hex()))
    out["confidence"] = conf
    out["k_star"] = [dict(eps=e, lam=l, value=ref.k_star(e, l)) for e, l in
                     [(0.05, 1.4), (0.01, 0.5), (0.999999, 1.0), (0.5, 10.0)]]
    out["ndcg"] = []
    for ids, rels, k in [([10, 11, 12], {10: 2, 12: 1, 13: 0}, 3), ([1, 2, 3], {1: 3, 2: 2, 3: 1}, 3),
                         ([1, 2], {}, 2), ([5, 6, 7, 8], {7: 1}, 10), ([5, 6, 7, 8], {9: 1}, 2)]:
        out["ndcg"].append(dict(ids=ids, rels={str(a): b for a, b in rels.items()}, k=k,
                                exp=ref.ndcg(ids, rels, k).hex(),
                                lin=ref.ndcg(ids, rels, k, linear=True).hex()))
    rng = np.random.default_rng(99)
    tp = []
    for _ in range(40):
        n = 1 + int(rng.integers(0, 200))
        row = (rng.random(n) * 10.0).tolist()
        k = 1 + int(rng.integers(0, 32))
        ids, sc, cnt = ref.twophase_batch(np.array([row]), k, 32)
        tp.append(dict(row=[float(x).hex() for x in row], k=k, cap=32, ids=ids[0, :cnt[0]].tolist(),
                       scores=hx(sc[0, :cnt[0]])))
    out["twophase"] = tp
    big = [100.0 + i for i in range(40)]
    small = [float(i) for i in range(1, 9)]
    for reset in (False, True):
        ids, sc, cnt = ref.twophase_batch(np.array([big + [0.0] * 0, small + [0.0] * 32]), 2, 32, reset)
        out["twophase_reset_%d" % reset] = dict(ids=ids[1, :cnt[1]].tolist(), scores=hx(sc[1, :cnt[1]]))
    return out


def c1_sample(nq=40):
    rc = ref.RefCorpus(100000)
    ids, ts, texts = rc.export()
    rq = ref.RefQueries(rc, 1000)
    ri = ref.RefIndex.from_corpus(rc)
    e = ri.export()
    out = dict(spec=dict(n_records=100000, vocab_size=5000, min_tok=5, max_tok=30, seed=42),
               n_docs=len(ids), ts_sha=sha(ts), n_terms=len(e["terms"]),
               n_postings=int(len(e["posting_rows"])), rows_sha=sha(e["posting_rows"]),
               tf_sha=sha(e["posting_weights"].astype(np.uint32)), idf_sha=sha(e["idf"]),
               order_key_sha=sha(e["order_key"]), doc_lens_sha=sha(e["doc_lens"]),
               avgdl=float(e["avgdl"]).hex(), queries=[])
    for i in range(nq):
        q = rq.terms[i]
        r_ids, r_sc, post = ri.search(q, 10)
        out["queries"].append(dict(terms=q, gold=int(rq.gold[i]), ts=int(rq.ts[i]),
                                   ids=r_ids.tolist(), scores=hx(r_sc), postings=post,
                                   margin=ref.confidence(r_sc, 0).hex()))
    return out


def temporal():
    rng = np.random.default_rng(42)
    n = 300
    ids = list(range(n))
    ts = [int(rng.integers(0, 60 * DAY)) for _ in range(n)]
    texts = [" ".join("t%d" % int(rng.integers(0, 40)) for _ in range(3 + int(rng.integers(0, 12))))
             for _ in range(n)]
    cases = []
    for eps, kmax in [(0.05, 4), (1e-9, 64), (0.9, 4)]:
        rt = ref.RefTemporal.from_records(ids, ts, texts, epsilon=eps, k_max=kmax,
                                          tok_mode=ref.TOK_MINIMAL)
        ws, we, nd = rt.partitions()
        qs = []
        for _ in range(40):
            q = ["t%d" % int(rng.integers(0, 40)) for _ in range(1 + int(rng.integers(0, 4)))]
            k = 1 + int(rng.integers(0, 10))
            r_ids, r_sc, searched, post = rt.topk(q, k)
            qs.append(dict(terms=q, k=k, ids=r_ids.tolist(), scores=hx(r_sc), searched=searched))
        cases.append(dict(epsilon=eps, k_max=kmax, lambda_hat=1.4, window_ms=7 * DAY,
                          partitions=len(ws), window_start=ws.tolist(), part_docs=nd.tolist(),
                          queries=qs))
    return dict(ids=ids, ts=ts, texts=texts, cases=cases)


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, fn in [("toy", toy), ("random_instances", random_instances), ("knowns", knowns),
                     ("c1_sample", c1_sample), ("temporal", temporal)]:
        with open(os.path.join(OUT, name + ".json"), "w") as f:
            json.dump(fn(), f, separators=(",", ":"))
        print("wrote", name)


if __name__ == "__main__":
    main()
