"""Full-size golden fixtures for BASELINE configs C2, C3 and C4 -- TEST
INFRASTRUCTURE, run here (where /root/reference compiles into oracle/_ref).

    python oracle/make_fullsize_golden.py [c2] [c3] [c4]

Everything below is computed by the UNMODIFIED reference library
(oracle/_ref/libhybridref.so):
  * the corpus and queries by hybrid::gen_corpus / gen_queries
    (src/workload.cpp:47-135) with the configs' WorkloadSpec / QuerySpec
    (SURVEY.md §8d), the index by hybrid::build_index (src/csr_index.cpp:
    232-324) or build_temporal_index (src/temporal_index.cpp:125-169);
  * SHA-256 digests of every CsrIndex array (terms, term_offsets,
    posting_rows, posting_weights, term_idfs, term_maxscores,
    term_order_keys, doc_lens, doc_ids, avgdl) -- the GPU box regenerates the
    index with the framework's native builder (libhm_synth) in seconds and
    must reproduce the digests bit for bit (tests/test_fullsize.py);
  * the reference's answers on a fixed sample of queries:
    C2 1,000 queries (every 10th) and C4 256 (every 16th) by
    CsrIndex::bm25_topk_maxscore (identical output to bm25_topk,
    acceptance.cpp:144-171), plus 64 C2 queries by the exhaustive bm25_topk
    for postings_touched; C3 1,000 queries (every 10th) by
    TemporalIndex::topk with partitions_searched.
The fixtures are small (ids + score bits); the box never reads
/root/reference.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden")
DAY = 24 * 3600 * 1000
CONFIGS = {
    "c2": dict(n_records=8841823, vocab_size=1000000, min_tok=20, max_tok=60, n_queries=10000,
               min_terms=3, max_terms=6, k=10, every=10),
    "c4": dict(n_records=8841823, vocab_size=1000000, min_tok=40, max_tok=80, n_queries=4096,
               min_terms=24, max_terms=32, k=100, every=16),
    "c3": dict(n_records=5000000, vocab_size=5000, min_tok=5, max_tok=30, n_queries=10000,
               min_terms=3, max_terms=6, k=10, every=10,
               time_span_ms=int(28 * DAY * 5000000 / 4052)),  # acceptance.cpp:101-104
}
WORKERS = os.cpu_count() or 8


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def digests(x):
    d = {k: sha(x[k]) for k in ("term_offsets", "posting_rows", "posting_weights", "idf", "maxscore",
                                "order_key", "doc_lens", "doc_ids")}
    d["terms"] = hashlib.sha256("\n".join(x["terms"]).encode()).hexdigest()
    d["avgdl"] = float(x["avgdl"]).hex()
    d["n_terms"] = len(x["terms"])
    d["n_postings"] = int(len(x["posting_rows"]))
    d["n_docs"] = int(len(x["doc_ids"]))
    return d


def queries_digest(terms):
    return hashlib.sha256("\n".join(" ".join(t) for t in terms).encode()).hexdigest()


def flat(name):
    c = CONFIGS[name]
    t0 = time.time()
    corpus = ref.RefCorpus(c["n_records"], vocab_size=c["vocab_size"], min_tok=c["min_tok"], max_tok=c["max_tok"])
    rq = ref.RefQueries(corpus, n_queries=c["n_queries"], min_terms=c["min_terms"], max_terms=c["max_terms"])
    print(f"{name}: corpus + queries {time.time() - t0:.0f}s", flush=True)
    ri = ref.RefIndex.from_corpus(corpus)
    del corpus
    print(f"{name}: build_index {time.time() - t0:.0f}s", flush=True)
    x = ri.export()
    meta = dict(config=c, index=digests(x), queries=queries_digest(rq.terms))
    del x
    sample = list(range(0, c["n_queries"], c["every"]))
    qs = [rq.terms[i] for i in sample]
    r = ri.search_batch(qs, c["k"], maxscore=True, workers=WORKERS)
    print(f"{name}: {len(qs)} maxscore queries {r['wall_ms'] / 1e3:.0f}s", flush=True)
    arrays = {f"{name}_sample": np.array(sample, np.uint32), f"{name}_ids": r["ids"],
              f"{name}_scores": r["scores"].view(np.uint64), f"{name}_n": r["n"]}
    if name == "c2":  # postings_touched of the exhaustive path on the first 64 sampled queries
        e = ri.search_batch(qs[:64], c["k"], maxscore=False, workers=WORKERS)
        assert (e["ids"] == r["ids"][:64]).all() and (e["n"] == r["n"][:64]).all()
        arrays["c2_postings64"] = e["postings"]
        print(f"c2: 64 exhaustive queries {e['wall_ms'] / 1e3:.0f}s", flush=True)
    meta["gold"] = [int(rq.gold[i]) for i in sample]
    return meta, arrays


def temporal():
    c = CONFIGS["c3"]
    t0 = time.time()
    corpus = ref.RefCorpus(c["n_records"], vocab_size=c["vocab_size"], min_tok=c["min_tok"], max_tok=c["max_tok"],
                           time_span_ms=c["time_span_ms"])
    rq = ref.RefQueries(corpus, n_queries=c["n_queries"], min_terms=c["min_terms"], max_terms=c["max_terms"])
    rt = ref.RefTemporal.from_corpus(corpus)
    print(f"c3: corpus + build_temporal_index {time.time() - t0:.0f}s", flush=True)
    ws, we, nd = rt.partitions()
    sample = list(range(0, c["n_queries"], c["every"]))
    k = c["k"]
    ids = np.zeros((len(sample), k), np.uint64)
    sc = np.zeros((len(sample), k), np.float64)
    n = np.zeros(len(sample), np.uint32)
    srch = np.zeros(len(sample), np.uint32)
    for j, i in enumerate(sample):
        a, s, m, _ = rt.topk(rq.terms[i], k)
        ids[j, :len(a)], sc[j, :len(a)], n[j], srch[j] = a, s, len(a), m
    print(f"c3: {len(sample)} TemporalIndex::topk {time.time() - t0:.0f}s", flush=True)
    meta = dict(config=c, partitions=len(nd), part_docs=sha(nd.astype(np.uint32)),
                window_start=int(ws[0]), queries=queries_digest(rq.terms),
                gold=[int(rq.gold[i]) for i in sample])
    arrays = {"c3_sample": np.array(sample, np.uint32), "c3_ids": ids, "c3_scores": sc.view(np.uint64),
              "c3_n": n, "c3_searched": srch}
    return meta, arrays


def main():
    which = sys.argv[1:] or ["c2", "c3", "c4"]
    os.makedirs(OUT, exist_ok=True)
    for name in which:
        meta, arrays = temporal() if name == "c3" else flat(name)
        with open(os.path.join(OUT, f"fullsize_{name}.json"), "w") as f:
            json.dump(meta, f, indent=1)
        np.savez_compressed(os.path.join(OUT, f"fullsize_{name}.npz"), **arrays)
        print(f"{name}: written", flush=True)


if __name__ == "__main__":
    main()
