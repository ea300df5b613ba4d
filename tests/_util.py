"""Shared test helpers: fixtures shaped like the reference's own tests
(proj/tests/test_csr.cpp:20-60, acceptance.cpp:61-79) and exact comparators."""
import numpy as np

from oracle import ref, restate
from paper_2605_25092_b200 import search, synth


def toy_docs():
    """Five-doc toy corpus of test_csr.cpp:20-28."""
    return [(0, "cat cat fish z00 z01 z02 z03 z04 z05 z06"),
            (1, "dog z10 z11 z12 z13 z14 z15 z16"),
            (2, "cat dog dog z20 z21 z22 z23 z24 z25 z26 z27 z28"),
            (3, "cat fish z30 z31 z32 z33 z34"),
            (4, "cat cat cat dog z40 z41 z42 z43 z44")]


def mt_uniform(rng, n):
    """uniform_u64 over numpy's Generator (fixtures only; not the reference rng)."""
    return int(rng.integers(0, n)) if n else 0


def random_instance(rng):
    """Random small instance in the shape of test_csr.cpp:35-52."""
    n_docs = 5 + mt_uniform(rng, 60)
    vocab = 8 + mt_uniform(rng, 25)
    docs = []
    for d in range(n_docs):
        ln = 2 + mt_uniform(rng, 15)
        docs.append((d, " ".join("t%d" % mt_uniform(rng, vocab) for _ in range(ln))))
    q = ["t%d" % mt_uniform(rng, vocab) for _ in range(1 + mt_uniform(rng, 4))]
    return docs, q


def export_to_csr(ref_index, build_params=(1.2, 0.75)):
    """Reference-built index -> search.CsrIndex (GPU-backed mirror)."""
    e = ref_index.export()
    return search.CsrIndex(e["terms"], e["term_offsets"], e["posting_rows"],
                           e["posting_weights"], e["idf"], e["order_key"], e["doc_lens"],
                           e["doc_ids"], e["avgdl"], search.Bm25Params(*build_params))


def assert_same(got_ids, got_scores, want_ids, want_scores, what=""):
    got_ids = np.asarray(got_ids, np.uint64)
    want_ids = np.asarray(want_ids, np.uint64)
    got_s = np.asarray(got_scores, np.float64)
    want_s = np.asarray(want_scores, np.float64)
    assert len(got_ids) == len(want_ids), f"{what}: length {len(got_ids)} != {len(want_ids)}"
    assert (got_ids == want_ids).all(), f"{what}: ids {got_ids} != {want_ids}"
    assert (got_s.view(np.uint64) == want_s.view(np.uint64)).all(), \
        f"{what}: scores {got_s.tolist()} != {want_s.tolist()}"


def check_batch(got, ids, sc, n, post=None, tau=0.10, what="batch"):
    """GPU batch result == oracle arrays, bit-exact, plus margin/skip."""
    assert (got["n"] == n).all(), f"{what}: counts differ at {np.nonzero(got['n'] != n)[0][:10]}"
    for i in range(len(n)):
        m = int(n[i])
        assert_same(got["ids"][i, :m], got["scores"][i, :m], ids[i, :m], sc[i, :m],
                    f"{what} query {i}")
        conf = restate.margin(sc[i, :m])
        assert got["conf"][i] == conf, f"{what} query {i}: conf {got['conf'][i]} != {conf}"
        assert bool(got["skip"][i]) == (conf >= tau), f"{what} query {i}: skip"
    if post is not None:
        assert (got["postings"] == post).all(), f"{what}: postings_touched differ"


def synth_setup(n_records, vocab, lo, hi, n_queries, min_terms=3, max_terms=6, k1=1.2, b=0.75,
                row_order=None):
    corpus = synth.Corpus(n_records=n_records, vocab_size=vocab, min_doc_tokens=lo,
                          max_doc_tokens=hi)
    queries = synth.Queries(corpus, n_queries=n_queries, min_terms=min_terms,
                            max_terms=max_terms)
    hx = synth.HostIndex(corpus, k1=k1, b=b, row_order=row_order)
    tids = [hx.resolve(queries.term_ranks[queries.offsets[i]:queries.offsets[i + 1]])
            for i in range(len(queries))]
    return corpus, queries, hx, tids


def ndcg10(ids_row, gold):
    return restate.ndcg(ids_row, {int(gold): 1}, 10)


__all__ = ["toy_docs", "random_instance", "export_to_csr", "assert_same", "check_batch",
           "synth_setup", "ndcg10", "ref", "restate", "search", "synth"]
