"""CPU: the native generator/builder (hm_synth) is bit-identical to the
reference's gen_corpus / gen_queries / build_index / build_temporal_index
(proj/src/workload.cpp:47-135, csr_index.cpp:232-324, temporal_index.cpp:125-169)."""
import numpy as np
import pytest

from oracle import ref
from paper_2605_25092_b200 import synth

pytestmark = pytest.mark.skipif(not ref.available(), reason="reference library not built")


@pytest.mark.parametrize("n,V,lo,hi,q_lo,q_hi", [(3000, 5000, 5, 30, 3, 6),
                                                  (20000, 100000, 20, 60, 3, 6),
                                                  (4000, 50000, 40, 80, 24, 32),
                                                  (1, 10, 1, 1, 1, 2)])
def test_generator_and_builder_bit_identical(n, V, lo, hi, q_lo, q_hi):
    rc = ref.RefCorpus(n, vocab_size=V, min_tok=lo, max_tok=hi)
    ids, ts, texts = rc.export()
    c = synth.Corpus(n_records=n, vocab_size=V, min_doc_tokens=lo, max_doc_tokens=hi, threads=3)
    _, _, ts2 = c.arrays()
    assert (ts == ts2).all() and (ids == np.arange(n)).all()
    assert c.texts() == texts
    rq = ref.RefQueries(rc, 300, q_lo, q_hi)
    q = synth.Queries(c, n_queries=300, min_terms=q_lo, max_terms=q_hi)
    assert all(q.terms(i) == rq.terms[i] for i in range(300))
    assert (q.gold == rq.gold).all() and (q.ts == rq.ts).all()
    e = ref.RefIndex.from_corpus(rc).export()
    hx = synth.HostIndex(c, threads=5)
    assert e["terms"] == hx.term_strings()
    for key in ["term_offsets", "posting_rows", "idf", "maxscore", "order_key", "doc_lens",
                "doc_ids"]:
        a, b = e[key], getattr(hx, key)
        assert a.dtype == b.dtype and a.tobytes() == b.tobytes(), key
    assert (e["posting_weights"] == hx.posting_tf).all() and e["avgdl"] == hx.avgdl


def test_thread_count_independence():
    c1 = synth.Corpus(n_records=70000, threads=1)
    c8 = synth.Corpus(n_records=70000, threads=8)
    for a, b in zip(c1.arrays(), c8.arrays()):
        assert (a == b).all()
    h1, h8 = synth.HostIndex(c1, threads=1), synth.HostIndex(c8, threads=8)
    for key in ["term_offsets", "posting_rows", "posting_tf", "idf", "maxscore"]:
        assert getattr(h1, key).tobytes() == getattr(h8, key).tobytes()


def test_constant_arrival_partitions_match_reference():
    """Partition bucketing of build_temporal_index (temporal_index.cpp:144-157)
    at the constant-arrival span of acceptance.cpp:101-104."""
    n = 20000
    span = int(28 * 24 * 3600 * 1000 * n / 4052)
    rc = ref.RefCorpus(n, time_span_ms=span)
    rt = ref.RefTemporal.from_corpus(rc, tok_mode=ref.TOK_STOPWORD)
    ws, we, nd = rt.partitions()
    c = synth.Corpus(n_records=n, time_span_ms=span)
    K, order, part, t0 = c.partition(7 * 24 * 3600 * 1000)
    assert K == len(ws) and t0 == ws[0]
    assert (np.diff(part) == nd).all()
    _, _, ts = c.arrays()
    # rows in partition order, insertion order kept inside a partition
    for j in range(K):
        rec = order[part[j]:part[j + 1]]
        assert (np.diff(rec.astype(np.int64)) > 0).all()
        assert ((ts[rec] >= ws[j]) & (ts[rec] < we[j])).all()


def test_permuted_build_keeps_global_statistics():
    c = synth.Corpus(n_records=30000, time_span_ms=int(28 * 24 * 3600 * 1000 * 30000 / 4052))
    K, order, part, _ = c.partition(7 * 24 * 3600 * 1000)
    flat = synth.HostIndex(c)
    perm = synth.HostIndex(c, row_order=order)
    assert flat.idf.tobytes() == perm.idf.tobytes()
    assert flat.order_key.tobytes() == perm.order_key.tobytes()
    assert flat.avgdl == perm.avgdl
    assert (perm.doc_ids == order).all()
    assert (perm.doc_lens == flat.doc_lens[order]).all()


def test_generator_rejects_bad_specs():
    with pytest.raises(RuntimeError):
        synth.Corpus(n_records=0)
    with pytest.raises(RuntimeError):
        synth.Corpus(n_records=10, min_doc_tokens=9, max_doc_tokens=3)
