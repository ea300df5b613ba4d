"""The reference's on-disk index (HIDX v1, proj/src/io.cpp:91-157, 223-232)
through the framework's native reader (hm_hidx_*).

Files are written by the UNMODIFIED reference (oracle/_ref: hybrid::save_index);
the reader must reproduce hybrid::load_index -- every array bit for bit, the
same rejections with the same messages (test_config_io.cpp:116-152 pins the
reference's truncation behaviour) -- and an index uploaded straight from the
file must search exactly like the reference on it.
"""
import struct

import numpy as np
import pytest

from _util import random_instance, ref, search, toy_docs

KEYS = ("term_offsets", "posting_rows", "posting_weights", "idf", "maxscore", "order_key",
        "doc_lens", "doc_ids")


def _ref_error(path):
    try:
        ref.RefIndex.load(path)
    except RuntimeError as e:
        return str(e)
    return None


def _our_error(path):
    try:
        search.Hidx(path)
    except RuntimeError as e:
        return str(e)
    return None


def test_hidx_arrays_identical_to_reference_load(tmp_path):
    rng = np.random.default_rng(7)
    for trial in range(20):
        docs, _ = random_instance(rng)
        ri = ref.RefIndex.from_texts(docs, ref.TOK_MINIMAL, k1=1.2 + 0.1 * (trial % 3), b=0.75)
        p = tmp_path / f"r{trial}.hidx"
        ri.save(p)
        want = ref.RefIndex.load(p).export()
        h = search.Hidx(p)
        got = h.arrays()
        assert h.terms() == want["terms"]
        for k in KEYS:
            assert got[k].dtype == want[k].dtype and (got[k].view(np.uint8) == want[k].view(np.uint8)).all(), k
        assert struct.pack("<d", got["avgdl"]) == struct.pack("<d", want["avgdl"])
        assert h.mode == 0 and abs(h.build_params.k1 - (1.2 + 0.1 * (trial % 3))) < 1e-12


def test_hidx_rejections_match_reference(tmp_path):
    ri = ref.RefIndex.from_texts(toy_docs(), ref.TOK_MINIMAL)
    good = tmp_path / "toy.hidx"
    ri.save(good)
    data = good.read_bytes()
    cases = {
        "magic": b"HIDY" + data[4:],
        "version": data[:4] + struct.pack("<I", 2) + data[8:],
        "conv": data[:26] + b"X" + data[27:],  # a byte of the idf-convention string
        "empty": b"",
    }
    for cut in (3, 9, 30, 60, len(data) // 2, len(data) - 8, len(data) - 1):
        cases[f"cut{cut}"] = data[:cut]
    for name, blob in cases.items():
        p = tmp_path / f"bad_{name}.hidx"
        p.write_bytes(blob)
        want = _ref_error(p)
        assert want is not None, name
        assert _our_error(p) == want, (name, _our_error(p), want)
    missing = str(tmp_path / "nope.hidx")
    assert _our_error(missing) == _ref_error(missing) == "cannot open " + missing


def test_hidx_abi_exports():
    L = search.lib()
    for sym in ("hm_hidx_load", "hm_hidx_view", "hm_hidx_term", "hm_hidx_maxscores", "hm_hidx_free",
                "hm_hidx_last_error"):
        assert hasattr(L, sym), sym


@pytest.mark.gpu
def test_hidx_device_index_searches_like_reference(gpu, tmp_path):
    corpus = ref.RefCorpus(30000, vocab_size=3000)
    ri = ref.RefIndex.from_corpus(corpus)
    queries = ref.RefQueries(corpus, n_queries=300)
    p = tmp_path / "c.hidx"
    ri.save(p)
    dev = search.DeviceIndex.from_hidx(p)
    idx = search.CsrIndex.load(p)
    for q in queries.terms[:300]:
        want_ids, want_sc, want_post = ri.search(q, 10)
        r = dev.search_lists([idx.resolve(q)], 10)
        n = int(r["n"][0])
        assert r["ids"][0, :n].tolist() == list(want_ids)
        assert (r["scores"][0, :n].view(np.uint64) == np.asarray(want_sc).view(np.uint64)).all()
        assert int(r["postings"][0]) == want_post


# ---------------------------------------------------------------- HTIX v1
DAY = 24 * 3600 * 1000


def _records(seed, n=400, vocab=60, span_days=45):
    rng = np.random.default_rng(seed)
    ids = np.arange(1, n + 1, dtype=np.uint64) * 7
    ts = rng.integers(0, span_days * DAY, n).astype(np.int64)
    texts = [" ".join("w%d" % rng.integers(0, vocab) for _ in range(rng.integers(2, 14))) for _ in range(n)]
    return ids, ts, texts


def test_htix_assembles_the_partition_ordered_flat_index(tmp_path):
    """The flat index assembled from HTIX equals the reference's own flat
    build over the records in partition order (same shared statistics,
    temporal_index.cpp:136-142), array for array."""
    for seed in range(4):
        ids, ts, texts = _records(seed)
        rt = ref.RefTemporal.from_records(ids, ts, texts)
        p = tmp_path / f"t{seed}.htix"
        rt.save(p)
        h = search.Htix(p)
        ws, we, nd = rt.partitions()
        assert (h.window_start == ws).all() and (h.window_end == we).all()
        assert (np.diff(h.part_row.astype(np.int64)) == nd).all() and h.total_docs == len(ids)
        # records in partition order: window index, stable by insertion
        t0 = int(ts.min())
        order = np.argsort((ts - t0) // (7 * DAY), kind="stable")
        flat = ref.RefIndex.from_texts([(int(ids[r]), texts[r]) for r in order], ref.TOK_MINIMAL).export()
        got = h.flat.arrays()
        assert h.flat.terms() == flat["terms"]
        for k in ("term_offsets", "posting_rows", "posting_weights", "idf", "order_key", "doc_lens", "doc_ids"):
            assert (got[k].view(np.uint8) == flat[k].view(np.uint8)).all(), (seed, k)


def test_htix_rejections_match_reference(tmp_path):
    ids, ts, texts = _records(9)
    rt = ref.RefTemporal.from_records(ids, ts, texts)
    good = tmp_path / "t.htix"
    rt.save(good)
    data = good.read_bytes()

    def ref_err(path):
        try:
            ref.RefTemporal.load(path)
        except RuntimeError as e:
            return str(e)
        return None

    def our_err(path):
        try:
            search.Htix(path)
        except RuntimeError as e:
            return str(e)
        return None

    cases = {"magic": b"HTIY" + data[4:], "version": data[:4] + struct.pack("<I", 3) + data[8:]}
    for cut in (2, 10, 50, len(data) // 3, len(data) - 20, len(data) - 1):
        cases[f"cut{cut}"] = data[:cut]
    for name, blob in cases.items():
        p = tmp_path / f"bad_{name}.htix"
        p.write_bytes(blob)
        want = ref_err(p)
        assert want is not None and our_err(p) == want, (name, our_err(p), want)


@pytest.mark.gpu
def test_htix_temporal_search_like_reference(gpu, tmp_path):
    """TemporalIndex::topk (temporal_index.cpp:72-123) on a HTIX file, through
    the framework's temporal path (newest partitions as a row window)."""
    ids, ts, texts = _records(11, n=3000, vocab=200, span_days=60)
    rt = ref.RefTemporal.from_records(ids, ts, texts)
    p = tmp_path / "t.htix"
    rt.save(p)
    tix, idx = search.Htix(p).temporal_index()
    rng = np.random.default_rng(5)
    queries = [["w%d" % rng.integers(0, 220) for _ in range(rng.integers(1, 5))] for _ in range(200)]
    tids = [idx.resolve(q) for q in queries]
    off = np.concatenate([[0], np.cumsum([len(t) for t in tids])]).astype(np.uint32)
    got = tix.topk_batch(off, np.array([x for t in tids for x in t], np.uint32), 10)
    for i, q in enumerate(queries):
        want_ids, want_sc = rt.topk(q, 10)[:2]
        n = int(got["n"][i])
        assert got["ids"][i, :n].tolist() == list(want_ids), q
        assert (got["scores"][i, :n].view(np.uint64) == np.asarray(want_sc).view(np.uint64)).all(), q


@pytest.mark.gpu
def test_htix_temporal_topk_with_ub_stop_like_reference(gpu, tmp_path):
    """TemporalIndex.topk per query (temporal_index.cpp:72-123), newest
    partition first with the upper-bound stop: same list, same
    partitions_searched and early_stopped as the reference."""
    ids, ts, texts = _records(13, n=2500, vocab=120, span_days=90)
    for eps, kmax in ((0.05, 4), (1e-9, 64)):
        rt = ref.RefTemporal.from_records(ids, ts, texts, epsilon=eps, k_max=kmax)
        p = tmp_path / f"t{kmax}.htix"
        rt.save(p)
        tix, idx = search.Htix(p).temporal_index()
        rng = np.random.default_rng(kmax)
        for _ in range(40):
            q = ["w%d" % rng.integers(0, 130) for _ in range(rng.integers(1, 4))]
            k = int(rng.integers(1, 12))
            for ub in (True, False):
                st = search.TemporalStats()
                got = tix.topk(q, k, stats=st, use_ub_stop=ub)
                w_ids, w_sc, w_srch, _ = rt.topk(q, k, use_ub_stop=ub)
                assert [d for d, _ in got] == w_ids.tolist(), (q, k, ub)
                assert np.array([s for _, s in got]).view(np.uint64).tolist() == \
                    np.asarray(w_sc).view(np.uint64).tolist()
                assert st.partitions_searched == w_srch, (q, k, ub)
