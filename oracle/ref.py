"""TEST INFRASTRUCTURE ONLY: ctypes handle on the UNMODIFIED reference library.

oracle/_ref/libhybridref.so is compiled by oracle/Makefile from the reference
sources where they lie (/root/reference/proj/src) plus oracle/ref_shim.cpp.
Only tests/, __graft_entry__.smoke() and bench.py's CPU baseline use this.
"""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libhybridref.so")
_L = None

TOK_MINIMAL, TOK_STOPWORD, TOK_FULL, TOK_PORTER = 0, 1, 2, 3


def available():
    return os.path.exists(LIB_PATH)


def lib():
    global _L
    if _L is not None:
        return _L
    if not available():
        raise ImportError(f"{LIB_PATH} missing: run `make -C oracle` where /root/reference exists")
    L = C.CDLL(LIB_PATH)
    vp, u64, u32, i64, dbl = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int64, C.c_double
    P = C.POINTER
    L.ref_last_error.restype = C.c_char_p
    L.ref_gen_corpus.argtypes = [u64, u64, u32, dbl, u32, u32, i64, P(vp)]
    L.ref_corpus_size.argtypes = [vp]
    L.ref_corpus_size.restype = u64
    L.ref_corpus_text_bytes.argtypes = [vp]
    L.ref_corpus_text_bytes.restype = u64
    L.ref_corpus_export.argtypes = [vp, P(u64), P(i64), C.c_char_p]
    L.ref_corpus_free.argtypes = [vp]
    L.ref_gen_queries.argtypes = [vp, u64, u32, u32, u64, P(vp)]
    L.ref_queries_size.argtypes = [vp]
    L.ref_queries_size.restype = u64
    L.ref_queries_text_bytes.argtypes = [vp]
    L.ref_queries_text_bytes.restype = u64
    L.ref_queries_export.argtypes = [vp, P(u32), P(u64), P(i64), C.c_char_p]
    L.ref_queries_free.argtypes = [vp]
    L.ref_build_index_texts.argtypes = [u64, P(u64), P(C.c_char_p), C.c_int, dbl, dbl, P(vp)]
    L.ref_build_index_corpus.argtypes = [vp, C.c_int, dbl, dbl, P(vp)]
    L.ref_index_from_arrays.argtypes = [u32, P(C.c_char_p), P(u64), P(u32), P(dbl), P(dbl),
                                        P(dbl), P(dbl), u32, P(u32), P(u64), dbl, dbl, dbl, P(vp)]
    L.ref_index_free.argtypes = [vp]
    L.ref_save_index.argtypes = [vp, C.c_char_p]
    L.ref_save_temporal.argtypes = [vp, C.c_char_p]
    L.ref_load_temporal.argtypes = [C.c_char_p, P(vp)]
    L.ref_load_index.argtypes = [C.c_char_p, P(vp)]
    L.ref_index_sizes.argtypes = [vp, P(u64)]
    L.ref_index_export.argtypes = [vp, C.c_char_p, P(u64), P(u32), P(dbl), P(dbl), P(dbl),
                                   P(dbl), P(u32), P(u64), P(dbl)]
    L.ref_search.argtypes = [vp, P(C.c_char_p), u32, u64, dbl, dbl, C.c_int, P(u64), P(dbl),
                             P(u32), P(u64)]
    L.ref_search_batch.argtypes = [vp, u32, P(u32), P(C.c_char_p), u64, dbl, dbl, C.c_int,
                                   C.c_uint, C.c_uint, P(u64), P(dbl), P(u32), P(u64), P(dbl),
                                   P(dbl)]
    L.ref_build_temporal.argtypes = [u64, P(u64), P(i64), P(C.c_char_p), i64, dbl, dbl, u32,
                                     C.c_int, dbl, dbl, P(vp)]
    L.ref_build_temporal_corpus.argtypes = [vp, i64, dbl, dbl, u32, C.c_int, dbl, dbl, P(vp)]
    L.ref_temporal_from_flat.argtypes = [u32, P(C.c_char_p), P(u64), P(u32), P(dbl), P(dbl), P(dbl), P(u32),
                                         P(u64), dbl, u32, P(u32), i64, i64, dbl, dbl, u32, dbl, dbl, P(vp)]
    L.ref_temporal_free.argtypes = [vp]
    L.ref_temporal_num_partitions.argtypes = [vp]
    L.ref_temporal_num_partitions.restype = u32
    L.ref_temporal_partitions.argtypes = [vp, P(i64), P(i64), P(u32)]
    L.ref_temporal_topk.argtypes = [vp, P(C.c_char_p), u32, u64, dbl, dbl, C.c_int, P(u64),
                                    P(dbl), P(u32), P(u32), P(u64)]
    L.ref_temporal_batch.argtypes = [vp, u32, P(u32), P(C.c_char_p), u64, dbl, dbl, C.c_uint,
                                     P(u64), P(dbl), P(u32), P(dbl)]
    L.ref_bm25_score.argtypes = [dbl] * 6
    L.ref_bm25_score.restype = dbl
    L.ref_confidence.argtypes = [P(dbl), u32, C.c_int, dbl, P(dbl)]
    L.ref_k_star.argtypes = [dbl, dbl, P(u32)]
    L.ref_ndcg.argtypes = [P(u64), P(dbl), u32, P(u64), P(u32), u32, u64, C.c_int, P(dbl)]
    L.ref_twophase_batch.argtypes = [u64, C.c_int, u32, u32, P(dbl), u64, P(u64), P(dbl), P(u32)]
    L.ref_bridge_ingest.argtypes = [u32, P(u64), P(u64), P(u32), P(dbl), P(vp)]
    L.ref_bridge_export.argtypes = [vp, P(u64), P(u64), P(u32), P(dbl)]
    L.ref_sparse_validate.argtypes = [P(u32), u32, P(dbl), u32]
    L.ref_bridge_batch.argtypes = [vp, u32, P(u64), P(u32), P(dbl), u64, C.c_int, C.c_uint,
                                   P(u64), P(dbl), P(u32), P(u64), P(dbl)]
    L.ref_bm25_on.argtypes = [vp, C.c_char_p]
    L.ref_hash_embed.argtypes = [C.c_char_p, u32, u64, P(C.c_float)]
    L.ref_dense_batch.argtypes = [u32, u64, P(C.c_float), P(u64), u32, u32, P(C.c_float), u64, C.c_uint,
                                  P(u64), P(dbl), P(u32), P(dbl)]
    L.ref_save_embeddings.argtypes = [u32, u64, P(C.c_float), P(u64), C.c_char_p]
    L.ref_agent_rrf.argtypes = [P(u64), P(dbl), u32, P(u64), P(dbl), u32, P(u64), P(i64), P(dbl), u32,
                                i64, C.c_char_p, dbl, dbl, i64, dbl, u64, P(u64), P(dbl), P(u32)]
    L.ref_bridge_from_arrays.argtypes = [u32, P(u64), P(u32), P(dbl), u32, P(u64), P(u32), dbl, P(vp)]
    _L = L
    return L


def _chk(rc):
    if rc != 0:
        raise RuntimeError(lib().ref_last_error().decode())


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _cstrs(strs):
    arr = (C.c_char_p * max(1, len(strs)))()
    arr[:len(strs)] = [s.encode() for s in strs]
    return arr


def _split(buf, n):
    parts = bytes(buf).split(b"\0")
    return [p.decode() for p in parts[:n]]


class RefCorpus:
    def __init__(self, n_records, seed=42, vocab_size=5000, zipf_s=1.1, min_tok=5, max_tok=30,
                 time_span_ms=0):
        h = C.c_void_p()
        _chk(lib().ref_gen_corpus(n_records, seed, vocab_size, zipf_s, min_tok, max_tok,
                                  time_span_ms, C.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_corpus_free(self.h)

    def export(self):
        L = lib()
        n = L.ref_corpus_size(self.h)
        ids = np.zeros(n, np.uint64)
        ts = np.zeros(n, np.int64)
        buf = C.create_string_buffer(int(L.ref_corpus_text_bytes(self.h)))
        L.ref_corpus_export(self.h, _p(ids, C.c_uint64), _p(ts, C.c_int64), buf)
        return ids, ts, _split(buf.raw, n)


class RefQueries:
    def __init__(self, corpus, n_queries=1000, min_terms=3, max_terms=6, seed=42):
        h = C.c_void_p()
        _chk(lib().ref_gen_queries(corpus.h, n_queries, min_terms, max_terms, seed, C.byref(h)))
        L = lib()
        n = L.ref_queries_size(h)
        nt = np.zeros(n, np.uint32)
        gold = np.zeros(n, np.uint64)
        ts = np.zeros(n, np.int64)
        buf = C.create_string_buffer(int(L.ref_queries_text_bytes(h)) + 1)
        L.ref_queries_export(h, _p(nt, C.c_uint32), _p(gold, C.c_uint64), _p(ts, C.c_int64), buf)
        flat = _split(buf.raw, int(nt.sum()))
        off = np.concatenate([[0], np.cumsum(nt)]).astype(np.int64)
        self.terms = [flat[off[i]:off[i + 1]] for i in range(n)]
        self.gold, self.ts = gold, ts
        L.ref_queries_free(h)


class RefIndex:
    """A reference hybrid::CsrIndex (built by the reference or adopted from arrays)."""

    def __init__(self, h):
        self.h = h

    @classmethod
    def from_texts(cls, docs, tok_mode=TOK_MINIMAL, k1=1.2, b=0.75):
        ids = np.array([d for d, _ in docs], dtype=np.uint64)
        texts = _cstrs([t for _, t in docs])
        h = C.c_void_p()
        _chk(lib().ref_build_index_texts(len(docs), _p(ids, C.c_uint64), texts, tok_mode, k1, b,
                                         C.byref(h)))
        return cls(h)

    @classmethod
    def from_corpus(cls, corpus, tok_mode=TOK_STOPWORD, k1=1.2, b=0.75):
        h = C.c_void_p()
        _chk(lib().ref_build_index_corpus(corpus.h, tok_mode, k1, b, C.byref(h)))
        return cls(h)

    @classmethod
    def from_arrays(cls, terms, term_offsets, posting_rows, posting_weights, idf, maxscore,
                    order_key, doc_lens, doc_ids, avgdl, k1=1.2, b=0.75):
        keep = [np.ascontiguousarray(term_offsets, np.uint64),
                np.ascontiguousarray(posting_rows, np.uint32),
                np.ascontiguousarray(posting_weights, np.float64),
                np.ascontiguousarray(idf, np.float64), np.ascontiguousarray(maxscore, np.float64),
                np.ascontiguousarray(order_key, np.float64),
                np.ascontiguousarray(doc_lens, np.uint32), np.ascontiguousarray(doc_ids, np.uint64)]
        h = C.c_void_p()
        _chk(lib().ref_index_from_arrays(
            len(terms), _cstrs(terms), _p(keep[0], C.c_uint64), _p(keep[1], C.c_uint32),
            _p(keep[2], C.c_double), _p(keep[3], C.c_double), _p(keep[4], C.c_double),
            _p(keep[5], C.c_double), len(doc_ids), _p(keep[6], C.c_uint32),
            _p(keep[7], C.c_uint64), avgdl, k1, b, C.byref(h)))
        return cls(h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_index_free(self.h)

    def save(self, path):
        """hybrid::save_index (io.cpp:223-227): a HIDX v1 file."""
        _chk(lib().ref_save_index(self.h, str(path).encode()))

    @classmethod
    def load(cls, path):
        """hybrid::load_index (io.cpp:229-232)."""
        h = C.c_void_p()
        _chk(lib().ref_load_index(str(path).encode(), C.byref(h)))
        return cls(h)

    def export(self):
        L = lib()
        s = np.zeros(4, np.uint64)
        L.ref_index_sizes(self.h, _p(s, C.c_uint64))
        nt, npst, nd, tb = (int(x) for x in s)
        out = dict(term_offsets=np.zeros(nt + 1, np.uint64), posting_rows=np.zeros(npst, np.uint32),
                   posting_weights=np.zeros(npst, np.float64), idf=np.zeros(nt, np.float64),
                   maxscore=np.zeros(nt, np.float64), order_key=np.zeros(nt, np.float64),
                   doc_lens=np.zeros(nd, np.uint32), doc_ids=np.zeros(nd, np.uint64))
        buf = C.create_string_buffer(tb + 1)
        avg = C.c_double()
        L.ref_index_export(self.h, buf, _p(out["term_offsets"], C.c_uint64),
                           _p(out["posting_rows"], C.c_uint32),
                           _p(out["posting_weights"], C.c_double), _p(out["idf"], C.c_double),
                           _p(out["maxscore"], C.c_double), _p(out["order_key"], C.c_double),
                           _p(out["doc_lens"], C.c_uint32), _p(out["doc_ids"], C.c_uint64),
                           C.byref(avg))
        out["terms"] = _split(buf.raw, nt)
        out["avgdl"] = avg.value
        return out

    def search(self, terms, k, k1=1.2, b=0.75, maxscore=False):
        """-> (ids, scores, postings_touched)"""
        cap = max(int(k), 1)
        ids = np.zeros(cap, np.uint64)
        sc = np.zeros(cap, np.float64)
        n = C.c_uint32()
        post = C.c_uint64()
        _chk(lib().ref_search(self.h, _cstrs(terms), len(terms), k, k1, b, 1 if maxscore else 0,
                              _p(ids, C.c_uint64), _p(sc, C.c_double), C.byref(n), C.byref(post)))
        return ids[:n.value].copy(), sc[:n.value].copy(), post.value

    def search_batch(self, queries, k, k1=1.2, b=0.75, maxscore=False, workers=1, warmup=0):
        """CLI-shaped parallel batch (hybridmem.cpp:58-71, 305-313).
        -> dict(ids[nq,k], scores[nq,k], n[nq], postings[nq], lat_ms[nq], wall_ms)"""
        nq = len(queries)
        flat = [t for q in queries for t in q]
        off = np.zeros(nq + 1, np.uint32)
        off[1:] = np.cumsum([len(q) for q in queries])
        ids = np.zeros((nq, k), np.uint64)
        sc = np.zeros((nq, k), np.float64)
        n = np.zeros(nq, np.uint32)
        post = np.zeros(nq, np.uint64)
        lat = np.zeros(nq, np.float64)
        wall = C.c_double()
        _chk(lib().ref_search_batch(self.h, nq, _p(off, C.c_uint32), _cstrs(flat), k, k1, b,
                                    1 if maxscore else 0, workers, warmup, _p(ids, C.c_uint64),
                                    _p(sc, C.c_double), _p(n, C.c_uint32), _p(post, C.c_uint64),
                                    _p(lat, C.c_double), C.byref(wall)))
        return dict(ids=ids, scores=sc, n=n, postings=post, lat_ms=lat, wall_ms=wall.value)



def sparse_pack(vectors):
    """[(indices, values), ...] -> (off u64[n+1], idx u32[nnz], val f64[nnz])"""
    off = np.zeros(len(vectors) + 1, np.uint64)
    off[1:] = np.cumsum([len(i) for i, _ in vectors])
    idx = np.concatenate([np.asarray(i, np.uint32) for i, _ in vectors]) if vectors else np.zeros(0, np.uint32)
    val = np.concatenate([np.asarray(v, np.float64) for _, v in vectors]) if vectors else np.zeros(0)
    return off, np.ascontiguousarray(idx, np.uint32), np.ascontiguousarray(val, np.float64)


def sparse_validate(indices, values):
    """SparseVector::validate (bridge.cpp:10-20); raises RuntimeError(message)."""
    i = np.ascontiguousarray(indices, np.uint32)
    v = np.ascontiguousarray(values, np.float64)
    _chk(lib().ref_sparse_validate(_p(i, C.c_uint32), len(i), _p(v, C.c_double), len(v)))


class RefBridge(RefIndex):
    """A reference Bridge-mode CsrIndex (bridge.cpp:22-73)."""

    @classmethod
    def from_vectors(cls, ids, vectors):
        """bridge_ingest over docs (ids[d], (indices, values))."""
        ids = np.ascontiguousarray(ids, np.uint64)
        off, idx, val = sparse_pack(vectors)
        h = C.c_void_p()
        _chk(lib().ref_bridge_ingest(len(ids), _p(ids, C.c_uint64), _p(off, C.c_uint64),
                                     _p(idx, C.c_uint32), _p(val, C.c_double), C.byref(h)))
        return cls(h)

    @classmethod
    def from_csr(cls, term_offsets, posting_rows, posting_weights, doc_ids, doc_lens, avgdl):
        """Adopt bridge_ingest-shaped CSR arrays (timing workloads)."""
        a = [np.ascontiguousarray(term_offsets, np.uint64), np.ascontiguousarray(posting_rows, np.uint32),
             np.ascontiguousarray(posting_weights, np.float64), np.ascontiguousarray(doc_ids, np.uint64),
             np.ascontiguousarray(doc_lens, np.uint32)]
        h = C.c_void_p()
        _chk(lib().ref_bridge_from_arrays(len(a[0]) - 1, _p(a[0], C.c_uint64), _p(a[1], C.c_uint32),
                                          _p(a[2], C.c_double), len(a[3]), _p(a[3], C.c_uint64),
                                          _p(a[4], C.c_uint32), avgdl, C.byref(h)))
        return cls(h)

    def export_vectors(self):
        """bridge_export (bridge.cpp:75-90) -> (ids, off, idx, val)"""
        x = self.export()
        nd, nnz = len(x["doc_ids"]), len(x["posting_rows"])
        ids = np.zeros(nd, np.uint64)
        off = np.zeros(nd + 1, np.uint64)
        idx = np.zeros(max(nnz, 1), np.uint32)
        val = np.zeros(max(nnz, 1), np.float64)
        _chk(lib().ref_bridge_export(self.h, _p(ids, C.c_uint64), _p(off, C.c_uint64),
                                     _p(idx, C.c_uint32), _p(val, C.c_double)))
        return ids, off, idx[:nnz], val[:nnz]

    def topk_batch(self, queries, k, maxscore=False, workers=1):
        """bridge_topk / bridge_topk_maxscore per query (bridge.cpp:112-204).
        -> dict(ids[nq,k], scores[nq,k], n[nq], postings[nq], wall_ms)"""
        nq = len(queries)
        off, idx, val = sparse_pack(queries)
        cap = max(int(k), 1)
        ids = np.zeros((nq, cap), np.uint64)
        sc = np.zeros((nq, cap), np.float64)
        n = np.zeros(nq, np.uint32)
        post = np.zeros(nq, np.uint64)
        wall = C.c_double()
        _chk(lib().ref_bridge_batch(self.h, nq, _p(off, C.c_uint64), _p(idx, C.c_uint32),
                                    _p(val, C.c_double), k, 1 if maxscore else 0, workers,
                                    _p(ids, C.c_uint64), _p(sc, C.c_double), _p(n, C.c_uint32),
                                    _p(post, C.c_uint64), C.byref(wall)))
        return dict(ids=ids, scores=sc, n=n, postings=post, wall_ms=wall.value)

    def bm25_error(self):
        """CsrIndex::bm25_topk on this index: the reference's refusal message."""
        rc = lib().ref_bm25_on(self.h, b"t0")
        return lib().ref_last_error().decode() if rc else None


def hash_embed(text, dim, seed):
    """hybrid::hash_embed (dense.cpp:54-84)."""
    out = np.zeros(dim, np.float32)
    _chk(lib().ref_hash_embed(text.encode(), dim, seed, _p(out, C.c_float)))
    return out


def dense_topk_batch(data, ids, queries, k, workers=1):
    """hybrid::dense_topk per query (dense.cpp:86-101) over the matrix
    (data [count x dim] fp32, ids).  -> dict(ids, scores, n, wall_ms)"""
    data = np.ascontiguousarray(data, np.float32)
    ids = np.ascontiguousarray(ids, np.uint64)
    queries = np.ascontiguousarray(queries, np.float32)
    nq, qdim = queries.shape
    cap = max(int(k), 1)
    o_ids = np.zeros((nq, cap), np.uint64)
    o_sc = np.zeros((nq, cap), np.float64)
    o_n = np.zeros(nq, np.uint32)
    wall = C.c_double()
    _chk(lib().ref_dense_batch(data.shape[1] if data.ndim == 2 else qdim, len(ids), _p(data, C.c_float),
                               _p(ids, C.c_uint64), nq, qdim, _p(queries, C.c_float), k, workers,
                               _p(o_ids, C.c_uint64), _p(o_sc, C.c_double), _p(o_n, C.c_uint32), C.byref(wall)))
    return dict(ids=o_ids, scores=o_sc, n=o_n, wall_ms=wall.value)


def save_embeddings(data, ids, path):
    """hybrid::save_embeddings (dense.cpp:103-118): a HEMB v1 file."""
    data = np.ascontiguousarray(data, np.float32)
    ids = np.ascontiguousarray(ids, np.uint64)
    _chk(lib().ref_save_embeddings(data.shape[1], len(ids), _p(data, C.c_float), _p(ids, C.c_uint64),
                                   str(path).encode()))


def agent_rrf(sparse, dense, records, query_ts, qtype=None, k_rrf=60.0, alpha=0.005,
              tau_ms=30 * 24 * 3600 * 1000, beta=0.0):
    """hybrid::agent_rrf (fusion.cpp:22-50).  sparse/dense: [(id, score)];
    records: {id: (ts_ms, weight)}.  -> [(id, score)] ranked."""
    s_ids = np.array([d for d, _ in sparse] or [0], np.uint64)
    s_sc = np.array([x for _, x in sparse] or [0.0])
    d_ids = np.array([d for d, _ in dense] or [0], np.uint64)
    d_sc = np.array([x for _, x in dense] or [0.0])
    r_ids = np.array(list(records) or [0], np.uint64)
    r_ts = np.array([records[r][0] for r in records] or [0], np.int64)
    r_w = np.array([records[r][1] for r in records] or [0.0])
    cap = len(sparse) + len(dense) + 1
    o_ids = np.zeros(cap, np.uint64)
    o_sc = np.zeros(cap)
    n = C.c_uint32()
    _chk(lib().ref_agent_rrf(_p(s_ids, C.c_uint64), _p(s_sc, C.c_double), len(sparse), _p(d_ids, C.c_uint64),
                             _p(d_sc, C.c_double), len(dense), _p(r_ids, C.c_uint64), _p(r_ts, C.c_int64),
                             _p(r_w, C.c_double), len(records), query_ts,
                             None if qtype is None else qtype.encode(), k_rrf, alpha, tau_ms, beta, cap,
                             _p(o_ids, C.c_uint64), _p(o_sc, C.c_double), C.byref(n)))
    return [(int(o_ids[i]), float(o_sc[i])) for i in range(n.value)]


class RefTemporal:
    def __init__(self, h):
        self.h = h

    @classmethod
    def from_records(cls, ids, ts, texts, window_ms=7 * 24 * 3600 * 1000, epsilon=0.05,
                     lambda_hat=1.4, k_max=4, tok_mode=TOK_MINIMAL, k1=1.2, b=0.75):
        ids = np.ascontiguousarray(ids, np.uint64)
        ts = np.ascontiguousarray(ts, np.int64)
        h = C.c_void_p()
        _chk(lib().ref_build_temporal(len(ids), _p(ids, C.c_uint64), _p(ts, C.c_int64),
                                      _cstrs(texts), window_ms, epsilon, lambda_hat, k_max,
                                      tok_mode, k1, b, C.byref(h)))
        return cls(h)

    @classmethod
    def from_flat(cls, terms, term_offsets, posting_rows, posting_weights, idf, order_key, doc_lens, doc_ids,
                  avgdl, part_row, t0, window_ms=7 * 24 * 3600 * 1000, epsilon=0.05, lambda_hat=1.4, k_max=4,
                  k1=1.2, b=0.75):
        """A reference TemporalIndex assembled from a partition-ordered flat
        index (ref_temporal_from_flat): partitions share the flat statistics."""
        keep = [np.ascontiguousarray(term_offsets, np.uint64), np.ascontiguousarray(posting_rows, np.uint32),
                np.ascontiguousarray(posting_weights, np.float64), np.ascontiguousarray(idf, np.float64),
                np.ascontiguousarray(order_key, np.float64), np.ascontiguousarray(doc_lens, np.uint32),
                np.ascontiguousarray(doc_ids, np.uint64), np.ascontiguousarray(part_row, np.uint32)]
        h = C.c_void_p()
        _chk(lib().ref_temporal_from_flat(
            len(terms), _cstrs(terms), _p(keep[0], C.c_uint64), _p(keep[1], C.c_uint32), _p(keep[2], C.c_double),
            _p(keep[3], C.c_double), _p(keep[4], C.c_double), _p(keep[5], C.c_uint32), _p(keep[6], C.c_uint64),
            avgdl, len(keep[7]) - 1, _p(keep[7], C.c_uint32), int(t0), window_ms, epsilon, lambda_hat, k_max,
            k1, b, C.byref(h)))
        return cls(h)

    @classmethod
    def from_corpus(cls, corpus, window_ms=7 * 24 * 3600 * 1000, epsilon=0.05, lambda_hat=1.4,
                    k_max=4, tok_mode=TOK_STOPWORD, k1=1.2, b=0.75):
        h = C.c_void_p()
        _chk(lib().ref_build_temporal_corpus(corpus.h, window_ms, epsilon, lambda_hat, k_max,
                                             tok_mode, k1, b, C.byref(h)))
        return cls(h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_temporal_free(self.h)

    def save(self, path):
        """hybrid::save_temporal_index (io.cpp:234-268): a HTIX v1 file."""
        _chk(lib().ref_save_temporal(self.h, str(path).encode()))

    @classmethod
    def load(cls, path):
        """hybrid::load_temporal_index (io.cpp:270-318)."""
        h = C.c_void_p()
        _chk(lib().ref_load_temporal(str(path).encode(), C.byref(h)))
        return cls(h)

    def partitions(self):
        K = lib().ref_temporal_num_partitions(self.h)
        ws = np.zeros(K, np.int64)
        we = np.zeros(K, np.int64)
        nd = np.zeros(K, np.uint32)
        lib().ref_temporal_partitions(self.h, _p(ws, C.c_int64), _p(we, C.c_int64),
                                      _p(nd, C.c_uint32))
        return ws, we, nd

    def topk(self, terms, k, k1=1.2, b=0.75, use_ub_stop=True):
        cap = max(int(k), 1)
        ids = np.zeros(cap, np.uint64)
        sc = np.zeros(cap, np.float64)
        n = C.c_uint32()
        srch = C.c_uint32()
        post = C.c_uint64()
        _chk(lib().ref_temporal_topk(self.h, _cstrs(terms), len(terms), k, k1, b,
                                     1 if use_ub_stop else 0, _p(ids, C.c_uint64),
                                     _p(sc, C.c_double), C.byref(n), C.byref(srch), C.byref(post)))
        return ids[:n.value].copy(), sc[:n.value].copy(), srch.value, post.value

    def topk_batch(self, queries, k, k1=1.2, b=0.75, workers=1):
        nq = len(queries)
        flat = [t for q in queries for t in q]
        off = np.zeros(nq + 1, np.uint32)
        off[1:] = np.cumsum([len(q) for q in queries])
        ids = np.zeros((nq, k), np.uint64)
        sc = np.zeros((nq, k), np.float64)
        n = np.zeros(nq, np.uint32)
        wall = C.c_double()
        _chk(lib().ref_temporal_batch(self.h, nq, _p(off, C.c_uint32), _cstrs(flat), k, k1, b,
                                      workers, _p(ids, C.c_uint64), _p(sc, C.c_double),
                                      _p(n, C.c_uint32), C.byref(wall)))
        return dict(ids=ids, scores=sc, n=n, wall_ms=wall.value)


def bm25_score(tf, idf, dl, avgdl, k1=1.2, b=0.75):
    return lib().ref_bm25_score(tf, idf, dl, avgdl, k1, b)


def confidence(scores, proxy=0, eps=1e-9):
    s = np.ascontiguousarray(scores, np.float64)
    out = C.c_double()
    _chk(lib().ref_confidence(_p(s, C.c_double), len(s), proxy, eps, C.byref(out)))
    return out.value


def k_star(eps, lam):
    out = C.c_uint32()
    _chk(lib().ref_k_star(eps, lam, C.byref(out)))
    return out.value


def ndcg(ids, rels, k, linear=False):
    ids = np.ascontiguousarray(ids, np.uint64)
    sc = np.zeros(len(ids), np.float64)
    rd = np.array(list(rels.keys()), np.uint64)
    rg = np.array(list(rels.values()), np.uint32)
    out = C.c_double()
    _chk(lib().ref_ndcg(_p(ids, C.c_uint64), _p(sc, C.c_double), len(ids), _p(rd, C.c_uint64),
                        _p(rg, C.c_uint32), len(rd), k, 1 if linear else 0, C.byref(out)))
    return out.value


def twophase_batch(rows, k, capacity, reset_sentinel=True):
    rows = np.ascontiguousarray(rows, np.float64)
    r, n = rows.shape
    ids = np.zeros((r, k), np.uint64)
    sc = np.zeros((r, k), np.float64)
    cnt = np.zeros(r, np.uint32)
    _chk(lib().ref_twophase_batch(capacity, 1 if reset_sentinel else 0, r, n,
                                  _p(rows, C.c_double), k, _p(ids, C.c_uint64), _p(sc, C.c_double),
                                  _p(cnt, C.c_uint32)))
    return ids, sc, cnt
