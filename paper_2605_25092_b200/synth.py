"""Python handle over the native synthetic generator / CSR builder (hm_synth.h).

Mirrors hybrid::gen_corpus / gen_queries / build_index
(/root/reference/proj/src/workload.cpp:47-135, src/csr_index.cpp:232-324) for
the generator's Zipf "w<rank>" corpora, bit-identically, multithreaded.
"""
import ctypes as C

import numpy as np

from . import _lib

_L = None


class WSpec(C.Structure):
    _fields_ = [("n_records", C.c_uint64), ("seed", C.c_uint64),
                ("recency_mass", C.c_double), ("recency_window", C.c_double),
                ("vocab_size", C.c_uint32), ("zipf_s", C.c_double),
                ("min_doc_tokens", C.c_uint32), ("max_doc_tokens", C.c_uint32),
                ("n_sessions", C.c_uint32), ("n_agents", C.c_uint32),
                ("time_span_ms", C.c_int64), ("t0_ms", C.c_int64)]


class QSpec(C.Structure):
    _fields_ = [("n_queries", C.c_uint64), ("min_terms", C.c_uint32),
                ("max_terms", C.c_uint32), ("paraphrase_noise", C.c_double),
                ("seed", C.c_uint64)]


def _lib_handle():
    global _L
    if _L is not None:
        return _L
    L = _lib.load("libhm_synth.so")
    vp, u64, u32, i64, dbl = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int64, C.c_double
    L.hm_synth_last_error.restype = C.c_char_p
    L.hm_wspec_default.argtypes = [C.POINTER(WSpec)]
    L.hm_qspec_default.argtypes = [C.POINTER(QSpec)]
    L.hm_synth_corpus_create.argtypes = [C.POINTER(WSpec), C.c_int, C.POINTER(vp)]
    L.hm_synth_queries_create.argtypes = [vp, C.POINTER(QSpec), C.POINTER(vp)]
    L.hm_synth_build.argtypes = [vp, dbl, dbl, C.POINTER(u32), C.c_int, C.POINTER(vp)]
    L.hm_synth_partition.argtypes = [vp, i64, C.POINTER(u32), C.POINTER(u32),
                                     C.POINTER(u32), C.POINTER(i64)]
    L.hm_synth_shard_counts.argtypes = [vp, u64, u64, C.c_int, vp, C.POINTER(u64)]
    L.hm_synth_build_shard.argtypes = [vp, dbl, dbl, u64, u64, vp, u64, u64, C.c_int, C.POINTER(vp)]
    for name in ("hm_synth_corpus_destroy", "hm_synth_queries_destroy", "hm_synth_index_destroy"):
        getattr(L, name).argtypes = [vp]
    for name, rt in [("hm_synth_corpus_n", u64), ("hm_synth_corpus_n_tokens", u64),
                     ("hm_synth_queries_n", u64), ("hm_synth_index_n_terms", u32),
                     ("hm_synth_index_n_postings", u64), ("hm_synth_index_n_docs", u32),
                     ("hm_synth_index_avgdl", dbl)]:
        getattr(L, name).argtypes = [vp]
        getattr(L, name).restype = rt
    for name in ("hm_synth_corpus_tokens", "hm_synth_corpus_offsets", "hm_synth_corpus_ts",
                 "hm_synth_queries_terms", "hm_synth_queries_offsets", "hm_synth_queries_gold",
                 "hm_synth_queries_ts", "hm_synth_queries_paraphrased",
                 "hm_synth_index_term_rank", "hm_synth_index_rank_to_tid",
                 "hm_synth_index_term_offsets", "hm_synth_index_posting_rows",
                 "hm_synth_index_posting_tf", "hm_synth_index_idf", "hm_synth_index_maxscore",
                 "hm_synth_index_order_key", "hm_synth_index_doc_lens", "hm_synth_index_doc_ids"):
        getattr(L, name).argtypes = [vp]
        getattr(L, name).restype = vp
    _L = L
    return L


def _check(rc):
    if rc != 0:
        raise RuntimeError(_lib_handle().hm_synth_last_error().decode())


def _view(ptr, n, dtype):
    """Copy a borrowed native array into numpy (owned, survives destroy)."""
    if n == 0:
        return np.zeros(0, dtype=dtype)
    buf = (C.c_char * (int(n) * np.dtype(dtype).itemsize)).from_address(ptr)
    return np.frombuffer(buf, dtype=dtype).copy()


def wspec(**kw):
    w = WSpec()
    _lib_handle().hm_wspec_default(C.byref(w))
    for k, v in kw.items():
        setattr(w, k, v)
    return w


def qspec(**kw):
    q = QSpec()
    _lib_handle().hm_qspec_default(C.byref(q))
    for k, v in kw.items():
        setattr(q, k, v)
    return q


class Corpus:
    """gen_corpus output: token ranks per record (token string = "w%d" % rank)."""

    def __init__(self, spec=None, threads=0, **kw):
        L = _lib_handle()
        self.spec = spec if spec is not None else wspec(**kw)
        h = C.c_void_p()
        _check(L.hm_synth_corpus_create(C.byref(self.spec), threads, C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None):
            _lib_handle().hm_synth_corpus_destroy(self._h)
            self._h = None

    @property
    def n(self):
        return _lib_handle().hm_synth_corpus_n(self._h)

    def arrays(self):
        L = _lib_handle()
        n, nt = L.hm_synth_corpus_n(self._h), L.hm_synth_corpus_n_tokens(self._h)
        return (_view(L.hm_synth_corpus_tokens(self._h), nt, np.uint32),
                _view(L.hm_synth_corpus_offsets(self._h), n + 1, np.uint64),
                _view(L.hm_synth_corpus_ts(self._h), n, np.int64))

    def texts(self):
        tok, off, _ = self.arrays()
        return [" ".join("w%d" % t for t in tok[off[i]:off[i + 1]]) for i in range(len(off) - 1)]

    def partition(self, window_ms):
        """(K, row_order, part_row, t0) of build_temporal_index's bucketing."""
        L = _lib_handle()
        K = C.c_uint32()
        t0 = C.c_int64()
        _check(L.hm_synth_partition(self._h, window_ms, C.byref(K), None, None, C.byref(t0)))
        order = np.zeros(self.n, dtype=np.uint32)
        part = np.zeros(K.value + 1, dtype=np.uint32)
        _check(L.hm_synth_partition(self._h, window_ms, C.byref(K),
                                    order.ctypes.data_as(C.POINTER(C.c_uint32)),
                                    part.ctypes.data_as(C.POINTER(C.c_uint32)), C.byref(t0)))
        return K.value, order, part, t0.value


class Queries:
    """gen_queries output."""

    def __init__(self, corpus, spec=None, **kw):
        L = _lib_handle()
        self.spec = spec if spec is not None else qspec(**kw)
        h = C.c_void_p()
        _check(L.hm_synth_queries_create(corpus._h, C.byref(self.spec), C.byref(h)))
        n = L.hm_synth_queries_n(h)
        off = _view(L.hm_synth_queries_offsets(h), n + 1, np.uint64)
        self.term_ranks = _view(L.hm_synth_queries_terms(h), int(off[-1]), np.uint32)
        self.offsets = off
        self.gold = _view(L.hm_synth_queries_gold(h), n, np.uint64)
        self.ts = _view(L.hm_synth_queries_ts(h), n, np.int64)
        self.paraphrased = _view(L.hm_synth_queries_paraphrased(h), n, np.uint8)
        L.hm_synth_queries_destroy(h)

    def __len__(self):
        return len(self.gold)

    def terms(self, i):
        """Query i as the reference's term strings."""
        pre = "syn_w" if self.paraphrased[i] else "w"
        return ["%s%d" % (pre, r) for r in self.term_ranks[self.offsets[i]:self.offsets[i + 1]]]


class HostIndex:
    """build_index output as numpy arrays (the reference CsrIndex fields)."""

    def __init__(self, corpus, k1=1.2, b=0.75, row_order=None, threads=0, _handle=None):
        L = _lib_handle()
        h = _handle
        if h is None:
            h = C.c_void_p()
            ro = None
            if row_order is not None:
                row_order = np.ascontiguousarray(row_order, dtype=np.uint32)
                ro = row_order.ctypes.data_as(C.POINTER(C.c_uint32))
            _check(L.hm_synth_build(corpus._h, k1, b, ro, threads, C.byref(h)))
        nt, npost, nd = (L.hm_synth_index_n_terms(h), L.hm_synth_index_n_postings(h),
                         L.hm_synth_index_n_docs(h))
        self.build_k1, self.build_b = k1, b
        self.avgdl = L.hm_synth_index_avgdl(h)
        self.term_rank = _view(L.hm_synth_index_term_rank(h), nt, np.uint32)
        self.rank_to_tid = _view(L.hm_synth_index_rank_to_tid(h), corpus.spec.vocab_size, np.uint32)
        self.term_offsets = _view(L.hm_synth_index_term_offsets(h), nt + 1, np.uint64)
        self.posting_rows = _view(L.hm_synth_index_posting_rows(h), npost, np.uint32)
        self.posting_tf = _view(L.hm_synth_index_posting_tf(h), npost, np.uint32)
        self.idf = _view(L.hm_synth_index_idf(h), nt, np.float64)
        self.maxscore = _view(L.hm_synth_index_maxscore(h), nt, np.float64)
        self.order_key = _view(L.hm_synth_index_order_key(h), nt, np.float64)
        self.doc_lens = _view(L.hm_synth_index_doc_lens(h), nd, np.uint32)
        self.doc_ids = _view(L.hm_synth_index_doc_ids(h), nd, np.uint64)
        L.hm_synth_index_destroy(h)

    @classmethod
    def shard(cls, corpus, row_lo, row_hi, global_df, n_global, len_sum_global, k1=1.2, b=0.75, threads=0):
        """Rows [row_lo, row_hi) of the flat index with the GLOBAL idf / avgdl
        (hm_synth_build_shard); maxscore is the shard's local maximum."""
        h = C.c_void_p()
        gdf = np.ascontiguousarray(global_df, np.uint64)
        _check(_lib_handle().hm_synth_build_shard(corpus._h, k1, b, row_lo, row_hi, gdf.ctypes.data,
                                                  n_global, len_sum_global, threads, C.byref(h)))
        return cls(corpus, k1, b, _handle=h)

    @property
    def n_terms(self):
        return len(self.term_rank)

    @property
    def n_docs(self):
        return len(self.doc_ids)

    def term_strings(self):
        return ["w%d" % r for r in self.term_rank]

    def resolve(self, ranks):
        """Zipf ranks -> term ids (0xFFFFFFFF when absent from the index)."""
        ranks = np.asarray(ranks, dtype=np.int64)
        out = np.full(len(ranks), 0xFFFFFFFF, dtype=np.uint32)
        ok = ranks < len(self.rank_to_tid)
        out[ok] = self.rank_to_tid[ranks[ok]]
        return out


def shard_counts(corpus, row_lo, row_hi, threads=0):
    """(df[vocab_size] by Zipf rank, length sum) of rows [row_lo, row_hi)."""
    df = np.zeros(corpus.spec.vocab_size, np.uint64)
    ls = C.c_uint64()
    _check(_lib_handle().hm_synth_shard_counts(corpus._h, row_lo, row_hi, threads, df.ctypes.data,
                                               C.byref(ls)))
    return df, ls.value
