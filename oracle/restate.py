"""TEST INFRASTRUCTURE ONLY: ctypes handle on the plain-C oracle restatement
(oracle/bm25_oracle.c -> oracle/lib/liboracle.so).  See bm25_oracle.h for the
reference file:line each function restates.  Only tests/, smoke() and the
bench's cpu_baseline leg import this; the product never does.
"""
import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "liboracle.so")
_L = None


class Slot(C.Structure):
    _fields_ = [("score", C.c_double), ("doc", C.c_uint64), ("valid", C.c_int)]


def lib():
    global _L
    if _L is not None:
        return _L
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `make -C oracle lib/liboracle.so`")
    L = C.CDLL(LIB_PATH)
    P = C.POINTER
    u64, u32, dbl = C.c_uint64, C.c_uint32, C.c_double
    L.or_bm25_score.argtypes = [dbl] * 6
    L.or_bm25_score.restype = dbl
    L.or_idf_from_df.argtypes = [u32, u32]
    L.or_idf_from_df.restype = dbl
    L.or_make_plan.argtypes = [P(dbl), P(u32), u32, P(u32), P(u32)]
    L.or_make_plan.restype = u32
    L.or_topk_batch.argtypes = [P(u64), P(u32), P(dbl), P(dbl), u32, P(u32), P(u64), dbl,
                                P(u32), P(u32), P(u32), u32, u64, dbl, dbl, u32, u32, P(u64),
                                P(dbl), P(u32), P(u64)]
    L.or_bridge_topk_batch.argtypes = [P(u64), P(u32), P(dbl), u32, u32, P(u64), P(u64), P(u32),
                                       P(dbl), u32, u64, u32, u32, P(u64), P(dbl), P(u32), P(u64)]
    L.or_dense_topk_batch.argtypes = [P(C.c_float), P(u64), u64, u32, P(C.c_float), u32, u64, P(u64),
                                      P(dbl), P(u32)]
    L.or_confidence.argtypes = [P(dbl), u32, C.c_int, dbl]
    L.or_confidence.restype = dbl
    L.or_k_star.argtypes = [dbl, dbl]
    L.or_k_star.restype = u32
    L.or_temporal_budget.argtypes = [dbl, dbl, u32, u32]
    L.or_temporal_budget.restype = u32
    L.or_ndcg_at_k.argtypes = [P(u64), u32, P(u64), P(u32), u32, u64, C.c_int]
    L.or_ndcg_at_k.restype = dbl
    L.or_twophase_init.argtypes = [P(Slot), u64]
    L.or_twophase_select.argtypes = [P(Slot), u64, C.c_int, P(dbl), u64, u64, P(u64), P(dbl),
                                     P(u32)]
    _L = L
    return L


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def bm25_score(tf, idf, dl, avgdl, k1=1.2, b=0.75):
    return lib().or_bm25_score(tf, idf, dl, avgdl, k1, b)


def make_plan(order_keys, tids):
    ok = np.ascontiguousarray(order_keys, np.float64)
    t = np.ascontiguousarray(tids, np.uint32)
    pt = np.zeros(max(1, len(t)), np.uint32)
    pm = np.zeros(max(1, len(t)), np.uint32)
    m = lib().or_make_plan(_p(ok, C.c_double), _p(t, C.c_uint32), len(t), _p(pt, C.c_uint32),
                           _p(pm, C.c_uint32))
    return pt[:m].copy(), pm[:m].copy()


class OracleIndex:
    """Raw CSR arrays the restatement scores over (the a4 layout of SURVEY §8a)."""

    def __init__(self, term_offsets, posting_rows, posting_weights, idf, order_key, doc_lens,
                 doc_ids, avgdl):
        self.term_offsets = np.ascontiguousarray(term_offsets, np.uint64)
        self.posting_rows = np.ascontiguousarray(posting_rows, np.uint32)
        self.posting_weights = np.ascontiguousarray(posting_weights, np.float64)
        self.idf = np.ascontiguousarray(idf, np.float64)
        self.order_key = np.ascontiguousarray(order_key, np.float64)
        self.doc_lens = np.ascontiguousarray(doc_lens, np.uint32)
        self.doc_ids = np.ascontiguousarray(doc_ids, np.uint64)
        self.avgdl = float(avgdl)

    @classmethod
    def from_host(cls, hx):
        return cls(hx.term_offsets, hx.posting_rows, hx.posting_tf.astype(np.float64), hx.idf,
                   hx.order_key, hx.doc_lens, hx.doc_ids, hx.avgdl)

    def plans(self, tid_lists):
        """-> (plan_off, plan_tid, plan_mult) for a list of resolved tid lists."""
        off = [0]
        pts, pms = [], []
        for tids in tid_lists:
            pt, pm = make_plan(self.order_key, tids)
            pts.append(pt)
            pms.append(pm)
            off.append(off[-1] + len(pt))
        cat = lambda xs: np.concatenate(xs).astype(np.uint32) if xs else np.zeros(0, np.uint32)
        return np.array(off, np.uint32), cat(pts), cat(pms)

    def topk(self, tid_lists, k, k1=1.2, b=0.75, row_lo=0, row_hi=None):
        """Exhaustive top-k per query. -> (ids[nq,k], scores[nq,k], n[nq], postings[nq])"""
        nq = len(tid_lists)
        off, pt, pm = self.plans(tid_lists)
        if len(pt) == 0:
            pt = np.zeros(1, np.uint32)
            pm = np.zeros(1, np.uint32)
        kk = max(int(k), 1)
        ids = np.zeros((nq, kk), np.uint64)
        sc = np.zeros((nq, kk), np.float64)
        n = np.zeros(nq, np.uint32)
        post = np.zeros(nq, np.uint64)
        hi = len(self.doc_ids) if row_hi is None else row_hi
        rc = lib().or_topk_batch(
            _p(self.term_offsets, C.c_uint64), _p(self.posting_rows, C.c_uint32),
            _p(self.posting_weights, C.c_double), _p(self.idf, C.c_double), len(self.doc_ids),
            _p(self.doc_lens, C.c_uint32), _p(self.doc_ids, C.c_uint64), self.avgdl,
            _p(off, C.c_uint32), _p(pt, C.c_uint32), _p(pm, C.c_uint32), nq, k, k1, b, row_lo, hi,
            _p(ids, C.c_uint64), _p(sc, C.c_double), _p(n, C.c_uint32), _p(post, C.c_uint64))
        if rc != 0:
            raise MemoryError("oracle allocation failed")
        if k == 0:
            n[:] = 0
        return ids, sc, n, post


class OracleBridge:
    """CPU restatement of the learned-sparse bridge (src/bridge.cpp:22-137)
    over a Bridge-mode CSR.  Test infrastructure only."""

    def __init__(self, term_offsets, posting_rows, posting_weights, doc_ids):
        self.term_offsets = np.ascontiguousarray(term_offsets, np.uint64)
        self.posting_rows = np.ascontiguousarray(posting_rows, np.uint32)
        self.posting_weights = np.ascontiguousarray(posting_weights, np.float64)
        self.doc_ids = np.ascontiguousarray(doc_ids, np.uint64)

    @classmethod
    def ingest(cls, ids, vectors):
        """bridge_ingest (bridge.cpp:22-73): CSC transpose, rows ascending per term."""
        dim = max([int(i[-1]) + 1 for i, _ in vectors if len(i)] or [0])
        rows = np.concatenate([np.full(len(i), r, np.uint32) for r, (i, _) in enumerate(vectors)] or
                              [np.zeros(0, np.uint32)])
        tids = np.concatenate([np.asarray(i, np.uint32) for i, _ in vectors] or [np.zeros(0, np.uint32)])
        vals = np.concatenate([np.asarray(v, np.float64) for _, v in vectors] or [np.zeros(0)])
        order = np.argsort(tids, kind="stable")  # stable: rows stay ascending per term
        off = np.zeros(dim + 1, np.uint64)
        off[1:] = np.cumsum(np.bincount(tids, minlength=dim)[:dim])
        return cls(off, rows[order], vals[order], ids)

    @property
    def n_terms(self):
        return len(self.term_offsets) - 1

    def topk(self, queries, k, row_lo=0, row_hi=None):
        """bridge_topk per query. -> (ids[nq,k], scores[nq,k], n[nq], postings[nq])"""
        nq = len(queries)
        off = np.zeros(nq + 1, np.uint64)
        off[1:] = np.cumsum([len(i) for i, _ in queries])
        qi = np.ascontiguousarray(np.concatenate([np.asarray(i, np.uint32) for i, _ in queries] or
                                                 [np.zeros(0, np.uint32)]), np.uint32)
        qv = np.ascontiguousarray(np.concatenate([np.asarray(v, np.float64) for _, v in queries] or
                                                 [np.zeros(0)]), np.float64)
        if len(qi) == 0:
            qi, qv = np.zeros(1, np.uint32), np.zeros(1)
        kk = max(int(k), 1)
        ids = np.zeros((nq, kk), np.uint64)
        sc = np.zeros((nq, kk), np.float64)
        n = np.zeros(nq, np.uint32)
        post = np.zeros(nq, np.uint64)
        hi = len(self.doc_ids) if row_hi is None else row_hi
        rc = lib().or_bridge_topk_batch(
            _p(self.term_offsets, C.c_uint64), _p(self.posting_rows, C.c_uint32),
            _p(self.posting_weights, C.c_double), self.n_terms, len(self.doc_ids),
            _p(self.doc_ids, C.c_uint64), _p(off, C.c_uint64), _p(qi, C.c_uint32), _p(qv, C.c_double),
            nq, k, row_lo, hi, _p(ids, C.c_uint64), _p(sc, C.c_double), _p(n, C.c_uint32),
            _p(post, C.c_uint64))
        if rc != 0:
            raise MemoryError("oracle allocation failed")
        if k == 0:
            n[:] = 0
        return ids, sc, n, post


def dense_topk(data, ids, queries, k):
    """CPU restatement of dense_topk (src/dense.cpp:86-101) per query row.
    -> (ids[nq,k], scores[nq,k], n[nq])"""
    data = np.ascontiguousarray(data, np.float32)
    ids = np.ascontiguousarray(ids, np.uint64)
    queries = np.ascontiguousarray(queries, np.float32)
    nq, dim = queries.shape
    kk = max(int(k), 1)
    o_ids = np.zeros((nq, kk), np.uint64)
    o_sc = np.zeros((nq, kk))
    n = np.zeros(nq, np.uint32)
    if lib().or_dense_topk_batch(_p(data, C.c_float), _p(ids, C.c_uint64), len(ids), dim,
                                 _p(queries, C.c_float), nq, k, _p(o_ids, C.c_uint64), _p(o_sc, C.c_double),
                                 _p(n, C.c_uint32)) != 0:
        raise MemoryError("oracle allocation failed")
    return o_ids, o_sc, n


def confidence(scores, proxy=0, eps=1e-9):
    s = np.ascontiguousarray(scores, np.float64)
    return lib().or_confidence(_p(s, C.c_double), len(s), proxy, eps)


def margin(scores, eps=1e-9):
    return confidence(scores, 0, eps)


def k_star(eps, lam):
    return lib().or_k_star(eps, lam)


def temporal_budget(eps, lam, k_max, K):
    return lib().or_temporal_budget(eps, lam, k_max, K)


def ndcg(ids, rels, k, linear=False):
    ids = np.ascontiguousarray(ids, np.uint64)
    rd = np.array(list(rels.keys()), np.uint64)
    rg = np.array(list(rels.values()), np.uint32)
    return lib().or_ndcg_at_k(_p(ids, C.c_uint64), len(ids), _p(rd, C.c_uint64),
                              _p(rg, C.c_uint32), len(rd), k, 1 if linear else 0)


class TwoPhase:
    """or_twophase_* with persistent slots (TwoPhaseSelector state)."""

    def __init__(self, capacity, reset_sentinel=True):
        self.cap = capacity
        self.reset = reset_sentinel
        self.slots = (Slot * capacity)()
        lib().or_twophase_init(self.slots, capacity)

    def select(self, scores, k):
        s = np.ascontiguousarray(scores, np.float64)
        ids = np.zeros(max(1, k), np.uint64)
        sc = np.zeros(max(1, k), np.float64)
        n = C.c_uint32()
        rc = lib().or_twophase_select(self.slots, self.cap, 1 if self.reset else 0,
                                      _p(s, C.c_double), len(s), k, _p(ids, C.c_uint64),
                                      _p(sc, C.c_double), C.byref(n))
        if rc != 0:
            raise ValueError("k must be in [1, capacity]")
        return ids[:n.value].copy(), sc[:n.value].copy()
