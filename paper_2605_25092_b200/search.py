"""Python mirror of the reference search API over the B200 C ABI (hm_b200.h).

Reference interfaces mirrored (paths under /root/reference/proj):
  Bm25Params                      include/hybrid/csr_index.hpp:15-18
  SearchStats                     include/hybrid/csr_index.hpp:37-39
  CsrIndex.bm25_topk / _maxscore  include/hybrid/csr_index.hpp:72-79
  TemporalIndex.topk              include/hybrid/temporal_index.hpp:63-66
  confidence (Margin)             include/hybrid/cascade.hpp:29-34
  the cmd_search batch loop       tools/hybridmem.cpp:227-313  -> search_batch
  SparseVector, bridge_ingest, bridge_export, bridge_topk(_maxscore)
                                  include/hybrid/bridge.hpp:12-40 -> BridgeIndex
  EmbeddingMatrix, dense_topk     include/hybrid/dense.hpp:13-34  -> DenseIndex
  rrf, agent_rrf, FusionParams    include/hybrid/fusion.hpp:17-49
  CascadeConfig, cascade_retrieve include/hybrid/cascade.hpp:19-61 (+ cascade_batch)

Every search runs on the GPU through libhm_b200.so; there is no CPU path.
Errors map to the reference's exception types (RuntimeError for
std::runtime_error, ValueError for std::invalid_argument, IndexError for
std::out_of_range).
"""
import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib

HM_FLAG_FORCE_EXACT = 1
HM_FLAG_DEBUG_NO_RESET = 2
HM_FLAG_TIMING = 4
HM_FLAG_EXHAUSTIVE = 16
HM_FLAG_SEED_ALL = 32
HM_FLAG_NO_SPLIT = 64
HM_FLAG_BOUND_ONLY = 512
HM_FLAG_NO_NESKIP = 128
HM_FLAG_NE_ALL = 256
NO_TERM = 0xFFFFFFFF
MAX_K = 256

_L = None


class CsrView(C.Structure):
    _fields_ = [("n_terms", C.c_uint32), ("term_offsets", C.c_void_p),
                ("posting_rows", C.c_void_p), ("posting_weights", C.c_void_p),
                ("posting_tf", C.c_void_p), ("term_idfs", C.c_void_p),
                ("term_order_keys", C.c_void_p), ("n_docs", C.c_uint32),
                ("doc_lens", C.c_void_p), ("doc_ids", C.c_void_p), ("avgdl", C.c_double)]


class QueryBatch(C.Structure):
    _fields_ = [("n_queries", C.c_uint32), ("q_off", C.c_void_p), ("q_tid", C.c_void_p),
                ("k", C.c_uint32), ("k1", C.c_double), ("b", C.c_double),
                ("tau", C.c_void_p), ("tau_default", C.c_double),
                ("epsilon_guard", C.c_double), ("row_lo", C.c_uint32),
                ("row_hi", C.c_uint32), ("flags", C.c_uint32),
                ("ext_bound", C.c_void_p), ("out_bound", C.c_void_p)]


class Results(C.Structure):
    _fields_ = [("ids", C.c_void_p), ("scores", C.c_void_p), ("n", C.c_void_p),
                ("conf", C.c_void_p), ("skip", C.c_void_p), ("postings", C.c_void_p)]


class BridgeView(C.Structure):
    _fields_ = [("n_terms", C.c_uint32), ("term_offsets", C.c_void_p),
                ("posting_rows", C.c_void_p), ("posting_weights", C.c_void_p),
                ("n_docs", C.c_uint32), ("doc_ids", C.c_void_p)]


class BridgeBatch(C.Structure):
    _fields_ = [("n_queries", C.c_uint32), ("q_off", C.c_void_p), ("q_idx", C.c_void_p),
                ("q_val", C.c_void_p), ("k", C.c_uint32), ("row_lo", C.c_uint32),
                ("row_hi", C.c_uint32), ("max_nnz", C.c_uint32), ("flags", C.c_uint32)]


class DenseView(C.Structure):
    _fields_ = [("dim", C.c_uint32), ("count", C.c_uint32), ("data", C.c_void_p), ("doc_ids", C.c_void_p)]


class DenseBatch(C.Structure):
    _fields_ = [("n_queries", C.c_uint32), ("dim", C.c_uint32), ("queries", C.c_void_p), ("k", C.c_uint32),
                ("flags", C.c_uint32)]


EXPORTS = ["hm_dense_create", "hm_dense_destroy", "hm_dense_search_batch", "hm_dense_search_batch_device",
           "hm_dense_last_timing", "hm_dense_last_stats",
           "hm_bridge_create", "hm_bridge_destroy", "hm_bridge_search_batch",
           "hm_bridge_search_batch_device", "hm_bridge_last_timing",
           "hm_index_create", "hm_index_destroy", "hm_index_device_bytes", "hm_index_format",
           "hm_search_batch", "hm_search_batch_device", "hm_last_batch_stats",
           "hm_last_batch_timing", "hm_last_batch_seed", "hm_last_batch_graph",
           "hm_hidx_load", "hm_hidx_last_error", "hm_hidx_view", "hm_hidx_term", "hm_hidx_maxscores",
           "hm_hidx_free", "hm_htix_load", "hm_htix_flat", "hm_htix_partitions", "hm_htix_params",
           "hm_htix_free",
           "hm_merge_shards_device", "hm_margin", "hm_last_error", "hm_search_batch_parts",
           "hm_last_batch_wide", "hm_last_batch_handover", "hm_vocab_create", "hm_vocab_destroy", "hm_vocab_size",
           "hm_vocab_resolve"]


def lib():
    global _L
    if _L is not None:
        return _L
    L = _lib.load("libhm_b200.so")
    P = C.POINTER
    L.hm_last_error.restype = C.c_char_p
    L.hm_index_create.argtypes = [P(CsrView), C.c_int, P(C.c_void_p)]
    L.hm_index_destroy.argtypes = [C.c_void_p]
    L.hm_index_device_bytes.argtypes = [C.c_void_p]
    L.hm_index_device_bytes.restype = C.c_uint64
    L.hm_index_format.argtypes = [C.c_void_p, P(C.c_uint32), P(C.c_uint32), P(C.c_uint32),
                                  P(C.c_uint64)]
    L.hm_search_batch.argtypes = [C.c_void_p, P(QueryBatch), P(Results)]
    L.hm_search_batch_device.argtypes = [C.c_void_p, P(QueryBatch), P(Results), C.c_void_p]
    L.hm_last_batch_stats.argtypes = [P(C.c_uint32), P(C.c_uint32)]
    L.hm_last_batch_timing.argtypes = [P(C.c_float), P(C.c_float), P(C.c_float)]
    L.hm_last_batch_seed.argtypes = [P(C.c_float), P(C.c_uint32)]
    L.hm_last_batch_graph.argtypes = [P(C.c_uint32)]
    L.hm_last_batch_wide.argtypes = [P(C.c_uint32)]
    L.hm_last_batch_handover.argtypes = [C.c_void_p, C.c_uint32]
    L.hm_search_batch_parts.argtypes = [C.c_void_p, P(QueryBatch), C.c_uint32, C.c_void_p, P(Results)]
    L.hm_vocab_create.argtypes = [C.c_void_p, C.c_void_p, C.c_uint32, P(C.c_void_p)]
    L.hm_vocab_destroy.argtypes = [C.c_void_p]
    L.hm_vocab_size.argtypes = [C.c_void_p]
    L.hm_vocab_size.restype = C.c_uint32
    L.hm_vocab_resolve.argtypes = [C.c_void_p, C.c_uint32, C.c_char_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_uint64, P(C.c_uint64), C.c_uint32]
    L.hm_hidx_load.argtypes = [C.c_char_p, P(C.c_void_p)]
    L.hm_hidx_last_error.restype = C.c_char_p
    L.hm_hidx_view.argtypes = [C.c_void_p, P(CsrView), P(C.c_uint32), P(C.c_double), P(C.c_double)]
    L.hm_hidx_term.argtypes = [C.c_void_p, C.c_uint32, P(C.c_char_p)]
    L.hm_hidx_term.restype = C.c_uint32
    L.hm_hidx_maxscores.argtypes = [C.c_void_p]
    L.hm_hidx_maxscores.restype = P(C.c_double)
    L.hm_hidx_free.argtypes = [C.c_void_p]
    L.hm_htix_load.argtypes = [C.c_char_p, P(C.c_void_p)]
    L.hm_htix_flat.argtypes = [C.c_void_p]
    L.hm_htix_flat.restype = C.c_void_p
    L.hm_htix_partitions.argtypes = [C.c_void_p, P(C.c_uint32), P(C.c_void_p), P(C.c_void_p), P(C.c_void_p)]
    L.hm_htix_params.argtypes = [C.c_void_p, P(C.c_int64), P(C.c_double), P(C.c_double), P(C.c_uint32),
                                 P(C.c_uint64)]
    L.hm_htix_free.argtypes = [C.c_void_p]
    L.hm_merge_shards_device.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_void_p,
                                         C.c_void_p, C.c_void_p, C.c_void_p, C.c_double,
                                         C.c_double, P(Results), C.c_void_p]
    L.hm_sharded_create.argtypes = [P(CsrView), C.c_void_p, C.c_uint32, P(C.c_void_p)]
    L.hm_sharded_destroy.argtypes = [C.c_void_p]
    L.hm_sharded_info.argtypes = [C.c_void_p, P(C.c_uint32), C.c_void_p, C.c_void_p, P(C.c_uint32)]
    L.hm_sharded_search_batch.argtypes = [C.c_void_p, P(QueryBatch), P(Results)]
    L.hm_margin.argtypes = [P(C.c_double), C.c_uint32, C.c_double]
    L.hm_margin.restype = C.c_double
    L.hm_dense_create.argtypes = [P(DenseView), C.c_int, P(C.c_void_p)]
    L.hm_dense_destroy.argtypes = [C.c_void_p]
    L.hm_dense_search_batch.argtypes = [C.c_void_p, P(DenseBatch), P(Results)]
    L.hm_dense_search_batch_device.argtypes = [C.c_void_p, P(DenseBatch), P(Results), C.c_void_p]
    L.hm_dense_last_timing.argtypes = [P(C.c_float)]
    L.hm_dense_last_stats.argtypes = [P(C.c_uint32), P(C.c_uint32), P(C.c_uint64)]
    L.hm_bridge_create.argtypes = [P(BridgeView), C.c_int, P(C.c_void_p)]
    L.hm_bridge_destroy.argtypes = [C.c_void_p]
    L.hm_bridge_search_batch.argtypes = [C.c_void_p, P(BridgeBatch), P(Results)]
    L.hm_bridge_search_batch_device.argtypes = [C.c_void_p, P(BridgeBatch), P(Results), C.c_void_p]
    L.hm_bridge_last_timing.argtypes = [P(C.c_float)]
    _L = L
    return L


def _check(rc):
    if rc == 0:
        return
    msg = lib().hm_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 3:
        raise IndexError(msg)
    raise RuntimeError(msg)


def _ptr(a):
    return None if a is None else a.ctypes.data


@dataclass
class Bm25Params:
    """hybrid::Bm25Params (csr_index.hpp:15-18)."""
    k1: float = 1.2
    b: float = 0.75


@dataclass
class SearchStats:
    """hybrid::SearchStats (csr_index.hpp:37-39); accumulates like the reference."""
    postings_touched: int = 0


class DeviceIndex:
    """An HBM-resident index (hm_index).  Arrays follow hybrid::CsrIndex."""

    def __init__(self, term_offsets, posting_rows, idf, order_key, doc_lens, doc_ids, avgdl,
                 posting_tf=None, posting_weights=None, device=0):
        self._keep = dict(
            term_offsets=np.ascontiguousarray(term_offsets, np.uint64),
            posting_rows=np.ascontiguousarray(posting_rows, np.uint32),
            idf=np.ascontiguousarray(idf, np.float64),
            order_key=np.ascontiguousarray(order_key, np.float64),
            doc_lens=np.ascontiguousarray(doc_lens, np.uint32),
            doc_ids=np.ascontiguousarray(doc_ids, np.uint64))
        if posting_tf is not None:
            self._keep["tf"] = np.ascontiguousarray(posting_tf, np.uint32)
        if posting_weights is not None:
            self._keep["w"] = np.ascontiguousarray(posting_weights, np.float64)
        k = self._keep
        v = CsrView(len(k["idf"]), _ptr(k["term_offsets"]), _ptr(k["posting_rows"]),
                    _ptr(k.get("w")), _ptr(k.get("tf")), _ptr(k["idf"]), _ptr(k["order_key"]),
                    len(k["doc_ids"]), _ptr(k["doc_lens"]), _ptr(k["doc_ids"]), float(avgdl))
        h = C.c_void_p()
        _check(lib().hm_index_create(C.byref(v), device, C.byref(h)))
        self._h = h
        self.device = device
        self.n_terms = len(k["idf"])
        self.n_docs = len(k["doc_ids"])
        self.df = np.diff(k["term_offsets"].astype(np.int64))
        self._keep = None  # borrowed only for the duration of create

    @classmethod
    def _adopt(cls, h, device, n_terms, n_docs, df):
        self = cls.__new__(cls)
        self._h, self.device, self.n_terms, self.n_docs, self.df, self._keep = h, device, n_terms, n_docs, df, None
        return self

    @classmethod
    def from_hidx(cls, path, device=0):
        """From a HIDX v1 file written by the reference's save_index."""
        return Hidx(path).device_index(device)

    @classmethod
    def from_host(cls, hx, device=0):
        """From a paper_2605_25092_b200.synth.HostIndex."""
        return cls(hx.term_offsets, hx.posting_rows, hx.idf, hx.order_key, hx.doc_lens,
                   hx.doc_ids, hx.avgdl, posting_tf=hx.posting_tf, device=device)

    def close(self):
        if getattr(self, "_h", None):
            lib().hm_index_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except TypeError:  # interpreter shutdown: module globals already cleared
            pass

    @property
    def device_bytes(self):
        return lib().hm_index_device_bytes(self._h)

    def format(self):
        rb, cb, nc = C.c_uint32(), C.c_uint32(), C.c_uint32()
        ne = C.c_uint64()
        _check(lib().hm_index_format(self._h, C.byref(rb), C.byref(cb), C.byref(nc), C.byref(ne)))
        return dict(row_bits=rb.value, code_bits=cb.value, n_codes=nc.value, n_escaped=ne.value)

    # ------------------------------------------------------------ batch API
    def search_batch(self, q_off, q_tid, k, k1=1.2, b=0.75, tau=None, tau_default=0.10,
                     epsilon_guard=1e-9, row_lo=0, row_hi=0, flags=0):
        """Host-buffer batch search (hm_search_batch).  q_off[nq+1], q_tid resolved term
        ids (NO_TERM for unknown).  Returns dict(ids[nq,k], scores[nq,k], n[nq],
        conf[nq], skip[nq], postings[nq], n_exact)."""
        q_off = np.ascontiguousarray(q_off, np.uint32)
        q_tid = np.ascontiguousarray(q_tid, np.uint32)
        nq = len(q_off) - 1
        kk = max(int(k), 1)
        out = dict(ids=np.zeros((nq, kk), np.uint64), scores=np.zeros((nq, kk), np.float64),
                   n=np.zeros(nq, np.uint32), conf=np.zeros(nq, np.float64),
                   skip=np.zeros(nq, np.uint8), postings=np.zeros(nq, np.uint64))
        tau_a = None if tau is None else np.ascontiguousarray(tau, np.float64)
        qb = QueryBatch(nq, _ptr(q_off), _ptr(q_tid) if len(q_tid) else None, int(k), k1, b,
                        _ptr(tau_a), tau_default, epsilon_guard, row_lo, row_hi, flags)
        r = Results(_ptr(out["ids"]), _ptr(out["scores"]), _ptr(out["n"]), _ptr(out["conf"]),
                    _ptr(out["skip"]), _ptr(out["postings"]))
        _check(lib().hm_search_batch(self._h, C.byref(qb), C.byref(r)))
        ne, nl = C.c_uint32(), C.c_uint32()
        lib().hm_last_batch_stats(C.byref(ne), C.byref(nl))
        out["n_exact"] = ne.value
        if k == 0:
            out["ids"] = out["ids"][:, :0]
            out["scores"] = out["scores"][:, :0]
        return out

    def search_parts(self, q_off, q_tid, k, part_row, k1=1.2, b=0.75, flags=0):
        """hm_search_batch_parts: every query searched inside each row range
        [part_row[p], part_row[p+1]) separately.  Returns dict(ids[P,nq,k],
        scores[P,nq,k], n[P,nq], postings[P,nq])."""
        q_off = np.ascontiguousarray(q_off, np.uint32)
        q_tid = np.ascontiguousarray(q_tid, np.uint32)
        part_row = np.ascontiguousarray(part_row, np.uint32)
        nq, P = len(q_off) - 1, len(part_row) - 1
        kk = max(int(k), 1)
        out = dict(ids=np.zeros((P, nq, kk), np.uint64), scores=np.zeros((P, nq, kk), np.float64),
                   n=np.zeros((P, nq), np.uint32), postings=np.zeros((P, nq), np.uint64))
        qb = QueryBatch(nq, _ptr(q_off), _ptr(q_tid) if len(q_tid) else None, int(k), k1, b,
                        None, 0.10, 1e-9, 0, 0, flags)
        r = Results(_ptr(out["ids"]), _ptr(out["scores"]), _ptr(out["n"]), None, None,
                    _ptr(out["postings"]))
        _check(lib().hm_search_batch_parts(self._h, C.byref(qb), P, _ptr(part_row), C.byref(r)))
        return out

    def search_lists(self, tid_lists, k, **kw):
        off = np.zeros(len(tid_lists) + 1, np.uint32)
        off[1:] = np.cumsum([len(t) for t in tid_lists])
        tids = (np.concatenate([np.asarray(t, np.uint32) for t in tid_lists])
                if tid_lists and off[-1] else np.zeros(0, np.uint32))
        return self.search_batch(off, tids, k, **kw)

    def search_batch_device(self, q_off, q_tid, out, k, k1=1.2, b=0.75, tau=None,
                            tau_default=0.10, epsilon_guard=1e-9, row_lo=0, row_hi=0, flags=0,
                            stream=None, ext_bound=None, out_bound=None):
        """Device-resident batch (torch CUDA tensors), enqueued on `stream`
        (default: torch's current stream).  `out` is a dict of torch tensors
        (ids[nq,k] int64, scores[nq,k] f64, n[nq] int32, conf[nq] f64,
        skip[nq] uint8, postings[nq] int64).  Doc shards: out_bound (float32[nq],
        with HM_FLAG_BOUND_ONLY) receives this shard's k-th-score bound;
        ext_bound (float32[nq]) is the MAX of the shards' bounds (hm_b200.h)."""
        import torch
        nq = q_off.numel() - 1
        st = stream if stream is not None else torch.cuda.current_stream(q_off.device)
        qb = QueryBatch(nq, q_off.data_ptr(), q_tid.data_ptr(), int(k), k1, b,
                        None if tau is None else tau.data_ptr(), tau_default, epsilon_guard,
                        row_lo, row_hi, flags,
                        None if ext_bound is None else ext_bound.data_ptr(),
                        None if out_bound is None else out_bound.data_ptr())
        r = Results(out["ids"].data_ptr(), out["scores"].data_ptr(), out["n"].data_ptr(),
                    out["conf"].data_ptr(), out["skip"].data_ptr(), out["postings"].data_ptr())
        _check(lib().hm_search_batch_device(self._h, C.byref(qb), C.byref(r), st.cuda_stream))
        if flags & HM_FLAG_TIMING:
            return last_timing()


class ShardedDeviceIndex:
    """Doc-sharded index over several devices of this process (hm_sharded_*):
    shard g = rows [n*g/G, n*(g+1)/G) on devices[g] with the flat statistics;
    one search call runs every shard concurrently and merges on devices[0]
    with one kernel reading the shards' lists over peer memory.  Results equal
    DeviceIndex.search_batch on the unsharded index."""

    def __init__(self, term_offsets, posting_rows, idf, order_key, doc_lens, doc_ids, avgdl,
                 devices, posting_tf=None, posting_weights=None):
        keep = dict(
            term_offsets=np.ascontiguousarray(term_offsets, np.uint64),
            posting_rows=np.ascontiguousarray(posting_rows, np.uint32),
            idf=np.ascontiguousarray(idf, np.float64),
            order_key=np.ascontiguousarray(order_key, np.float64),
            doc_lens=np.ascontiguousarray(doc_lens, np.uint32),
            doc_ids=np.ascontiguousarray(doc_ids, np.uint64))
        if posting_tf is not None:
            keep["tf"] = np.ascontiguousarray(posting_tf, np.uint32)
        if posting_weights is not None:
            keep["w"] = np.ascontiguousarray(posting_weights, np.float64)
        v = CsrView(len(keep["idf"]), _ptr(keep["term_offsets"]), _ptr(keep["posting_rows"]),
                    _ptr(keep.get("w")), _ptr(keep.get("tf")), _ptr(keep["idf"]), _ptr(keep["order_key"]),
                    len(keep["doc_ids"]), _ptr(keep["doc_lens"]), _ptr(keep["doc_ids"]), float(avgdl))
        devs = np.ascontiguousarray(devices, np.int32)
        h = C.c_void_p()
        _check(lib().hm_sharded_create(C.byref(v), _ptr(devs), len(devs), C.byref(h)))
        self._h = h
        self.n_docs = len(keep["doc_ids"])

    @classmethod
    def from_host(cls, hx, devices):
        return cls(hx.term_offsets, hx.posting_rows, hx.idf, hx.order_key, hx.doc_lens,
                   hx.doc_ids, hx.avgdl, devices, posting_tf=hx.posting_tf)

    def info(self):
        """dict(n_shards, shard_row[G+1], devices[G], p2p[G])."""
        n = C.c_uint32()
        _check(lib().hm_sharded_info(self._h, C.byref(n), None, None, None))
        G = n.value
        rows = np.zeros(G + 1, np.uint32)
        devs = np.zeros(G, np.int32)
        mask = C.c_uint32()
        _check(lib().hm_sharded_info(self._h, C.byref(n), _ptr(rows), _ptr(devs), C.byref(mask)))
        return dict(n_shards=G, shard_row=rows, devices=devs,
                    p2p=np.array([(mask.value >> g) & 1 for g in range(G)], bool))

    def search_batch(self, q_off, q_tid, k, k1=1.2, b=0.75, tau=None, tau_default=0.10,
                     epsilon_guard=1e-9, row_lo=0, row_hi=0, flags=0):
        """hm_sharded_search_batch; same arguments and outputs as DeviceIndex.search_batch."""
        q_off = np.ascontiguousarray(q_off, np.uint32)
        q_tid = np.ascontiguousarray(q_tid, np.uint32)
        nq = len(q_off) - 1
        kk = max(int(k), 1)
        out = dict(ids=np.zeros((nq, kk), np.uint64), scores=np.zeros((nq, kk), np.float64),
                   n=np.zeros(nq, np.uint32), conf=np.zeros(nq, np.float64),
                   skip=np.zeros(nq, np.uint8), postings=np.zeros(nq, np.uint64))
        tau_a = None if tau is None else np.ascontiguousarray(tau, np.float64)
        qb = QueryBatch(nq, _ptr(q_off), _ptr(q_tid) if len(q_tid) else None, int(k), k1, b,
                        _ptr(tau_a), tau_default, epsilon_guard, row_lo, row_hi, flags)
        r = Results(_ptr(out["ids"]), _ptr(out["scores"]), _ptr(out["n"]), _ptr(out["conf"]),
                    _ptr(out["skip"]), _ptr(out["postings"]))
        _check(lib().hm_sharded_search_batch(self._h, C.byref(qb), C.byref(r)))
        if k == 0:
            out["ids"] = out["ids"][:, :0]
            out["scores"] = out["scores"][:, :0]
        return out

    def close(self):
        if getattr(self, "_h", None):
            lib().hm_sharded_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except TypeError:  # interpreter shutdown: module globals already cleared
            pass


def last_timing():
    """(ms_plan, ms_search, ms_exact) of this thread's last HM_FLAG_TIMING batch."""
    a, b, c = C.c_float(), C.c_float(), C.c_float()
    lib().hm_last_batch_timing(C.byref(a), C.byref(b), C.byref(c))
    return a.value, b.value, c.value


def last_graph():
    """0 eager, 1 captured into a CUDA graph, 2 replayed (this thread's last batch)."""
    m = C.c_uint32()
    lib().hm_last_batch_graph(C.byref(m))
    return m.value


class Vocab:
    """hm_vocab: term strings -> term ids for whole batches of query strings
    (make_plan's lookup, csr_index.cpp:31-48; the whitespace split of
    load_queries_tsv, io.cpp:389-391), resolved by native threads."""

    def __init__(self, terms):
        enc = [t.encode() for t in terms]
        arr = (C.c_char_p * max(len(enc), 1))(*enc)
        lens = np.array([len(e) for e in enc] or [0], np.uint32)
        h = C.c_void_p()
        _check(lib().hm_vocab_create(arr, _ptr(lens), len(enc), C.byref(h)))
        self._h = h

    def __len__(self):
        return lib().hm_vocab_size(self._h)

    def resolve_text(self, text, text_off, n_threads=0):
        """text: bytes of all queries; text_off[nq+1] byte offsets -> (q_off, q_tid)."""
        text_off = np.ascontiguousarray(text_off, np.uint64)
        nq = len(text_off) - 1
        q_off = np.zeros(nq + 1, np.uint32)
        cap = max(len(text) // 2 + 1, 1)  # a token takes >= 1 byte + 1 separator
        q_tid = np.zeros(cap, np.uint32)
        n = C.c_uint64()
        _check(lib().hm_vocab_resolve(self._h, nq, text, _ptr(text_off), _ptr(q_off), _ptr(q_tid),
                                      cap, C.byref(n), n_threads))
        return q_off, q_tid[:n.value]

    def resolve(self, queries, n_threads=0):
        """list of query strings -> (q_off, q_tid)."""
        enc = [q.encode() for q in queries]
        off = np.zeros(len(enc) + 1, np.uint64)
        off[1:] = np.cumsum([len(e) for e in enc])
        return self.resolve_text(b"".join(enc), off, n_threads)

    def close(self):
        if getattr(self, "_h", None):
            lib().hm_vocab_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except TypeError:  # interpreter shutdown: module globals already cleared
            pass


def last_handover(nq):
    """uint8[nq]: 1 where the last HM_FLAG_TIMING batch's query ran on the tile
    sweep (handed over by the seeded pass), 0 where the seeded pass served it."""
    f = np.zeros(nq, np.uint32)
    _check(lib().hm_last_batch_handover(_ptr(f), nq))
    return f.astype(np.uint8)


def last_wide():
    """Queries of this thread's last batch served by the wide path (k > 256 or
    plans of more than 256 distinct terms; kernels/wide.cu)."""
    n = C.c_uint32()
    lib().hm_last_batch_wide(C.byref(n))
    return n.value


def last_seed():
    """(ms_seed, n_handed_over): the seeded MaxScore pass of this thread's last
    batch (its time on HM_FLAG_TIMING batches; queries left to the exhaustive kernel)."""
    a, n = C.c_float(), C.c_uint32()
    lib().hm_last_batch_seed(C.byref(a), C.byref(n))
    return a.value, n.value


def last_stats():
    """(n_exact_fallback, n_kernel_launches) of this thread's last batch."""
    ne, nl = C.c_uint32(), C.c_uint32()
    lib().hm_last_batch_stats(C.byref(ne), C.byref(nl))
    return ne.value, nl.value


def merge_shards_device(shard_ids, shard_scores, shard_n, out, k, tau=None, tau_default=0.10,
                        epsilon_guard=1e-9, stream=None):
    """hm_merge_shards_device over torch CUDA tensors [G,nq,k] / [G,nq]."""
    import torch
    G, nq = shard_n.shape
    st = stream if stream is not None else torch.cuda.current_stream(shard_n.device)
    r = Results(out["ids"].data_ptr(), out["scores"].data_ptr(), out["n"].data_ptr(),
                out["conf"].data_ptr(), out["skip"].data_ptr(), None)
    _check(lib().hm_merge_shards_device(G, nq, k, shard_ids.data_ptr(), shard_scores.data_ptr(),
                                        shard_n.data_ptr(),
                                        None if tau is None else tau.data_ptr(), tau_default,
                                        epsilon_guard, C.byref(r), st.cuda_stream))


def bm25_score(tf, idf, doc_len, avgdl, p=None):
    """csr_index.cpp:10-15, the reference's operation order."""
    p = p or Bm25Params()
    norm = doc_len / avgdl if avgdl > 0.0 else 1.0
    return idf * tf * (p.k1 + 1.0) / (tf + p.k1 * (1.0 - p.b + p.b * norm))


MARGIN, TOP1_FRACTION, ENTROPY_COMPLEMENT, CLASSIFIER = 0, 1, 2, 3


def confidence(scores, proxy=MARGIN, epsilon_guard=1e-9):
    """cascade::confidence (cascade.cpp:10-38) for every proxy, same
    operation order (the device computes Margin in the batch epilogue)."""
    if proxy == CLASSIFIER:
        raise ValueError("Classifier proxy has no score-based confidence")
    s = [float(x) for x in scores]
    if not s or s[0] <= 0.0:
        return 0.0
    if proxy == MARGIN:
        return 0.0 if len(s) < 2 else (s[0] - s[1]) / max(s[0], epsilon_guard)
    if proxy == TOP1_FRACTION:
        tot = 0.0
        for x in s:
            tot += x
        return s[0] / max(tot, epsilon_guard)
    if proxy == ENTROPY_COMPLEMENT:
        if len(s) < 2:
            return 0.0
        tot = 0.0
        for x in s:
            tot += x
        if tot <= 0.0:
            return 0.0
        h = 0.0
        for x in s:
            pi = x / tot
            if pi > 0.0:
                h -= pi * math.log(pi)
        return 1.0 - h / math.log(float(len(s)))
    return 0.0


def margin(scores, epsilon_guard=1e-9):
    """Margin confidence (src/cascade.cpp:15-21)."""
    s = np.ascontiguousarray(scores, np.float64)
    return lib().hm_margin(s.ctypes.data_as(C.POINTER(C.c_double)), len(s), epsilon_guard)


# ---------------------------------------------------------------- reference-shaped API
class CsrIndex:
    """Mirror of hybrid::CsrIndex (csr_index.hpp:44-87) whose searches run on the GPU.

    `terms` (alphabetical; tid = position) and the CSR arrays are the reference's
    fields; the device copy is created lazily on first search and cached."""

    def __init__(self, terms, term_offsets, posting_rows, posting_weights, term_idfs,
                 term_order_keys, doc_lens, doc_ids, avgdl, build_params=None, device=0):
        self.terms = list(terms)
        self.vocab = {t: i for i, t in enumerate(self.terms)}
        self.term_offsets = np.asarray(term_offsets, np.uint64)
        self.posting_rows = np.asarray(posting_rows, np.uint32)
        self.posting_weights = np.asarray(posting_weights, np.float64)
        self.term_idfs = np.asarray(term_idfs, np.float64)
        self.term_order_keys = np.asarray(term_order_keys, np.float64)
        self.doc_lens = np.asarray(doc_lens, np.uint32)
        self.doc_ids = np.asarray(doc_ids, np.uint64)
        self.avgdl = float(avgdl)
        self.build_params = build_params or Bm25Params()
        self.device = device
        self._dev = None
        self._maxscores = {}

    @classmethod
    def load(cls, path, device=0):
        """hybrid::load_index (io.cpp:229-232) of a HIDX v1 file, native reader."""
        hd = Hidx(path)
        a = hd.arrays()
        if hd.mode != 0:
            raise RuntimeError("BM25 scoring requires a BM25-mode index")
        return cls(hd.terms(), a["term_offsets"], a["posting_rows"], a["posting_weights"], a["idf"],
                   a["order_key"], a["doc_lens"], a["doc_ids"], a["avgdl"], hd.build_params, device)

    @classmethod
    def from_host(cls, hx, device=0):
        idx = cls(hx.term_strings(), hx.term_offsets, hx.posting_rows,
                  hx.posting_tf.astype(np.float64), hx.idf, hx.order_key, hx.doc_lens,
                  hx.doc_ids, hx.avgdl, Bm25Params(hx.build_k1, hx.build_b), device)
        return idx

    def num_docs(self):
        return len(self.doc_ids)

    def num_postings(self):
        return len(self.posting_rows)

    def dev(self):
        if self._dev is None:
            self._dev = DeviceIndex(self.term_offsets, self.posting_rows, self.term_idfs,
                                    self.term_order_keys, self.doc_lens, self.doc_ids,
                                    self.avgdl, posting_weights=self.posting_weights,
                                    device=self.device)
        return self._dev

    def resolve(self, query_terms):
        return [self.vocab.get(t, NO_TERM) for t in query_terms]

    def bm25_topk(self, query_terms, k, p=None, stats=None, flags=0):
        """-> list[(doc_id, score)] ranked (score desc, id asc) (csr_index.cpp:77-104)."""
        p = p or Bm25Params()
        r = self.dev().search_lists([self.resolve(query_terms)], k, k1=p.k1, b=p.b, flags=flags)
        if stats is not None:
            stats.postings_touched += int(r["postings"][0])
        n = int(r["n"][0])
        return [(int(r["ids"][0, i]), float(r["scores"][0, i])) for i in range(n)]

    # MaxScore's output is identical to the exhaustive path (csr_index.hpp:77-79,
    # acceptance.cpp:144-171); the GPU path serves both with the same kernel.
    bm25_topk_maxscore = bm25_topk

    def bm25_term_score(self, term_id, posting_index, p=None):
        """csr_index.cpp:61-75: one posting's score (IndexError on ranges)."""
        p = p or Bm25Params()
        if term_id >= len(self.terms):
            raise IndexError("term_id out of range")
        lo, hi = int(self.term_offsets[term_id]), int(self.term_offsets[term_id + 1])
        if posting_index >= hi - lo:
            raise IndexError("posting_index out of term range")
        i = lo + posting_index
        return bm25_score(float(self.posting_weights[i]), float(self.term_idfs[term_id]),
                          float(self.doc_lens[self.posting_rows[i]]), self.avgdl, p)

    def compute_term_maxscores(self, p=None):
        """Per-term maximum posting score (csr_index.hpp:81-82), host-side,
        in bm25_score's operation order (vectorised over the postings)."""
        p = p or Bm25Params()
        df = np.diff(self.term_offsets.astype(np.int64))
        idf = np.repeat(self.term_idfs, df)
        tf = self.posting_weights
        dl = self.doc_lens[self.posting_rows].astype(np.float64)
        norm = dl / self.avgdl if self.avgdl > 0.0 else np.ones_like(dl)
        sc = idf * tf * (p.k1 + 1.0) / (tf + p.k1 * (1.0 - p.b + p.b * norm))
        out = np.zeros(len(self.terms))
        nz = df > 0
        if len(sc):
            out[nz] = np.maximum.reduceat(sc, self.term_offsets[:-1][nz].astype(np.int64))
        return out

    def query_upper_bound(self, query_terms, term_maxscores=None):
        """Sum of the known query terms' maxscores, duplicates counted
        (csr_index.hpp:84-86)."""
        if term_maxscores is None:  # cached per build parameters (one pass over P)
            key = (self.build_params.k1, self.build_params.b)
            if key not in self._maxscores:
                self._maxscores[key] = self.compute_term_maxscores(self.build_params)
            term_maxscores = self._maxscores[key]
        ms = term_maxscores
        ub = 0.0
        for t in query_terms:
            i = self.vocab.get(t)
            if i is not None:
                ub += float(ms[i])
        return ub

    def search_batch(self, queries, k, p=None, tau=None, tau_default=0.10, row_lo=0, row_hi=0,
                     flags=0, epsilon_guard=1e-9):
        """Batch of string queries (the cmd_search loop, hybridmem.cpp:227-313)."""
        p = p or Bm25Params()
        return self.dev().search_lists([self.resolve(q) for q in queries], k, k1=p.k1, b=p.b,
                                       tau=tau, tau_default=tau_default, epsilon_guard=epsilon_guard,
                                       row_lo=row_lo, row_hi=row_hi, flags=flags)


class Hidx:
    """A HIDX v1 file (the reference's save_index output, io.cpp:91-157) parsed
    by the framework's native reader; `arrays()` views its host arrays."""

    def __init__(self, path=None, handle=None, owner=None):
        L = lib()
        if handle is None:
            h = C.c_void_p()
            if L.hm_hidx_load(str(path).encode(), C.byref(h)) != 0:
                raise RuntimeError(L.hm_hidx_last_error().decode())
        else:  # a view into another container (an HTIX's flat index)
            h = C.c_void_p(handle)
        self._h, self._owner = h, owner
        self.view = CsrView()
        mode, k1, b = C.c_uint32(), C.c_double(), C.c_double()
        L.hm_hidx_view(h, C.byref(self.view), C.byref(mode), C.byref(k1), C.byref(b))
        self.mode, self.build_params = mode.value, Bm25Params(k1.value, b.value)

    def terms(self):
        L, out, p = lib(), [], C.c_char_p()
        for t in range(self.view.n_terms):
            n = L.hm_hidx_term(self._h, t, C.byref(p))
            out.append(C.string_at(p, n).decode())
        return out

    def arrays(self):
        v, nt, nd = self.view, self.view.n_terms, self.view.n_docs
        cts = {np.uint64: C.c_uint64, np.uint32: C.c_uint32, np.float64: C.c_double}

        def arr(ptr, n, dt):
            if not n:
                return np.zeros(0, dt)
            p = C.cast(ptr, C.POINTER(cts[dt]))
            return np.ctypeslib.as_array(p, (n,)).astype(dt, copy=True)
        P = int(arr(v.term_offsets, nt + 1, np.uint64)[-1]) if nt else 0
        return dict(term_offsets=arr(v.term_offsets, nt + 1, np.uint64),
                    posting_rows=arr(v.posting_rows, P, np.uint32),
                    posting_weights=arr(v.posting_weights, P, np.float64),
                    idf=arr(v.term_idfs, nt, np.float64),
                    maxscore=arr(lib().hm_hidx_maxscores(self._h), nt, np.float64),
                    order_key=arr(v.term_order_keys, nt, np.float64),
                    doc_lens=arr(v.doc_lens, nd, np.uint32), doc_ids=arr(v.doc_ids, nd, np.uint64),
                    avgdl=v.avgdl)

    def bridge_index(self, device=0):
        """A Bridge-mode file (mode 1) uploaded straight to a DeviceBridge."""
        if self.mode != 1:
            raise RuntimeError("bridge scoring requires a bridge-mode index")
        v = self.view
        bv = BridgeView(v.n_terms, v.term_offsets, v.posting_rows, v.posting_weights, v.n_docs, v.doc_ids)
        h = C.c_void_p()
        _check(lib().hm_bridge_create(C.byref(bv), device, C.byref(h)))
        return DeviceBridge._adopt(h, device, v.n_terms, v.n_docs)

    def device_index(self, device=0):
        """Upload straight from the parsed file (no Python copies)."""
        if self.mode != 0:
            raise RuntimeError("BM25 scoring requires a BM25-mode index")
        h = C.c_void_p()
        _check(lib().hm_index_create(C.byref(self.view), device, C.byref(h)))
        return DeviceIndex._adopt(h, device, self.view.n_terms, self.view.n_docs,
                                  np.diff(self.arrays()["term_offsets"].astype(np.int64)))

    def close(self):
        if getattr(self, "_h", None):
            if getattr(self, "_owner", None) is None:
                lib().hm_hidx_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except TypeError:  # interpreter shutdown: module globals already cleared
            pass


class Htix:
    """A HTIX v1 file (save_temporal_index, io.cpp:234-268) read by the native
    reader as one partition-ordered flat index over the shared statistics."""

    def __init__(self, path):
        L = lib()
        h = C.c_void_p()
        if L.hm_htix_load(str(path).encode(), C.byref(h)) != 0:
            raise RuntimeError(L.hm_hidx_last_error().decode())
        self._h = h
        self.flat = Hidx(handle=L.hm_htix_flat(h), owner=self)
        K = C.c_uint32()
        pr, ws, we = C.c_void_p(), C.c_void_p(), C.c_void_p()
        L.hm_htix_partitions(h, C.byref(K), C.byref(pr), C.byref(ws), C.byref(we))
        n = K.value
        self.part_row = np.ctypeslib.as_array(C.cast(pr, C.POINTER(C.c_uint32)), (n + 1,)).copy()
        self.window_start = np.ctypeslib.as_array(C.cast(ws, C.POINTER(C.c_int64)), (n,)).copy() if n else np.zeros(0, np.int64)
        self.window_end = np.ctypeslib.as_array(C.cast(we, C.POINTER(C.c_int64)), (n,)).copy() if n else np.zeros(0, np.int64)
        w, e, lam, km, td = C.c_int64(), C.c_double(), C.c_double(), C.c_uint32(), C.c_uint64()
        L.hm_htix_params(h, C.byref(w), C.byref(e), C.byref(lam), C.byref(km), C.byref(td))
        self.params = TemporalParams(w.value, e.value, lam.value, km.value)
        self.total_docs = td.value

    def temporal_index(self, device=0):
        """(TemporalIndex on the device, the CsrIndex mirror for term lookup)."""
        a = self.flat.arrays()
        idx = CsrIndex(self.flat.terms(), a["term_offsets"], a["posting_rows"], a["posting_weights"],
                       a["idf"], a["order_key"], a["doc_lens"], a["doc_ids"], a["avgdl"],
                       self.flat.build_params, device)
        return TemporalIndex(self.flat.device_index(device), self.part_row, self.params, host=idx), idx

    def close(self):
        if getattr(self, "_h", None):
            self.flat._h = None
            lib().hm_htix_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except TypeError:  # interpreter shutdown: module globals already cleared
            pass


def k_star(epsilon, lam):
    """temporal_index.cpp:9-17."""
    if not (0.0 < epsilon < 1.0):
        raise ValueError("epsilon must be in (0,1)")
    if not lam > 0.0:
        raise ValueError("lambda must be > 0")
    return max(1, int(math.ceil(math.log(1.0 / epsilon) / lam)))


@dataclass
class TemporalParams:
    """hybrid::TemporalParams (temporal_index.hpp:12-17)."""
    window_ms: int = 7 * 24 * 3600 * 1000
    epsilon: float = 0.05
    lambda_hat: float = 1.4
    k_max_partitions: int = 4


@dataclass
class TemporalStats:
    """hybrid::TemporalStats (temporal_index.hpp:33-37)."""
    partitions_searched: int = 0
    postings_touched: int = 0
    early_stopped: bool = False


class TemporalIndex:
    """Time-partitioned index on one device (temporal_index.hpp:40-72).

    Rows are laid out partition by partition (oldest first, insertion order
    inside a partition) and every partition shares the flat corpus statistics
    (temporal_index.cpp:136-142), so the newest `budget` partitions are a row
    suffix and scoring them is the flat kernel restricted to that row window.
    The result equals the reference's greedy most-recent-first merge
    (temporal_index.cpp:72-123)."""

    def __init__(self, flat_dev, part_row, params=None, host=None):
        self.dev = flat_dev
        self.part_row = np.asarray(part_row, np.uint32)
        self.params = params or TemporalParams()
        self.host = host  # CsrIndex mirror of the flat arrays (vocabulary, partition bounds)

    def partition_upper_bound(self, i, query_terms):
        """temporal_index.cpp:58-70: sum of partition i's term maxscores over
        the query terms (duplicates counted).  A partition's maxscores are the
        build-parameter scores of its own postings under the shared flat
        statistics (temporal_index.cpp:136-142)."""
        if i >= self.num_partitions():
            raise IndexError("partition index out of range")
        h = self.host
        lo, hi = int(self.part_row[i]), int(self.part_row[i + 1])
        bp = h.build_params
        ub = 0.0
        cache = {}
        for t in query_terms:
            tid = h.vocab.get(t)
            if tid is None:
                continue
            if tid not in cache:
                a, b = int(h.term_offsets[tid]), int(h.term_offsets[tid + 1])
                rows = h.posting_rows[a:b]
                s0 = a + int(np.searchsorted(rows, lo))
                s1 = a + int(np.searchsorted(rows, hi))
                ms = 0.0
                if s1 > s0:
                    tf = h.posting_weights[s0:s1]
                    dl = h.doc_lens[h.posting_rows[s0:s1]].astype(np.float64)
                    norm = dl / h.avgdl if h.avgdl > 0.0 else np.ones_like(dl)
                    sc = h.term_idfs[tid] * tf * (bp.k1 + 1.0) / (tf + bp.k1 * (1.0 - bp.b + bp.b * norm))
                    ms = float(sc.max())
                cache[tid] = ms
            ub += cache[tid]
        return ub

    def topk(self, query_terms, k, p=None, stats=None, use_ub_stop=True):
        """TemporalIndex::topk (temporal_index.cpp:72-123) for one query:
        -> [(DocId, score)]; stats: TemporalStats (partitions_searched /
        early_stopped as the reference; postings in the exhaustive accounting
        of hm_results.postings)."""
        lists, st = self.topk_many([query_terms], k, p, use_ub_stop)
        if stats is not None:
            stats.partitions_searched += st[0].partitions_searched
            stats.postings_touched += st[0].postings_touched
            stats.early_stopped = stats.early_stopped or st[0].early_stopped
        return lists[0]

    def topk_many(self, queries, k, p=None, use_ub_stop=True):
        """TemporalIndex::topk for a batch of string queries: every partition of
        the budget min(k*, k_max, K) searched for every query in ONE device call
        (hm_search_batch_parts), the per-partition lists merged newest first
        with the reference's admissible upper-bound stop.
        -> (lists of [(DocId, score)], [TemporalStats])."""
        p = p or Bm25Params()
        nq = len(queries)
        out = [[] for _ in range(nq)]
        stats = [TemporalStats() for _ in range(nq)]
        K = self.num_partitions()
        if K == 0 or k == 0 or nq == 0:
            return out, stats
        first = K - self.budget()
        bp = self.host.build_params
        ub_valid = p.k1 == bp.k1 and p.b == bp.b
        tids = [self.host.resolve(q) for q in queries]
        off = np.zeros(nq + 1, np.uint32)
        off[1:] = np.cumsum([len(t) for t in tids])
        flat = np.array([x for t in tids for x in t], np.uint32)
        r = self.dev.search_parts(off, flat, k, self.part_row[first:], k1=p.k1, b=p.b)
        key = lambda e: (-e[1], e[0])  # noqa: E731  (RankedList::better order)
        for q in range(nq):
            cur, st = out[q], stats[q]
            for i in range(K - 1, first - 1, -1):
                c = i - first
                st.partitions_searched += 1
                st.postings_touched += int(r["postings"][c, q])
                m = int(r["n"][c, q])
                new = list(zip(r["ids"][c, q, :m].tolist(), r["scores"][c, q, :m].tolist()))
                cur[:] = sorted(cur + new, key=key)[:k]  # partitions hold disjoint documents
                if use_ub_stop and ub_valid and i > first and len(cur) == k:
                    rest = max([0.0] + [self.partition_upper_bound(j, queries[q]) for j in range(first, i)])
                    if cur[-1][1] > rest:
                        st.early_stopped = True
                        break
        return out, stats

    def num_partitions(self):
        return len(self.part_row) - 1

    def budget(self):
        K = self.num_partitions()
        if K == 0:
            return 0
        p = self.params
        return min(k_star(p.epsilon, p.lambda_hat), p.k_max_partitions, K)

    def window(self):
        K = self.num_partitions()
        first = K - self.budget()
        return int(self.part_row[first]), int(self.part_row[K])

    def topk_batch(self, q_off, q_tid, k, k1=1.2, b=0.75, **kw):
        if self.num_partitions() == 0 or k == 0:
            nq = len(q_off) - 1
            return dict(ids=np.zeros((nq, 0), np.uint64), scores=np.zeros((nq, 0)),
                        n=np.zeros(nq, np.uint32), conf=np.zeros(nq), skip=np.zeros(nq, np.uint8),
                        postings=np.zeros(nq, np.uint64), n_exact=0)
        lo, hi = self.window()
        if hi <= lo:  # newest partitions are empty: nothing to score
            nq = len(q_off) - 1
            return dict(ids=np.zeros((nq, max(k, 1)), np.uint64),
                        scores=np.zeros((nq, max(k, 1))), n=np.zeros(nq, np.uint32),
                        conf=np.zeros(nq), skip=(np.zeros(nq) >= kw.get("tau_default", 0.10)
                                                 ).astype(np.uint8),
                        postings=np.zeros(nq, np.uint64), n_exact=0)
        return self.dev.search_batch(q_off, q_tid, k, k1=k1, b=b, row_lo=lo, row_hi=hi, **kw)


# ------------------------------------------------------------------ bridge
class SparseVector:
    """hybrid::SparseVector (bridge.hpp:12-19): strictly increasing term ids,
    positive values."""

    def __init__(self, indices=(), values=()):
        self.indices = np.ascontiguousarray(indices, np.uint32)
        self.values = np.ascontiguousarray(values, np.float64)

    def nnz(self):
        return len(self.indices)

    def validate(self):
        """bridge.cpp:10-20 (std::invalid_argument -> ValueError, same messages)."""
        if len(self.indices) != len(self.values):
            raise ValueError("indices/values length mismatch")
        if len(self.indices) > 1 and not (np.diff(self.indices.astype(np.int64)) > 0).all():
            raise ValueError("sparse vector indices must be strictly increasing")
        if not (self.values > 0.0).all():
            raise ValueError("sparse vector values must be > 0")


def _sparse_batch(queries):
    off = np.zeros(len(queries) + 1, np.uint64)
    off[1:] = np.cumsum([q.nnz() for q in queries])
    idx = np.concatenate([q.indices for q in queries]) if off[-1] else np.zeros(0, np.uint32)
    val = np.concatenate([q.values for q in queries]) if off[-1] else np.zeros(0, np.float64)
    return off, np.ascontiguousarray(idx, np.uint32), np.ascontiguousarray(val, np.float64)


class DeviceBridge:
    """An HBM-resident Bridge-mode index (hm_bridge): rows, learned weights,
    DocIds in the reference's CsrIndex layout."""

    def __init__(self, term_offsets, posting_rows, posting_weights, doc_ids, device=0):
        keep = (np.ascontiguousarray(term_offsets, np.uint64), np.ascontiguousarray(posting_rows, np.uint32),
                np.ascontiguousarray(posting_weights, np.float64), np.ascontiguousarray(doc_ids, np.uint64))
        v = BridgeView(len(keep[0]) - 1, _ptr(keep[0]), _ptr(keep[1]), _ptr(keep[2]), len(keep[3]),
                       _ptr(keep[3]))
        h = C.c_void_p()
        _check(lib().hm_bridge_create(C.byref(v), device, C.byref(h)))
        self._h, self.device, self.n_terms, self.n_docs = h, device, len(keep[0]) - 1, len(keep[3])

    @classmethod
    def _adopt(cls, h, device, n_terms, n_docs):
        self = cls.__new__(cls)
        self._h, self.device, self.n_terms, self.n_docs = h, device, n_terms, n_docs
        return self

    def close(self):
        if getattr(self, "_h", None):
            lib().hm_bridge_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except TypeError:  # interpreter shutdown: module globals already cleared
            pass

    def search_batch(self, queries, k, row_lo=0, row_hi=0, flags=0):
        """Host-buffer batch (hm_bridge_search_batch) over SparseVectors.
        -> dict(ids[nq,k], scores[nq,k], n[nq], postings[nq])"""
        off, idx, val = _sparse_batch(queries)
        return self.search_arrays(off, idx, val, k, row_lo, row_hi, flags)

    def search_arrays(self, q_off, q_idx, q_val, k, row_lo=0, row_hi=0, flags=0):
        q_off = np.ascontiguousarray(q_off, np.uint64)
        q_idx = np.ascontiguousarray(q_idx, np.uint32)
        q_val = np.ascontiguousarray(q_val, np.float64)
        nq = len(q_off) - 1
        kk = max(int(k), 1)
        out = dict(ids=np.zeros((nq, kk), np.uint64), scores=np.zeros((nq, kk), np.float64),
                   n=np.zeros(nq, np.uint32), postings=np.zeros(nq, np.uint64))
        qb = BridgeBatch(nq, _ptr(q_off), _ptr(q_idx) if len(q_idx) else None,
                         _ptr(q_val) if len(q_val) else None, int(k), row_lo, row_hi, 0, flags)
        r = Results(_ptr(out["ids"]), _ptr(out["scores"]), _ptr(out["n"]), None, None,
                    _ptr(out["postings"]))
        _check(lib().hm_bridge_search_batch(self._h, C.byref(qb), C.byref(r)))
        if k == 0:
            out["ids"] = out["ids"][:, :0]
            out["scores"] = out["scores"][:, :0]
        return out

    def search_batch_device(self, q_off, q_idx, q_val, out, k, max_nnz, row_lo=0, row_hi=0, flags=0,
                            stream=None):
        """Device-resident batch (torch CUDA tensors: q_off int64, q_idx int32,
        q_val f64; out ids/scores/n/postings), enqueued on `stream`."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(q_off.device)
        qb = BridgeBatch(q_off.numel() - 1, q_off.data_ptr(), q_idx.data_ptr(), q_val.data_ptr(), int(k),
                         row_lo, row_hi, int(max_nnz), flags)
        r = Results(out["ids"].data_ptr(), out["scores"].data_ptr(), out["n"].data_ptr(), None, None,
                    out["postings"].data_ptr())
        _check(lib().hm_bridge_search_batch_device(self._h, C.byref(qb), C.byref(r), st.cuda_stream))
        if flags & HM_FLAG_TIMING:
            t = C.c_float()
            lib().hm_bridge_last_timing(C.byref(t))
            return t.value


class BridgeIndex:
    """A Bridge-mode hybrid::CsrIndex (bridge_ingest, bridge.cpp:22-73) whose
    searches run on the GPU (bridge_topk / bridge_topk_maxscore,
    bridge.cpp:112-204: identical outputs, one device path)."""

    def __init__(self, term_offsets, posting_rows, posting_weights, doc_ids, doc_lens, avgdl,
                 term_maxscores, device=0):
        self.term_offsets = np.ascontiguousarray(term_offsets, np.uint64)
        self.posting_rows = np.ascontiguousarray(posting_rows, np.uint32)
        self.posting_weights = np.ascontiguousarray(posting_weights, np.float64)
        self.doc_ids = np.ascontiguousarray(doc_ids, np.uint64)
        self.doc_lens = np.ascontiguousarray(doc_lens, np.uint32)
        self.avgdl = avgdl
        self.term_maxscores = np.ascontiguousarray(term_maxscores, np.float64)
        self.device = device
        self._dev = None

    @property
    def n_terms(self):
        return len(self.term_offsets) - 1

    def num_docs(self):
        return len(self.doc_ids)

    def num_postings(self):
        return len(self.posting_rows)

    @property
    def dev(self):
        if self._dev is None:
            self._dev = DeviceBridge(self.term_offsets, self.posting_rows, self.posting_weights,
                                     self.doc_ids, self.device)
        return self._dev

    def bridge_topk(self, query_vec, k, stats=None):
        """-> [(DocId, score), ...] ranked (score desc, DocId asc)."""
        query_vec.validate()
        r = self.dev.search_batch([query_vec], min(int(k), self.num_docs()))  # k > N: same list
        if stats is not None:
            stats.postings_touched += int(r["postings"][0])
        n = int(r["n"][0])
        return [(int(i), float(s)) for i, s in zip(r["ids"][0, :n], r["scores"][0, :n])]

    def bridge_topk_maxscore(self, query_vec, k, stats=None):
        return self.bridge_topk(query_vec, k, stats)

    def search_batch(self, queries, k, row_lo=0, row_hi=0, flags=0):
        return self.dev.search_batch(queries, k, row_lo, row_hi, flags)


def bridge_ingest(doc_vectors, device=0):
    """bridge_ingest (bridge.cpp:22-73): [(DocId, SparseVector)] -> BridgeIndex.
    Duplicate ids raise RuntimeError("duplicate doc id: X"); vectors are validated."""
    seen = set()
    dim = 0
    for doc_id, vec in doc_vectors:
        if doc_id in seen:
            raise RuntimeError(f"duplicate doc id: {doc_id}")
        seen.add(doc_id)
        vec.validate()
        if vec.nnz():
            dim = max(dim, int(vec.indices[-1]) + 1)
    n = len(doc_vectors)
    lens = np.array([v.nnz() for _, v in doc_vectors], np.uint32)
    rows = np.repeat(np.arange(n, dtype=np.uint32), lens)
    tids = np.concatenate([v.indices for _, v in doc_vectors]) if lens.sum() else np.zeros(0, np.uint32)
    vals = np.concatenate([v.values for _, v in doc_vectors]) if lens.sum() else np.zeros(0)
    order = np.argsort(tids, kind="stable")  # per-term postings in doc order (rows ascend)
    off = np.zeros(dim + 1, np.uint64)
    off[1:] = np.cumsum(np.bincount(tids, minlength=dim)[:dim])
    w = vals[order]
    maxw = np.zeros(dim)
    if len(w):
        np.maximum.at(maxw, tids[order], w)
    len_sum = 0.0
    for x in lens:  # sequential double sum, as the reference (bridge.cpp:47)
        len_sum += float(x)
    avgdl = 0.0 if n == 0 else len_sum / n
    ids = np.array([d for d, _ in doc_vectors], np.uint64)
    return BridgeIndex(off, rows[order], w, ids, lens, avgdl, maxw, device)


def bridge_export(idx):
    """bridge_export (bridge.cpp:75-90): the exact inverse of bridge_ingest."""
    n = idx.num_docs()
    df = np.diff(idx.term_offsets.astype(np.int64))
    tids = np.repeat(np.arange(idx.n_terms, dtype=np.uint32), df)
    order = np.argsort(idx.posting_rows, kind="stable")  # term-major stays ascending per doc
    rows = idx.posting_rows[order]
    cuts = np.searchsorted(rows, np.arange(n + 1))
    t, w = tids[order], idx.posting_weights[order]
    return [(int(idx.doc_ids[d]), SparseVector(t[cuts[d]:cuts[d + 1]], w[cuts[d]:cuts[d + 1]]))
            for d in range(n)]


# ------------------------------------------------------------------ dense
DENSE_MAX_K = 256


class DenseIndex:
    """An HBM-resident hybrid::EmbeddingMatrix (dense.hpp:13-22): row-major
    fp32 unit vectors + DocIds.  dense_topk runs on the GPU, bit-identical to
    the reference (src/dense.cpp:86-101)."""

    def __init__(self, data, doc_ids, device=0):
        data = np.ascontiguousarray(data, np.float32)
        doc_ids = np.ascontiguousarray(doc_ids, np.uint64)
        if data.ndim != 2 or data.shape[0] != len(doc_ids):
            raise ValueError("embedding dimension mismatch")
        self.dim, self.count = int(data.shape[1]), int(data.shape[0])
        v = DenseView(self.dim, self.count, _ptr(data), _ptr(doc_ids))
        h = C.c_void_p()
        _check(lib().hm_dense_create(C.byref(v), device, C.byref(h)))
        self._h, self.device = h, device

    def close(self):
        if getattr(self, "_h", None):
            lib().hm_dense_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except TypeError:  # interpreter shutdown: module globals already cleared
            pass

    def search_batch(self, queries, k, flags=0):
        """queries [nq x dim] fp32 -> dict(ids[nq,k], scores[nq,k], n[nq])"""
        q = np.ascontiguousarray(queries, np.float32)
        if q.ndim == 1:
            q = q[None, :]
        nq = q.shape[0]
        kk = max(int(k), 1)
        out = dict(ids=np.zeros((nq, kk), np.uint64), scores=np.zeros((nq, kk)), n=np.zeros(nq, np.uint32))
        b = DenseBatch(nq, q.shape[1], _ptr(q), int(k), flags)
        r = Results(_ptr(out["ids"]), _ptr(out["scores"]), _ptr(out["n"]), None, None, None)
        _check(lib().hm_dense_search_batch(self._h, C.byref(b), C.byref(r)))
        return out

    def search_batch_device(self, queries, out, k, flags=0, stream=None):
        """Device-resident batch (torch CUDA tensors: queries [nq,dim] f32;
        out ids int64 / scores f64 [nq,k], n int32 [nq])."""
        import torch
        st = stream if stream is not None else torch.cuda.current_stream(queries.device)
        b = DenseBatch(queries.shape[0], queries.shape[1], queries.data_ptr(), int(k), flags)
        r = Results(out["ids"].data_ptr(), out["scores"].data_ptr(), out["n"].data_ptr(), None, None, None)
        _check(lib().hm_dense_search_batch_device(self._h, C.byref(b), C.byref(r), st.cuda_stream))
        if flags & HM_FLAG_TIMING:
            t = C.c_float()
            lib().hm_dense_last_timing(C.byref(t))
            return t.value

    @staticmethod
    def last_stats():
        """(path, n_overflow, n_candidates) of this thread's last dense batch
        (hm_dense_last_stats; candidates only for HM_FLAG_TIMING batches)."""
        p, o, c = C.c_uint32(), C.c_uint32(), C.c_uint64()
        lib().hm_dense_last_stats(C.byref(p), C.byref(o), C.byref(c))
        return p.value, o.value, c.value

    def dense_topk(self, query_vec, k):
        """hybrid::dense_topk: -> [(DocId, score)] over every row (ties by DocId)."""
        q = np.asarray(query_vec, np.float32)
        if q.shape != (self.dim,):
            raise ValueError("query dimension mismatch")
        r = self.search_batch(q[None, :], min(int(k), self.count))
        n = int(r["n"][0])
        return [(int(i), float(s)) for i, s in zip(r["ids"][0, :n], r["scores"][0, :n])]


# ------------------------------------------------------------------ fusion
@dataclass
class FusionParams:
    """hybrid::FusionParams (fusion.hpp:17-33)."""
    k_rrf: float = 60.0
    alpha: float = 0.005
    tau_ms: int = 30 * 24 * 3600 * 1000
    tau_overrides_ms: dict = None
    beta: float = 0.0
    recency_qtypes: set = None
    apply_bonus_when_qtype_unknown: bool = True

    def tau_for(self, qtype):
        if qtype is not None and self.tau_overrides_ms and qtype in self.tau_overrides_ms:
            return self.tau_overrides_ms[qtype]
        return self.tau_ms


def _ranked(scores):
    """RankedList::sort_and_truncate over all entries: (score desc, DocId asc)."""
    return sorted(scores.items(), key=lambda e: (-e[1], e[0]))


def rrf(lists, k_rrf):
    """Reciprocal rank fusion (fusion.cpp:8-21), same operation order."""
    if not k_rrf > 0.0:
        raise ValueError("k_rrf must be > 0")
    score = {}
    for lst in lists:
        for r, (doc, _) in enumerate(lst):
            score[doc] = score.get(doc, 0.0) + 1.0 / (k_rrf + float(r + 1))
    return _ranked(score)


def agent_rrf(sparse, dense, records, query_ts_ms, qtype, p):
    """agent_rrf (fusion.cpp:23-50): RRF + alpha*exp(-dt/tau) + beta*w.
    records: callable DocId -> object with ts_ms / weight, or None."""
    fused = dict(rrf([sparse, dense], p.k_rrf))
    if not p.recency_qtypes:
        bonus_on = qtype is not None or p.apply_bonus_when_qtype_unknown
    elif qtype is not None:
        bonus_on = qtype in p.recency_qtypes
    else:
        bonus_on = p.apply_bonus_when_qtype_unknown
    tau = float(p.tau_for(qtype))
    for doc in list(fused):
        rec = records(doc)
        if rec is None:
            raise RuntimeError(f"record missing from lookup: {doc}")
        if bonus_on and p.alpha > 0.0:
            dt = float(max(0, query_ts_ms - rec.ts_ms))
            fused[doc] += p.alpha * math.exp(-dt / tau)
        if p.beta != 0.0:
            fused[doc] += p.beta * rec.weight
    return _ranked(fused)


@dataclass
class CascadeConfig:
    """hybrid::CascadeConfig (cascade.hpp:19-27), Margin proxy."""
    conf_threshold: float = 0.10
    per_qtype_thresholds: dict = None
    skip_cost_ms: float = 0.4
    escalate_cost_ms: float = 53.2
    epsilon_guard: float = 1e-9


@dataclass
class CascadeDecision:
    results: list
    escalated: bool
    confidence: float
    accounted_cost_ms: float


def cascade_retrieve(k, cfg, bm25_fn, dense_fn, records, query_ts_ms, fusion, qtype=None):
    """cascade_retrieve (cascade.cpp:44-101) with the Margin proxy: BM25
    always; skip dense when the confidence clears tau, else agent_rrf."""
    sparse = bm25_fn(k)
    conf = margin([s for _, s in sparse], cfg.epsilon_guard)
    tau = cfg.conf_threshold
    if qtype is not None and cfg.per_qtype_thresholds and qtype in cfg.per_qtype_thresholds:
        tau = cfg.per_qtype_thresholds[qtype]
    if conf >= tau:
        return CascadeDecision(sparse, False, conf, cfg.skip_cost_ms)
    fused = agent_rrf(sparse, dense_fn(k), records, query_ts_ms, qtype, fusion)[:k]
    return CascadeDecision(fused, True, conf, cfg.escalate_cost_ms)


def cascade_batch(csr, dense, query_terms, query_vecs, k, records, query_ts_ms, fusion=None, cfg=None,
                  p=None):
    """The cascade over a whole batch on the GPU: one BM25 batch (Margin +
    skip computed on the device), one dense batch over the escalated
    queries only, agent_rrf on the host (O(k) per query).  Per query it
    equals cascade_retrieve with bm25_fn = bm25_topk, dense_fn = dense_topk.
    -> list[CascadeDecision]"""
    fusion = fusion or FusionParams()
    cfg = cfg or CascadeConfig()
    p = p or Bm25Params()
    r = csr.search_batch(query_terms, k, p, tau_default=cfg.conf_threshold, epsilon_guard=cfg.epsilon_guard)
    esc = [i for i in range(len(query_terms)) if not r["skip"][i]]
    dres = dense.search_batch(np.asarray(query_vecs, np.float32)[esc], min(int(k), dense.count)) if esc else None
    out = []
    ei = {q: j for j, q in enumerate(esc)}
    for i in range(len(query_terms)):
        n = int(r["n"][i])
        sparse = [(int(d), float(x)) for d, x in zip(r["ids"][i, :n], r["scores"][i, :n])]
        conf = float(r["conf"][i])
        if i not in ei:
            out.append(CascadeDecision(sparse, False, conf, cfg.skip_cost_ms))
            continue
        j = ei[i]
        m = int(dres["n"][j])
        dl = [(int(d), float(x)) for d, x in zip(dres["ids"][j, :m], dres["scores"][j, :m])]
        ts = query_ts_ms[i] if np.ndim(query_ts_ms) else query_ts_ms
        out.append(CascadeDecision(agent_rrf(sparse, dl, records, ts, None, fusion)[:k], True, conf,
                                   cfg.escalate_cost_ms))
    return out
