"""CPU: the C-ABI library loads, exports every symbol include/hm_b200.h declares,
and fails loudly (no CPU fallback) when no GPU is present."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2605_25092_b200 import _lib, search, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(hm_[a-z0-9_]+)\s*\(", text)))


def test_hm_b200_exports_every_declared_symbol():
    names = declared("hm_b200.h")
    assert "hm_search_batch" in names and "hm_index_create" in names
    lib = ctypes.CDLL(os.path.join(_lib.LIB_DIR, "libhm_b200.so"))
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(search.EXPORTS) <= set(names)


def test_hm_synth_exports_every_declared_symbol():
    names = declared("hm_synth.h")
    lib = ctypes.CDLL(os.path.join(_lib.LIB_DIR, "libhm_synth.so"))
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_margin_export_matches_reference_rule():
    assert abs(search.margin([8.74, 2.13, 1.40, 0.91, 0.83]) - 0.756) <= 1e-3
    assert abs(search.margin([4.21, 3.97, 3.48, 3.11, 2.96]) - 0.057) <= 1e-3
    assert search.margin([]) == 0.0 and search.margin([5.0]) == 0.0 and search.margin([0.0, 0.0]) == 0.0


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_gpu():
    hx = synth.HostIndex(synth.Corpus(n_records=100))
    with pytest.raises(RuntimeError, match="no CUDA device"):
        search.DeviceIndex.from_host(hx)
    # the bridge and dense channels fail the same way (no CPU scoring path)
    bi = search.bridge_ingest([(1, search.SparseVector([0, 3], [0.5, 1.0]))])
    with pytest.raises(RuntimeError, match="no CUDA device"):
        bi.bridge_topk(search.SparseVector([0], [1.0]), 5)
    with pytest.raises(RuntimeError, match="no CUDA device"):
        search.DenseIndex(np.ones((4, 8), np.float32), np.arange(4, dtype=np.uint64))


def test_bridge_and_dense_argument_errors_before_any_device_work():
    """Malformed inputs are rejected with the reference's messages by the host
    side of the ABI (SparseVector::validate, bridge.cpp:10-20; EmbeddingMatrix
    shape checks, dense.cpp:44-52) -- no GPU needed to see them."""
    with pytest.raises(ValueError, match="strictly increasing"):
        search.SparseVector([2, 2], [1.0, 1.0]).validate()
    with pytest.raises(ValueError, match="must be > 0"):
        search.bridge_ingest([(1, search.SparseVector([0], [0.0]))])
    with pytest.raises(ValueError, match="embedding dimension mismatch"):
        search.DenseIndex(np.ones((4, 8), np.float32), np.arange(3, dtype=np.uint64))


def test_sm100a_cubin_present():
    """The library carries sm_100a SASS (not a PTX-only or other-arch build)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          os.path.join(_lib.LIB_DIR, "libhm_b200.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_k_star_and_temporal_budget_host_logic():
    assert search.k_star(0.05, 1.4) == 3 and search.k_star(0.01, 0.5) == 10
    assert search.k_star(0.999999, 1.0) == 1
    for bad in [(0.0, 1.0), (1.0, 1.0), (0.05, 0.0)]:
        with pytest.raises(ValueError):
            search.k_star(*bad)
    t = search.TemporalIndex(None, np.array([0, 5, 9, 9, 20], np.uint32))
    assert t.num_partitions() == 4 and t.budget() == 3 and t.window() == (5, 20)
    t.params.k_max_partitions = 1
    assert t.window() == (9, 20)


def test_confidence_proxies_and_term_scores_mirror_reference():
    """The host-side pieces of the mirror: every confidence proxy
    (cascade.cpp:10-38), bm25_score, bm25_term_score, compute_term_maxscores
    and query_upper_bound against the reference library, bit for bit."""
    from oracle import ref
    rng = np.random.default_rng(3)
    lists = [[8.74, 2.13, 1.40, 0.91, 0.83], [4.21, 3.97, 3.48, 3.11, 2.96], [5.0], [], [0.0, 0.0],
             list(np.sort(rng.random(10))[::-1] * 7)]
    for sc in lists:
        for proxy in (0, 1, 2):
            assert search.confidence(sc, proxy) == ref.confidence(sc, proxy), (sc, proxy)
    with pytest.raises(ValueError):
        search.confidence([1.0, 0.5], search.CLASSIFIER)
    from _util import export_to_csr, toy_docs
    ri = ref.RefIndex.from_texts(toy_docs(), ref.TOK_MINIMAL)
    csr = export_to_csr(ri)
    e = ri.export()
    for t in range(len(e["terms"])):
        for j in range(int(e["term_offsets"][t + 1] - e["term_offsets"][t])):
            i = int(e["term_offsets"][t]) + j
            want = ref.bm25_score(float(e["posting_weights"][i]), float(e["idf"][t]),
                                  float(e["doc_lens"][e["posting_rows"][i]]), e["avgdl"])
            assert csr.bm25_term_score(t, j) == want
    assert (csr.compute_term_maxscores().view(np.uint64) == e["maxscore"].view(np.uint64)).all()
    q = ["cat", "dog", "cat", "unicorn"]
    assert csr.query_upper_bound(q, e["maxscore"]) == sum(float(e["maxscore"][e["terms"].index(t)]) for t in q
                                                          if t in e["terms"])
    with pytest.raises(IndexError, match="term_id out of range"):
        csr.bm25_term_score(len(e["terms"]), 0)
    with pytest.raises(IndexError, match="posting_index out of term range"):
        csr.bm25_term_score(0, 99)
