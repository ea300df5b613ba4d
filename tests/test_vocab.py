"""CPU: the native query-string resolver (hm_vocab_*; make_plan's vocab lookup,
csr_index.cpp:31-48, and load_queries_tsv's whitespace split, io.cpp:389-391)
equals Python's str.split + dict lookup, single- and multi-threaded."""
import numpy as np
import pytest

from paper_2605_25092_b200 import search

NO = search.NO_TERM


def py_resolve(vocab, queries):
    ids = {t: i for i, t in enumerate(vocab)}
    toks = [[ids.get(t, NO) for t in q.split()] for q in queries]
    off = np.zeros(len(queries) + 1, np.uint32)
    off[1:] = np.cumsum([len(t) for t in toks])
    flat = np.array([x for t in toks for x in t], np.uint32)
    return off, flat


def test_resolve_matches_split_and_lookup():
    rng = np.random.default_rng(3)
    vocab = sorted({"w%d" % i for i in range(5000)} | {"a", "ab", "abcdefgh", "abcdefghi", "ünï"})
    v = search.Vocab(vocab)
    assert len(v) == len(vocab)
    seps = [" ", "  ", "\t", " \n", "\r\v\f "]
    queries = ["", "   ", "a", "ab abcdefgh abcdefghi ünï zz", "\tw1\tw2 ", "w99999"]
    for _ in range(10000):
        words = ["w%d" % rng.integers(0, 6000) for _ in range(rng.integers(0, 9))]
        queries.append("".join(w + seps[rng.integers(0, len(seps))] for w in words))
    want = py_resolve(vocab, queries)
    for th in (1, 0, 7):
        got = v.resolve(queries, n_threads=th)
        assert (got[0] == want[0]).all() and (got[1] == want[1]).all()


def test_duplicate_vocabulary_rejected():
    with pytest.raises(ValueError, match="duplicate term"):
        search.Vocab(["a", "b", "a"])


def test_capacity_error():
    v = search.Vocab(["a"])
    with pytest.raises(IndexError):
        import ctypes as C
        off = np.array([0, 5], np.uint64)
        qo = np.zeros(2, np.uint32)
        qt = np.zeros(1, np.uint32)
        n = C.c_uint64()
        search._check(search.lib().hm_vocab_resolve(v._h, 1, b"a a a", search._ptr(off), search._ptr(qo),
                                                    search._ptr(qt), 1, C.byref(n), 1))
    assert n.value == 3
