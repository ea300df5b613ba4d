"""An index whose rows repeat DocIds (identical documents stored twice under
one id, as a caller's records may): equal (score, DocId) pairs must all be
emitted -- the epilogue's rank counting and the slab merge order them by row
/ list -- and the answers equal the C restatement of the reference."""
import numpy as np
import pytest

from _util import check_batch, restate, search

pytestmark = pytest.mark.gpu


def build(docs, ids):
    V = 1 + max(t for d in docs for t in d)
    post = [[] for _ in range(V)]
    for r, d in enumerate(docs):
        for t, f in sorted(d.items()):
            post[t].append((r, f))
    off = np.zeros(V + 1, np.uint64)
    off[1:] = np.cumsum([len(p) for p in post])
    rows = np.array([r for p in post for r, _ in p], np.uint32)
    tf = np.array([f for p in post for _, f in p], np.uint32)
    N = len(docs)
    lens = np.array([sum(d.values()) for d in docs], np.uint32)
    avgdl = float(lens.sum()) / N
    df = np.diff(off.astype(np.int64))
    idf = np.log(1.0 + (N - df + 0.5) / (df + 0.5))
    k1, b = 1.2, 0.75
    ms = np.zeros(V)
    for t in range(V):
        if df[t]:
            rr, ff = rows[off[t]:off[t + 1]].astype(np.int64), tf[off[t]:off[t + 1]].astype(np.float64)
            ms[t] = (idf[t] * ff * (k1 + 1) / (ff + k1 * (1 - b + b * lens[rr] / avgdl))).max()
    ids = np.asarray(ids, np.uint64)
    dev = search.DeviceIndex(off, rows, idf, ms, lens, ids, avgdl, posting_tf=tf)
    orc = restate.OracleIndex(off, rows, tf.astype(np.float64), idf, ms, lens, ids, avgdl)
    return dev, orc


def test_repeated_doc_ids(gpu):
    rng = np.random.default_rng(21)
    docs, ids = [], []
    for r in range(60000):
        d = {int(rng.integers(3, 200)): int(rng.integers(1, 4)) for _ in range(int(rng.integers(3, 10)))}
        if r % 500 == 0:
            d[1] = 2
        if r % 61 == 0:
            d[2] = 1
        docs.append(d)
        ids.append(1000 + r)
    # every 500th document stored again further down under the same id (same
    # terms: the same score), and a few more copies of the first one
    for r in range(0, 60000, 500):
        docs.append(dict(docs[r]))
        ids.append(ids[r])
    for _ in range(5):
        docs.append(dict(docs[0]))
        ids.append(ids[0])
    dev, orc = build(docs, ids)
    qs = [[1], [1, 2], [1, 5, 6], [2, 1, 7], [1, 1, 2]]
    for k in (1, 5, 10, 40):
        want = orc.topk(qs, k)
        for flags in (0, search.HM_FLAG_NO_SPLIT, search.HM_FLAG_SEED_ALL | search.HM_FLAG_NO_SPLIT,
                      search.HM_FLAG_EXHAUSTIVE):
            got = dev.search_lists(qs, k, flags=flags)
            check_batch(got, *want, what=f"repeated DocIds k={k} flags={flags}")
