"""Edge cases of the seeded pass's essential-score hash table
(csrc/kernels/search_seed.cu, stage 3): table overflow (hand-over to the
sweep with the seeds' bound), no essential terms beyond the seed term (stage
skipped), fewer seeds than k (no fixed-point scale: hand-over), rows holding
both the seed term and essential terms (flagged, never admitted twice), row
windows cutting the chunks.  HM_FLAG_SEED_ALL makes the pass try every query;
every answer must equal the C restatement of the reference bit for bit."""
import numpy as np
import pytest

from _util import check_batch, restate, search

pytestmark = pytest.mark.gpu


def build(docs):
    """docs: list of per-doc {term: tf}; rows = docs in order, DocId = 7 * row + 3."""
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
    ids = np.arange(N, dtype=np.uint64) * 7 + 3
    dev = search.DeviceIndex(off, rows, idf, ms, lens, ids, avgdl, posting_tf=tf)
    orc = restate.OracleIndex(off, rows, tf.astype(np.float64), idf, ms, lens, ids, avgdl)
    return dev, orc


def run(dev, orc, queries, k, row_lo=0, row_hi=0):
    """Both ways a small batch runs: whole queries (HM_FLAG_NO_SPLIT) and row
    slabs of each query (the default for small batches, merged afterwards)."""
    ids, sc, n, post = orc.topk(queries, k, row_lo=row_lo, row_hi=row_hi or dev.n_docs)
    for extra in (search.HM_FLAG_NO_SPLIT, 0):
        got = dev.search_lists(queries, k, flags=search.HM_FLAG_SEED_ALL | extra, row_lo=row_lo, row_hi=row_hi)
        check_batch(got, ids, sc, n, post, what=f"seed hash k={k} window=({row_lo},{row_hi}) flags={extra}")


def test_hash_overflow_and_seed_rows(gpu):
    """200,000 docs (13 tiles): term 1 is in 150,000 of them -- too many to be
    the seed term (at most 131,072 postings) -- and weighted 20x in the query,
    so it is essential next to the seed term 2; with ~12,000 of its postings
    per tile a single tile overflows the 4,096-slot table: the query goes to
    the sweep with the seeds' bound.  Seed rows that also hold term 1 are
    flagged in the table."""
    rng = np.random.default_rng(5)
    docs = []
    for r in range(200000):
        d = {0: 1}  # everywhere: non-essential
        if r % 4 != 0:
            d[1] = int(rng.integers(1, 4))
        if r % 2000 == 0:
            d[2] = 1  # 100 postings: the seed term
        for _ in range(int(rng.integers(2, 8))):
            d[3 + int(rng.integers(0, 400))] = 1
        docs.append(d)
    dev, orc = build(docs)
    heavy = [2] + [1] * 20 + [0]
    qs = [heavy, [2, 1, 0], [2, 0], heavy + [7], [1, 2]]
    for k in (1, 10, 100):
        run(dev, orc, qs, k)
    # the overflow really happened: the heavy queries went to the sweep
    dev.search_lists(qs, 10, flags=search.HM_FLAG_SEED_ALL | search.HM_FLAG_NO_SPLIT | search.HM_FLAG_TIMING)
    handed = search.last_handover(len(qs))
    assert handed[0] and handed[3], handed


def test_few_seeds_and_no_essential_terms(gpu):
    """A seed term with fewer postings than k (no bound: the query is handed
    over) and queries whose only essential term is the seed term (the hash
    stage is skipped)."""
    rng = np.random.default_rng(9)
    docs = []
    for r in range(40000):
        d = {int(rng.integers(10, 60)): int(rng.integers(1, 3)) for _ in range(int(rng.integers(3, 12)))}
        if r % 5000 == 0:
            d[1] = 2  # 8 postings < k = 10
        if r % 37 == 0:
            d[2] = 1  # rare-ish
        docs.append(d)
    dev, orc = build(docs)
    qs = [[1, 10, 11], [1], [2, 10], [2, 1, 10, 11, 12], [2, 2, 10]]
    for k in (1, 10, 50):
        run(dev, orc, qs, k)


def test_windows_cut_chunks(gpu):
    """Row windows starting and ending inside tiles: the chunks' segments
    are clipped to the window."""
    rng = np.random.default_rng(13)
    docs = []
    for r in range(70000):
        d = {int(rng.integers(20, 300)): int(rng.integers(1, 4)) for _ in range(int(rng.integers(3, 15)))}
        if r % 3 == 0:
            d[1] = 1
        if r % 97 == 0:
            d[2] = int(rng.integers(1, 3))
        docs.append(d)
    dev, orc = build(docs)
    qs = [[2, 1, 20], [2, 1], [2, 21, 22, 1], [1, 2, 25, 26, 27, 28]]
    for lo, hi in [(0, 0), (16000, 50000), (123, 69999), (40000, 40100)]:
        run(dev, orc, qs, 10, row_lo=lo, row_hi=hi)
