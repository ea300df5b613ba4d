"""Small batches through every kernel path, for compute-sanitizer
(memcheck / racecheck / initcheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize.py

Runs C1-shaped searches (default path, HM_FLAG_SEED_ALL, HM_FLAG_EXHAUSTIVE,
HM_FLAG_FORCE_EXACT, a row window, k=100, other Bm25Params) and checks them
against the C restatement of the reference (oracle/)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import restate
from paper_2605_25092_b200 import search, synth


def main():
    c = synth.Corpus(n_records=20000, vocab_size=2000)
    q = synth.Queries(c, n_queries=96)
    hx = synth.HostIndex(c)
    dev = search.DeviceIndex.from_host(hx)
    orc = restate.OracleIndex.from_host(hx)
    tids = [hx.resolve(q.term_ranks[q.offsets[i]:q.offsets[i + 1]]) for i in range(len(q))]
    cases = [dict(), dict(flags=search.HM_FLAG_SEED_ALL), dict(flags=search.HM_FLAG_EXHAUSTIVE),
             dict(flags=search.HM_FLAG_FORCE_EXACT), dict(row_lo=3000, row_hi=17000),
             dict(row_lo=3000, row_hi=17000, flags=search.HM_FLAG_SEED_ALL), dict(k=100),
             dict(k1=0.9, b=0.4, flags=search.HM_FLAG_SEED_ALL), dict(flags=search.HM_FLAG_NE_ALL),
             dict(k=300), dict(flags=search.HM_FLAG_SEED_ALL | search.HM_FLAG_NO_SPLIT)]
    for kw in cases:
        k = kw.pop("k", 10)
        got = dev.search_lists(tids, k, **kw)
        okw = {x: kw[x] for x in ("k1", "b", "row_lo", "row_hi") if x in kw}
        ids, sc, n, _ = orc.topk(tids, k, **okw)
        assert (got["n"] == n).all(), kw
        for i in range(len(tids)):
            assert (got["ids"][i, :n[i]] == ids[i, :n[i]]).all(), (kw, i)
            assert (got["scores"][i, :n[i]].view(np.uint64) == sc[i, :n[i]].view(np.uint64)).all(), (kw, i)
    # a larger index: long seed terms enumerated tile by tile, windows cutting tiles
    c2 = synth.Corpus(n_records=200000, vocab_size=5000)
    q2 = synth.Queries(c2, n_queries=64)
    hx2 = synth.HostIndex(c2)
    dev2 = search.DeviceIndex.from_host(hx2)
    orc2 = restate.OracleIndex.from_host(hx2)
    t2 = [hx2.resolve(q2.term_ranks[q2.offsets[i]:q2.offsets[i + 1]]) for i in range(len(q2))]
    for lo, hi in ((0, 0), (12345, 190001), (70000, 70000 + 40000)):
        got = dev2.search_lists(t2, 10, row_lo=lo, row_hi=hi, flags=search.HM_FLAG_SEED_ALL)
        ids, sc, n, _ = orc2.topk(t2, 10, row_lo=lo, row_hi=hi or hx2.n_docs)
        assert (got["n"] == n).all()
        for i in range(len(t2)):
            assert (got["ids"][i, :n[i]] == ids[i, :n[i]]).all(), (lo, hi, i)
    # doc-sharded search behind the C ABI: three shards on this device, the
    # gather + merge kernel reading their lists (peer memory on a multi-GPU box)
    sh = search.ShardedDeviceIndex.from_host(hx2, [0, 0, 0])
    off = np.zeros(len(t2) + 1, np.uint32)
    off[1:] = np.cumsum([len(t) for t in t2])
    for k in (10, 300):
        got = sh.search_batch(off, np.concatenate(t2).astype(np.uint32), k)
        ids, sc, n, _ = orc2.topk(t2, k)
        assert (got["n"] == n).all()
        for i in range(len(t2)):
            assert (got["ids"][i, :n[i]] == ids[i, :n[i]]).all(), ("sharded", k, i)
    print("sanitize cases ok:", len(cases) + 5)


if __name__ == "__main__":
    main()
