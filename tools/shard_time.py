"""Per-rank device time of the doc-sharded C2 batch (development aid): the G
shards of the corpus (rows [g n/G, (g+1) n/G), global statistics) built on
cuda:0; each shard's bound pass (HM_FLAG_BOUND_ONLY: its k best seed scores per
query), the k-th largest over the shards, then rank 0's
bounded search -- the compute of one rank of `bench.py --gpus G` (bound pass +
search; the NCCL all-reduce of 10K floats, the all-gather of 10K x 10
candidates and the merge come on top).  "unbounded" = the plain local top-k.

    python tools/shard_time.py [G,G,...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_25092_b200 import search, shard, synth  # noqa: E402

Gs = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,4,8").split(",")]
corpus, queries = bench.gen(bench.C2)
hx = synth.HostIndex(corpus)
del corpus
q_off = queries.offsets.astype(np.uint32)
tids = hx.resolve(queries.term_ranks)
nq, k = len(q_off) - 1, 10
b = bench.DevBatch(torch, torch.device("cuda", 0), q_off, tids, k)
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")


def timed(fn, reps=5, warm=2):
    ts = []
    for r in range(warm + reps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if r >= warm:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


base = None
for G in Gs:
    devs = []
    for g in range(G):
        d = shard.shard_host_index(hx, g, G)
        devs.append(search.DeviceIndex(d["term_offsets"], d["posting_rows"], d["idf"], d["order_key"],
                                       d["doc_lens"], d["doc_ids"], d["avgdl"], posting_tf=d["posting_tf"]))
    plain = timed(lambda: devs[0].search_batch_device(b.off, b.tid, b.out, k))
    if G == 1:
        base = plain
        print(f"G=1: {plain:.2f} ms", flush=True)
        continue
    bounds = [torch.zeros((nq, k), dtype=torch.float32, device="cuda") for _ in range(G)]
    for g in range(G):
        devs[g].search_batch_device(b.off, b.tid, b.out, k, flags=search.HM_FLAG_BOUND_ONLY, out_bound=bounds[g])
    gmax = torch.topk(torch.cat(bounds, dim=1), k, dim=1).values[:, k - 1].contiguous()
    t_bound = timed(lambda: devs[0].search_batch_device(b.off, b.tid, b.out, k, flags=search.HM_FLAG_BOUND_ONLY,
                                                        out_bound=bounds[0]))
    t_main = timed(lambda: devs[0].search_batch_device(b.off, b.tid, b.out, k, ext_bound=gmax))
    try:  # development counters of a -DHM_SEED_STATS scratch build (HM_LIB_DIR): reset
        import ctypes
        from paper_2605_25092_b200 import _lib
        _stats = _lib.load("libhm_b200.so").hm_seed_stats
        _arr = (ctypes.c_ulonglong * 40)()
        _stats(_arr, 1)
    except (AttributeError, OSError):
        _stats = None
    tm = devs[0].search_batch_device(b.off, b.tid, b.out, k, ext_bound=gmax, flags=search.HM_FLAG_TIMING)
    sd = search.last_seed()
    if _stats:
        _stats(_arr, 1)
        v = list(_arr)
        nq_s = max(v[0], 1)
        print(f"    bounded seeded pass per query: cycles prologue {v[6] / nq_s:.0f} seeds {v[7] / nq_s:.0f} "
              f"candidates {v[8] / max(v[11], 1):.0f} epilogue {v[9] / max(v[11], 1):.0f}; chunks {v[12] / nq_s:.1f}; "
              f"served {v[11]}, NE probes/q {v[5] / nq_s:.0f}", flush=True)
    tot = t_bound + t_main
    print(f"G={G}: shard {devs[0].n_docs} docs: unbounded {plain:.2f} ms ({base / plain / G * 100:.0f} % of linear); "
          f"bounds {t_bound:.2f} + bounded search {t_main:.2f} = {tot:.2f} ms ({base / tot / G * 100:.0f} % of linear) "
          f"[bounded: seeded {sd[0]:.2f} ms, {sd[1]} handed over, sweep {tm[1]:.2f} ms]",
          flush=True)
    del devs
    torch.cuda.empty_cache()
