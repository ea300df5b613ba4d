"""Per-rank device time of the doc-sharded C2 batch (development aid): shard 0
of G (rows [0, n/G), global statistics) searched alone on cuda:0 for G = 1, 2,
4, 8 -- the compute part of each rank in `bench.py --gpus G` (the NCCL
all-gather of 10K x 10 candidates and the merge come on top).

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
# measurement of a cross-rank bound (scratch build -DHM_DEBUG_TAU_BOUND only):
# every shard starts from FRAC x the query's global k-th score
FRAC = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
corpus, queries = bench.gen(bench.C2)
hx = synth.HostIndex(corpus)
del corpus
q_off = queries.offsets.astype(np.uint32)
tids = hx.resolve(queries.term_ranks)
base = None
for G in Gs:
    d = shard.shard_host_index(hx, 0, G)
    dev = search.DeviceIndex(d["term_offsets"], d["posting_rows"], d["idf"], d["order_key"], d["doc_lens"],
                             d["doc_ids"], d["avgdl"], posting_tf=d["posting_tf"])
    b = bench.DevBatch(torch, torch.device("cuda", 0), q_off, tids, 10)
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    if FRAC and G == 1:
        bench.time_device_steps(torch, dev, b, 1, 1, flush)
        r = b.host()
        kth = np.where(r["n"] >= 10, r["scores"][:, 9], 0.0)
        gbound = torch.from_numpy(kth * 2.0 ** -61 * FRAC).cuda()
    if FRAC and G > 1:
        ms, kern = [], []
        for rep in range(8):
            flush.zero_()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            tm = dev.search_batch_device(b.off, b.tid, b.out, 10, tau=gbound, flags=search.HM_FLAG_TIMING)
            e1.record()
            torch.cuda.synchronize()
            if rep >= 3:
                ms.append(e0.elapsed_time(e1))
                kern.append((tm, search.last_seed()))
    else:
        ms, kern = bench.time_device_steps(torch, dev, b, 5, 3, flush)
    t = float(np.median(ms))
    base = base or t
    print(f"G={G}: rank-0 shard {len(d['doc_ids'])} docs, batch {t:.2f} ms (seeded {kern[-1][1][0]:.2f} ms, "
          f"handed {kern[-1][1][1]}, sweep {kern[-1][0][1]:.2f} ms) -> compute speed-up {base / t:.2f}x "
          f"({base / t / G * 100:.0f} % of linear)", flush=True)
    try:  # development counters of a -DHM_SEED_STATS scratch build (HM_LIB_DIR)
        import ctypes
        from paper_2605_25092_b200 import _lib
        arr = (ctypes.c_ulonglong * 32)()
        _lib.load("libhm_b200.so").hm_seed_stats(arr, 1)
        v = list(arr)
        nq = max(v[0], 1)
        print(f"    seeded per query: cycles prologue {v[6] / nq:.0f} seeds {v[7] / nq:.0f} "
              f"candidates {v[8] / max(v[11], 1):.0f} epilogue {v[9] / max(v[11], 1):.0f}; chunks {v[12] / nq:.1f}; "
              f"seeds {v[1] / nq:.0f}, NE probes {v[5] / nq:.0f}", flush=True)
    except (AttributeError, OSError):
        pass
    del dev
    torch.cuda.empty_cache()
