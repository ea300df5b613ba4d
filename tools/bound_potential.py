"""Measurement aid (scratch build with -DHM_DEBUG_TAU_BOUND only): how fast
would a config's sweep be if every query started with its exact k-th score as
the bound?  Runs the batch once, derives each query's final k-th selection
score (score * 2^-61, minus a safe slack), feeds it back as the starting bound
(through the tau array of the scratch build) and times both runs, checking
the results are identical."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_25092_b200 import search, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0  # bound = frac * exact k-th score
cfg = {"c2": bench.C2, "c4": bench.C4}[name]
corpus, queries = bench.gen(cfg)
hx = synth.HostIndex(corpus)
del corpus
dev = search.DeviceIndex.from_host(hx)
k = cfg["k"]
b = bench.DevBatch(torch, torch.device("cuda", 0), queries.offsets.astype(np.uint32), hx.resolve(queries.term_ranks), k)


def run(tau, reps=3):
    ts = []
    for r in range(reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dev.search_batch_device(b.off, b.tid, b.out, k, tau=tau)
        e1.record()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), b.host()


t0, r0 = run(None)
kth = np.where(r0["n"] >= k, r0["scores"][:, k - 1], 0.0)
bound = kth * 2.0 ** -61 * (1 - 1e-4) * frac
t1, r1 = run(torch.from_numpy(bound).cuda())
same = all((r0[x] == r1[x]).all() for x in ("ids", "n")) and (r0["scores"].view(np.uint64) == r1["scores"].view(np.uint64)).all()
print(f"{name}: no bound {t0:.2f} ms, exact k-th score x {frac} as the starting bound {t1:.2f} ms, identical={same}")
