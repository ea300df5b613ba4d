"""Measurement aid: how fast would a config's batch be if every query started
with (a fraction of) its exact k-th score as the bound?  Runs the batch once,
derives each query's final k-th selection score (score * 2^-61, minus a safe
slack), feeds it back as ext_bound (the doc shards' bound input) and times
the batch under several flag sets, checking the results are identical.

    python tools/bound_potential.py c2|c4 [frac] [flags,flags,...]

flags 16 = HM_FLAG_EXHAUSTIVE (every query on the tile sweep), 1024 =
HM_FLAG_NO_BLOCK_SKIP."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_25092_b200 import search, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0  # bound = frac * exact k-th score
fsets = [int(f) for f in (sys.argv[3] if len(sys.argv) > 3 else "0,16,1040").split(",")]
cfg = {"c2": bench.C2, "c4": bench.C4}[name]
corpus, queries = bench.gen(cfg)
hx = synth.HostIndex(corpus)
del corpus
dev = search.DeviceIndex.from_host(hx)
k = cfg["k"]
b = bench.DevBatch(torch, torch.device("cuda", 0), queries.offsets.astype(np.uint32), hx.resolve(queries.term_ranks), k)


def run(ext, flags, reps=3):
    ts = []
    for r in range(reps + 1):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dev.search_batch_device(b.off, b.tid, b.out, k, ext_bound=ext, flags=flags)
        e1.record()
        torch.cuda.synchronize()
        if r:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), b.host()


t0, r0 = run(None, 0)
kth = np.where(r0["n"] >= k, r0["scores"][:, k - 1], 0.0)
ext = torch.from_numpy((kth * 2.0 ** -61 * (1 - 1e-4) * frac).astype(np.float32)).cuda()
print(f"{name}: no bound, flags 0: {t0:.2f} ms", flush=True)
for fl in fsets:
    for e, lab in ((None, "no bound"), (ext, f"bound {frac} x k-th")):
        t1, r1 = run(e, fl)
        same = all((r0[x] == r1[x]).all() for x in ("ids", "n")) and \
            (r0["scores"].view(np.uint64) == r1["scores"].view(np.uint64)).all()
        print(f"{name}: {lab}, flags {fl}: {t1:.2f} ms identical={same}", flush=True)
