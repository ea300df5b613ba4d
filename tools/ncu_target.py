"""One batch of a BASELINE config on cuda:0, for ncu (development / evidence aid).

    ncu --set full ... -k regex:'search_seed|search_fast|exact_kernel|plan_kernel' -s <n> \
        python tools/ncu_target.py c2|c4 [--exhaustive]

Builds the config's index, runs one warm-up batch (bakes the postings for
k1=1.2 b=0.75), then one measured batch with HM_FLAG_TIMING (eager launches,
no CUDA-graph replay).  A batch launches five matching kernels (plan, seeded
pass, the essential-term sweep -- empty on C2 -- the sweep, exact): -s 5 -c 5
captures the measured batch.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2605_25092_b200 import search, synth  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    cfg = {"c2": bench.C2, "c4": bench.C4}[name]
    extra = search.HM_FLAG_EXHAUSTIVE if "--exhaustive" in sys.argv else 0
    if "--flags" in sys.argv:
        extra |= int(sys.argv[sys.argv.index("--flags") + 1])
    corpus, queries = bench.gen(cfg)
    hx = synth.HostIndex(corpus)
    del corpus
    dev = search.DeviceIndex.from_host(hx)
    b = bench.DevBatch(torch, torch.device("cuda", 0), queries.offsets.astype(np.uint32),
                       hx.resolve(queries.term_ranks), cfg["k"])
    for flags in (extra, extra | search.HM_FLAG_TIMING):
        torch.cuda.synchronize()
        tm = dev.search_batch_device(b.off, b.tid, b.out, cfg["k"], flags=flags)
        torch.cuda.synchronize()
    print("timing (plan, sweep, exact) ms:", tm, "seeded (ms, handed):", search.last_seed())


if __name__ == "__main__":
    main()
