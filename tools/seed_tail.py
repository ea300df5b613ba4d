"""Development aid (scratch build with -DHM_SEED_STATS, HM_LIB_DIR): the
seeded pass's tail on C2 -- the spread of its CTAs' exit times (first ->
last, mean -> last) over three batches."""
import sys, os, ctypes
sys.path.insert(0, '/root/repo')
import numpy as np, torch, bench
from paper_2605_25092_b200 import search, synth, _lib
corpus, queries = bench.gen(bench.C2)
hx = synth.HostIndex(corpus); del corpus
dev = search.DeviceIndex.from_host(hx)
b = bench.DevBatch(torch, torch.device("cuda", 0), queries.offsets.astype(np.uint32), hx.resolve(queries.term_ranks), 10)
fn = _lib.load("libhm_b200.so").hm_seed_stats
arr = (ctypes.c_ulonglong * 40)()
for r in range(3):
    dev.search_batch_device(b.off, b.tid, b.out, 10, flags=search.HM_FLAG_TIMING)
fn(arr, 1)
for r in range(3):
    dev.search_batch_device(b.off, b.tid, b.out, 10, flags=search.HM_FLAG_TIMING)
    torch.cuda.synchronize()
    fn(arr, 1)
    v = list(arr)
    print("seeded ms", search.last_seed(), "CTAs", v[23], "first->last exit us", (v[20] - v[21]) / 1e3, "mean->last us", (v[20] - v[22] / v[23] * 1024) / 1e3)
