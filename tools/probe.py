"""Quick perf probe (development aid): time one config's batch on the GPU."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_25092_b200 import search, synth

def main(n=8841823, V=1000000, lo=20, hi=60, nq=10000, mint=3, maxt=6, k=10, reps=3, temporal=False):
    t = time.time()
    kw = dict(n_records=n, vocab_size=V, min_doc_tokens=lo, max_doc_tokens=hi)
    if temporal:  # C3: constant arrival rate (acceptance.cpp:101-104), weekly partitions
        kw["time_span_ms"] = int(28 * 86400000 * n / 4052)
    c = synth.Corpus(**kw)
    q = synth.Queries(c, n_queries=nq, min_terms=mint, max_terms=maxt)
    row_lo = row_hi = 0
    if temporal:
        K, order, part, _ = c.partition(7 * 86400000)
        hx = synth.HostIndex(c, row_order=order)
        tix = search.TemporalIndex(None, part)
        row_lo, row_hi = tix.window()
        print(f"temporal: {K} partitions, budget {tix.budget()}, window rows [{row_lo},{row_hi}) = {row_hi - row_lo} docs")
    else:
        hx = synth.HostIndex(c)
    print(f"gen+build {time.time()-t:.1f}s P={len(hx.posting_rows)}", flush=True)
    t = time.time(); dev = search.DeviceIndex.from_host(hx); print(f"upload {time.time()-t:.1f}s fmt={dev.format()} bytes={dev.device_bytes/1e9:.2f}GB", flush=True)
    tids = hx.resolve(q.term_ranks)
    off = q.offsets.astype(np.uint32)
    df = np.diff(hx.term_offsets.astype(np.int64))
    post = sum(int(df[np.unique(tids[off[i]:off[i+1]])].sum()) for i in range(nq))  # flat (whole-corpus) postings
    dq_off = torch.from_numpy(off.astype(np.int32)).cuda(); dq_tid = torch.from_numpy(tids.astype(np.int32)).cuda()
    out = dict(ids=torch.zeros(nq, k, dtype=torch.int64, device='cuda'), scores=torch.zeros(nq, k, dtype=torch.float64, device='cuda'),
               n=torch.zeros(nq, dtype=torch.int32, device='cuda'), conf=torch.zeros(nq, dtype=torch.float64, device='cuda'),
               skip=torch.zeros(nq, dtype=torch.uint8, device='cuda'), postings=torch.zeros(nq, dtype=torch.int64, device='cuda'))
    for r in range(reps + 1):
        torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); dev.search_batch_device(dq_off, dq_tid, out, k, flags=int(os.environ.get('HM_PROBE_FLAGS', '0')), row_lo=row_lo, row_hi=row_hi); e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        wpost = int(out["postings"].sum().item())  # postings inside the window
        if r == reps:
            fl = int(os.environ.get('HM_PROBE_FLAGS', '0')) | search.HM_FLAG_TIMING
            dev.search_batch_device(dq_off, dq_tid, out, k, flags=fl, row_lo=row_lo, row_hi=row_hi)
            print("timing (plan, exhaustive, exact) ms:", search.last_timing(), " seeded (ms, handed over):", search.last_seed())
        print(f"rep {r}: {ms:.2f} ms  {nq/ms*1e3:.0f} qps  eff {wpost*8/ms/1e6:.0f} GB/s (8B/posting)  phys {wpost*4/ms/1e6:.0f} GB/s", flush=True)
    t = time.time(); r = dev.search_batch(off, tids, k, row_lo=row_lo, row_hi=row_hi); print(f"host api {time.time()-t:.3f}s n_exact={r['n_exact']}")

if __name__ == "__main__":
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    nq = int(sys.argv[2]) if len(sys.argv) > 2 else None
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    if cfg == "c1": main(100000, 5000, 5, 30, nq or 1000, reps=reps)
    elif cfg == "c4": main(8841823, 1000000, 40, 80, nq or 4096, 24, 32, 100, reps=reps)
    elif cfg == "c3": main(5000000, 5000, 5, 30, nq or 10000, reps=reps, temporal=True)
    else: main(nq=nq or 10000, reps=reps)
