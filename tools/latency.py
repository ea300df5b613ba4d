"""Batch-size sweep on C2 (SURVEY §8d "GPU timing"): per batch size, 20+
repeated batches after warm-up; device time (CUDA events around the device-
buffer call) and end-to-end host time through the host-buffer C ABI, both as
p50 / p99 over batches, plus "from strings" (vocabulary lookup + planning on
the host included).  Batches are different query slices every repetition.

    python tools/latency.py [reps]
"""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_25092_b200 import search, synth  # noqa: E402


def pct(x, p):
    return float(np.percentile(np.asarray(x), p))


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    c = synth.Corpus(n_records=8841823, vocab_size=1000000, min_doc_tokens=20, max_doc_tokens=60)
    q = synth.Queries(c, n_queries=60000, min_terms=3, max_terms=6)
    hx = synth.HostIndex(c)
    dev = search.DeviceIndex.from_host(hx)
    tids = hx.resolve(q.term_ranks)
    off = q.offsets.astype(np.int64)
    strs = hx.term_strings()
    vocab = {w: i for i, w in enumerate(strs)}  # the reference's CsrIndex::vocab
    rows = []
    for B in [int(x) for x in os.environ.get('HM_LAT_SIZES', '1,10,100,1000,10000,50000').split(',')]:
        k = 10
        out = dict(ids=torch.zeros(B, k, dtype=torch.int64, device="cuda"),
                   scores=torch.zeros(B, k, dtype=torch.float64, device="cuda"),
                   n=torch.zeros(B, dtype=torch.int32, device="cuda"),
                   conf=torch.zeros(B, dtype=torch.float64, device="cuda"),
                   skip=torch.zeros(B, dtype=torch.uint8, device="cuda"),
                   postings=torch.zeros(B, dtype=torch.int64, device="cuda"))
        dev_ms, e2e_ms, str_ms = [], [], []
        nrep = reps if B < 50000 else max(5, reps // 4)
        for r in range(nrep + 3):
            s0 = (r * B) % (60000 - B + 1)
            o = off[s0:s0 + B + 1] - off[s0]
            t = tids[off[s0]:off[s0 + B]]
            d_off = torch.from_numpy(o.astype(np.int32)).cuda()
            d_tid = torch.from_numpy(t.astype(np.int32)).cuda()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dev.search_batch_device(d_off, d_tid, out, k)
            e1.record()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            dev.search_batch(o.astype(np.uint32), t, k)
            t1 = time.perf_counter()
            # from strings: the query terms as text, resolved through the
            # vocabulary on the host (make_plan's lookup), then the same call
            qs = [[strs[x] for x in t[o[i]:o[i + 1]]] for i in range(B)]
            t2 = time.perf_counter()
            rt = np.fromiter((vocab.get(w, search.NO_TERM) for qq in qs for w in qq), np.uint32)
            so = np.zeros(B + 1, np.uint32)
            so[1:] = np.cumsum([len(qq) for qq in qs])
            dev.search_batch(so, rt, k)
            t3 = time.perf_counter()
            if r >= 3:
                dev_ms.append(e0.elapsed_time(e1))
                e2e_ms.append((t1 - t0) * 1e3)
                str_ms.append((t3 - t2) * 1e3)
        rows.append((B, pct(dev_ms, 50), pct(dev_ms, 99), pct(e2e_ms, 50), pct(e2e_ms, 99), pct(str_ms, 50)))
        print(f"B={B:6d}  device p50 {rows[-1][1]:8.3f} ms p99 {rows[-1][2]:8.3f} ms  ({B / rows[-1][1] * 1e3:10.0f} q/s)"
              f"  host-API p50 {rows[-1][3]:8.3f} p99 {rows[-1][4]:8.3f} ms  from strings p50 {rows[-1][5]:8.3f} ms",
              flush=True)


if __name__ == "__main__":
    main()
