"""A/B probe (development aid): one config's batch under several flag sets on
cuda:0 -- device time (CUDA events, median of reps) and bit-identity of every
output against the first flag set.

    python tools/ab.py c2|c4|c1 [nq] [reps] [flags,flags,...]
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
    C1 = dict(n_records=100000, vocab_size=5000, min_doc_tokens=5, max_doc_tokens=30, n_queries=1000, min_terms=3,
              max_terms=6, k=10)
    cfg = dict({"c1": C1, "c2": bench.C2, "c4": bench.C4}[name])
    if len(sys.argv) > 2 and int(sys.argv[2]):
        cfg["n_queries"] = int(sys.argv[2])
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    fsets = [int(f) for f in (sys.argv[4] if len(sys.argv) > 4 else "0,128,16").split(",")]
    corpus, queries = bench.gen(cfg)
    hx = synth.HostIndex(corpus)
    del corpus
    dev = search.DeviceIndex.from_host(hx)
    k = cfg["k"]
    b = bench.DevBatch(torch, torch.device("cuda", 0), queries.offsets.astype(np.uint32),
                       hx.resolve(queries.term_ranks), k)
    ref = None
    for fl in fsets:
        ts = []
        for r in range(reps + 1):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dev.search_batch_device(b.off, b.tid, b.out, k, flags=fl)
            e1.record()
            torch.cuda.synchronize()
            if r:
                ts.append(e0.elapsed_time(e1))
        tm = dev.search_batch_device(b.off, b.tid, b.out, k, flags=fl | search.HM_FLAG_TIMING)
        torch.cuda.synchronize()
        got = {n: t.cpu().numpy().copy() for n, t in b.out.items()}
        same = ""
        if ref is None:
            ref = got
        else:
            bad = [n for n in got if not np.array_equal(got[n].view(np.uint8), ref[n].view(np.uint8))]
            same = "identical" if not bad else f"DIFFER in {bad}"
        st = ""
        try:
            import ctypes
            from paper_2605_25092_b200 import _lib
            fn = _lib.load("libhm_b200.so").hm_dev_stats
            arr = (ctypes.c_ulonglong * 8)()
            fn(arr, 1)  # counts over the reps + the timing batch
            st = " stats/query=" + str([round(v / ((reps + 2) * cfg["n_queries"]), 1) for v in arr])
        except AttributeError:
            pass
        try:
            import ctypes
            from paper_2605_25092_b200 import _lib
            fn = _lib.load("libhm_b200.so").hm_seed_stats
            arr = (ctypes.c_ulonglong * 40)()
            fn(arr, 1)
            v = list(arr)
            nq_seed = max(v[0], 1)
            st += (f" seed: queries={v[0]} served={v[11]} emax_handover={v[10]} seeds/q={v[1] / nq_seed:.0f} "
                   f"seed_probes/q={v[2] / nq_seed:.0f} Eposts/q={v[3] / nq_seed:.0f} seed_probe_slots/q={v[4] / nq_seed:.0f} "
                   f"NE_probe_slots/q={v[31] / nq_seed:.0f} "
                   f"NEprobes/q={v[5] / nq_seed:.0f} cycles/q prologue={v[6] / nq_seed:.0f} seeds={v[7] / nq_seed:.0f} "
                   f"cand={v[8] / max(v[11], 1):.0f} epilogue={v[9] / max(v[11], 1):.0f} "
                   f"chunks/q={v[12] / nq_seed:.1f} insert={v[13] / nq_seed:.0f} (segments {v[15] / nq_seed:.0f}) scan={v[14] / nq_seed:.0f} "
                   f"hashed_q={v[17]} TE/hq={v[16] / max(v[17], 1):.0f} seeds/hq={v[18] / max(v[17], 1):.0f} "
                   f"short_tables_cycles/q={v[24] / nq_seed:.0f} short_postings/q={v[25] / nq_seed:.0f} "
                   f"seed_collect/q={v[26] / nq_seed:.0f} seed_a/q={v[27] / nq_seed:.0f} seed_scoring/q={v[28] / nq_seed:.0f} "
                   f"many_seeds_q={v[29]} final_kth/q={v[30] / nq_seed:.0f} "
                   f"epilogue(gather,kth,surv,rescore,sort,out)/fin=" +
                   str([round(v[i] / max(v[38], 1)) for i in range(32, 38)]))
        except AttributeError:
            pass
        print(f"{name} flags={fl:4d}: {np.median(ts):8.2f} ms  {cfg['n_queries'] / np.median(ts) * 1e3:10.0f} q/s  "
              f"timing={tm} seeded={search.last_seed()} {same}{st}", flush=True)


if __name__ == "__main__":
    main()
