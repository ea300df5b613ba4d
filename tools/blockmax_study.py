"""CPU study (numpy, development aid; not a product path): how much of a C2
query's postings a block-max skip would leave to stream -- per row block
(unit of U rows) the upper bound sum_t c_t * max impact of t in the block;
blocks whose bound is below the threshold (the final k-th score theta, an
optimistic stand-in for any running bound) need no streaming and no scan.

    python tools/blockmax_study.py [stride] [U,U,...]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_25092_b200 import synth  # noqa: E402

stride = int(sys.argv[1]) if len(sys.argv) > 1 else 50
Us = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1024,2048,16384").split(",")]
corpus, q = bench.gen(bench.C2)
hx = synth.HostIndex(corpus)
off = hx.term_offsets.astype(np.int64)
rows = hx.posting_rows
tf = hx.posting_tf.astype(np.float32)
dl = hx.doc_lens.astype(np.float32)
N = hx.n_docs
k1, b = 1.2, 0.75
Kd = (k1 * (1 - b + b * dl / hx.avgdl)).astype(np.float32)
tids_all = hx.resolve(q.term_ranks)
qo = q.offsets
K = 10
acc = np.zeros(N, np.float64)
res = {U: [] for U in Us}
for qi in range(0, len(qo) - 1, stride):
    ts = tids_all[qo[qi]:qo[qi + 1]]
    ts = ts[ts != 0xFFFFFFFF]
    u, mult = np.unique(ts, return_counts=True)
    acc[:] = 0
    imps = []
    for t, mu in zip(u, mult):
        r = rows[off[t]:off[t + 1]]
        f = tf[off[t]:off[t + 1]]
        w = mu * hx.idf[t] * f * (k1 + 1) / (f + Kd[r])
        acc[r] += w
        imps.append((r, w))
    SHORT = 32 * ((N + 16383) // 16384)  # short terms: df <= 32 x tiles (no per-unit table)
    GLOBAL_SHORT = os.environ.get("GLOBAL_SHORT") == "1"
    PRESENCE_SHORT = os.environ.get("PRESENCE_SHORT") == "1"
    theta = np.partition(acc, N - K)[N - K]
    post = sum(len(r) for r, _ in imps)
    for U in Us:
        nb = (N + U - 1) // U
        ub = np.zeros(nb)
        cnt = []
        for r, w in imps:
            blk = r // U
            mx = np.zeros(nb)
            if GLOBAL_SHORT and len(r) <= SHORT:
                mx[:] = w.max()
            elif PRESENCE_SHORT and len(r) <= SHORT:
                mx[blk] = w.max()
            else:
                np.maximum.at(mx, blk, w)
            ub += mx
            cnt.append(np.bincount(blk, minlength=nb))
        r3 = []
        for fr in (1.0, 0.97, 0.9):
            live = ub * (1 + 1e-6) >= fr * theta
            kept = sum(c[live].sum() for c in cnt)
            r3 += [live.mean(), kept / post]
        res[U].append(tuple(r3) + (post,))
for U in Us:
    a = np.array(res[U])
    for name, sel in (("all", a[:, -1] >= 0), ("post>4M", a[:, -1] > 4e6)):
        b_ = a[sel]
        w = b_[:, -1] / b_[:, -1].sum()
        print(f"U={U:6d} {name:8s} n={len(b_)}: posting-weighted (live blocks, postings left) at theta "
              f"({np.sum(w * b_[:, 0]):.3f}, {np.sum(w * b_[:, 1]):.3f}), 0.97 theta ({np.sum(w * b_[:, 2]):.3f}, "
              f"{np.sum(w * b_[:, 3]):.3f}), 0.9 theta ({np.sum(w * b_[:, 4]):.3f}, {np.sum(w * b_[:, 5]):.3f})")
