"""CPU study (numpy, development aid; not a product path): on a sample of C2
queries, what the seeded MaxScore pass sees -- seed term, its bound L vs the
final k-th score theta, why a query is handed to the tile sweep, and what
alternative starting bounds (per-term champion lists: the C postings of each
plan term with the largest impact, scored completely) would give.

    python tools/c2_study.py [stride] [C] [c2|c4]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2605_25092_b200 import synth  # noqa: E402

stride = int(sys.argv[1]) if len(sys.argv) > 1 else 50
CH = int(sys.argv[2]) if len(sys.argv) > 2 else 64
CFG = {"c2": bench.C2, "c4": bench.C4}[sys.argv[3] if len(sys.argv) > 3 else "c2"]
t0 = time.time()
corpus, q = bench.gen(CFG)
hx = synth.HostIndex(corpus)
print("built", round(time.time() - t0, 1), flush=True)
off = hx.term_offsets.astype(np.int64)
rows = hx.posting_rows
tf = hx.posting_tf.astype(np.float32)
dl = hx.doc_lens.astype(np.float32)
idf = hx.idf
N = hx.n_docs
k1, b = 1.2, 0.75
Kd = (k1 * (1 - b + b * dl / hx.avgdl)).astype(np.float32)
tids_all = hx.resolve(q.term_ranks)
qo = q.offsets
SEEDMAX, EMAX = 131072, 131072
K = CFG["k"]
acc = np.zeros(N, np.float64)
stats = []
for qi in range(0, len(qo) - 1, stride):
    ts = tids_all[qo[qi]:qo[qi + 1]]
    ts = ts[ts != 0xFFFFFFFF]
    u, mult = np.unique(ts, return_counts=True)
    m = len(u)
    acc[:] = 0
    ms = np.zeros(m)
    df = np.array([off[t + 1] - off[t] for t in u])
    imps = []
    for j, (t, mu) in enumerate(zip(u, mult)):
        r = rows[off[t]:off[t + 1]]
        f = tf[off[t]:off[t + 1]]
        w = f * (k1 + 1) / (f + Kd[r])
        c = mu * idf[t]
        acc[r] += c * w
        ms[j] = c * w.max()
        imps.append((r, c * w))
    theta = np.partition(acc, N - K)[N - K]
    post = df.sum()
    # seed term: largest bound among df <= SEEDMAX
    cand = [j for j in range(m) if df[j] <= SEEDMAX]
    seed = max(cand, key=lambda j: ms[j]) if cand else -1
    L = 0.0
    if seed >= 0:
        sr = imps[seed][0]
        L = np.sort(acc[sr])[-K] if len(sr) >= K else 0.0
    reason = "served"
    if seed < 0:
        reason = "no_seed"
    elif not (post >= 65536 and df[seed] * m * 32 < post):
        reason = "cost"
    order = np.argsort(ms, kind="stable")

    def ess(th):
        P, ne = 0.0, set()
        for j in order:
            if P + ms[j] < th:
                P += ms[j]
                ne.add(j)
            else:
                break
        return ne, P

    ne_L, ubL = ess(L)
    ne_post = sum(df[j] for j in range(m) if j not in ne_L and j != seed)
    if reason == "served" and ne_post > EMAX:
        reason = "emax"
    ne_t, ubt = ess(theta)
    e_post_theta = sum(df[j] for j in range(m) if j not in ne_t)
    # champion lists: top-CH impacts of every term, docs scored completely
    champ = np.concatenate([r[np.argsort(-w)[:CH]] for r, w in imps])
    champ = np.unique(champ)
    Lc = np.sort(acc[champ])[-K] if len(champ) >= K else 0.0
    ne_c, _ = ess(Lc)
    e_post_c = sum(df[j] for j in range(m) if j not in ne_c)
    # candidates of the essential-term sweep at theta: rows with an essential
    # term whose essential partial + NE bound reaches theta
    accE = np.zeros(N)
    for j in range(m):
        if j not in ne_t:
            accE[imps[j][0]] += imps[j][1]
    ncand = int(((accE > 0) & (accE + ubt >= theta)).sum())
    stats.append((reason, m, post, df[seed] if seed >= 0 else -1, theta, L, Lc, e_post_theta, e_post_c, ncand,
                  len(ne_t), len(ne_c)))
    if len(stats) % 20 == 1:
        print(qi, stats[-1], flush=True)

import collections  # noqa: E402

by = collections.defaultdict(list)
for s in stats:
    by[s[0]].append(s)
for r, v in by.items():
    a = np.array([x[1:] for x in v], np.float64)
    print(f"{r:7s} n={len(v):4d}  m={a[:, 0].mean():.1f}  post={a[:, 1].mean():.3g}  seed_df={a[:, 2].mean():.3g}  "
          f"L/theta={np.mean(a[:, 4] / a[:, 3]):.3f}  Lc/theta={np.mean(a[:, 5] / a[:, 3]):.3f}  "
          f"Epost@theta={a[:, 6].mean():.3g}  Epost@Lc={a[:, 7].mean():.3g}  cand@theta={a[:, 8].mean():.3g}  "
          f"|NE|@theta={a[:, 9].mean():.2f} |NE|@Lc={a[:, 10].mean():.2f}")
