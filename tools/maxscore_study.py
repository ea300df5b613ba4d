"""CPU study (numpy, development aid): on a sample of C2 queries, with the final
k-th score known, how many postings would doc-level MaxScore stream (essential
terms) and how many (row, non-essential term) probes would it need?"""
import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_2605_25092_b200 import synth
t=time.time()
c = synth.Corpus(n_records=8841823, vocab_size=1000000, min_doc_tokens=20, max_doc_tokens=60)
q = synth.Queries(c, n_queries=10000, min_terms=3, max_terms=6)
hx = synth.HostIndex(c)
print("built", time.time()-t, flush=True)
off = hx.term_offsets.astype(np.int64); rows = hx.posting_rows; tf = hx.posting_tf.astype(np.float64)
dl = hx.doc_lens.astype(np.float64); avgdl = hx.avgdl; idf = hx.idf
N = hx.n_docs; k1, b = 1.2, 0.75
Kd = k1 * (1 - b + b * dl / avgdl)
tids = hx.resolve(q.term_ranks); qo = q.offsets
tot_post = tot_E = tot_cand = tot_cand_rows = 0; nq = 0
for qi in range(0, 10000, 100):
    ts = tids[qo[qi]:qo[qi+1]]
    u, mult = np.unique(ts, return_counts=True)
    acc = np.zeros(N); imp = {}
    ms = {}
    for t, mu in zip(u, mult):
        r = rows[off[t]:off[t+1]]; f = tf[off[t]:off[t+1]]
        w = f * (k1 + 1) / (f + Kd[r])
        imp[t] = (r, w)
        acc[r] += mu * idf[t] * w
        ms[t] = mu * idf[t] * w.max()
    theta = np.sort(acc)[-10]
    order = sorted(u, key=lambda t: ms[t])
    P = 0; NE = []
    for t in order:
        if P + ms[t] < theta: P += ms[t]; NE.append(t)
        else: break
    E = [t for t in u if t not in NE]
    accE = np.zeros(N)
    for t in E:
        r, w = imp[t]; accE[r] += dict(zip(u, mult))[t] * idf[t] * w
    ubne = sum(ms[t] for t in NE)
    cand = (accE > 0) & (accE + ubne >= theta)
    post = sum(off[t+1]-off[t] for t in u); pe = sum(off[t+1]-off[t] for t in E)
    tot_post += post; tot_E += pe; tot_cand += cand.sum() * len(NE); tot_cand_rows += cand.sum(); nq += 1
    if qi % 2000 == 0: print(qi, "post", post, "E", pe, "|NE|", len(NE), "cand", cand.sum(), flush=True)
print(f"queries {nq}: postings/q {tot_post/nq:.0f}  E postings/q {tot_E/nq:.0f} ({tot_E/tot_post:.3f})  cand rows/q {tot_cand_rows/nq:.0f}  probes/q {tot_cand/nq:.0f}")
