#!/usr/bin/env python
"""bench.py -- batched BM25 top-k + cascade margin on B200 (BASELINE configs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline (BASELINE.json configs[1], SURVEY.md §8d "C2"): the reference
generator's MS MARCO-shaped synthetic Zipf corpus, 8,841,823 docs (V=1M,
s=1.1, 20-60 tokens), 10,000 queries of 3-6 terms, top-10, k1=1.2 b=0.75,
Margin proxy tau=0.10.  Inputs come from the native generator + builder,
bit-identical to the reference's gen_corpus / build_index at this very size
(tests/test_fullsize.py).  A "step" is one batch of the 10K queries through
the hot path (plan, seeded MaxScore pass, exhaustive tile sweep for the
queries it hands over, exact fallback; for N>1 also the NCCL all-gather of k
candidates per query and the device merge).

  value               queries/s, index and batch resident in HBM, L2 flushed
                      (256 MB write) before every timed step
  e2e                 the same through the host-buffer C ABI call
                      hm_search_batch (H2D of the batch, D2H of the results)
  e2e_from_strings    query STRINGS in host memory -> hm_vocab_resolve
                      (native threads) -> hm_search_batch, per step
  roofline            the dominant kernel of the headline step, plus
                      roofline.headline: every kernel of the step with its
                      bytes and binding roof (ncu summary in profiles/)
  configs.c3 / .c4    BASELINE configs 3 and 4 on the same GPU (N=1 only):
                      qps, p50/p99 batch latency, effective / physical
                      roofline, parity sample vs the reference's answers
                      (tests/golden/fullsize_*), CPU baseline
  cpu_baseline        the reference library (oracle/_ref) on the host cores
--impl reference times the reference's own CPU path: the index built by the
reference's gen_corpus + build_index (no framework code), MaxScore (the
fastest reference path, byte-identical output) on a rotating sample of the
same 10K queries, all host threads.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BM25 queries/sec, top-10, 8.8M docs; p50/p99 latency; HBM roofline frac"
DAY = 24 * 3600 * 1000
C2 = dict(n_records=8841823, vocab_size=1000000, min_doc_tokens=20, max_doc_tokens=60,
          n_queries=10000, min_terms=3, max_terms=6, k=10)
C4 = dict(n_records=8841823, vocab_size=1000000, min_doc_tokens=40, max_doc_tokens=80,
          n_queries=4096, min_terms=24, max_terms=32, k=100)
C1 = dict(n_records=100000, vocab_size=5000, min_doc_tokens=5, max_doc_tokens=30,
          n_queries=1000, min_terms=3, max_terms=6, k=10)
C3 = dict(n_records=5000000, vocab_size=5000, min_doc_tokens=5, max_doc_tokens=30,
          n_queries=10000, min_terms=3, max_terms=6, k=10,
          time_span_ms=int(28 * DAY * 5000000 / 4052))  # constant arrival (acceptance.cpp:101-104)
WORKLOAD = ("C2: MS MARCO-shaped synthetic Zipf corpus (reference generator, seed 42), "
            "8,841,823 docs, V=1M, s=1.1, 20-60 tokens; 10,000 queries of 3-6 terms; top-10; "
            "BM25 k1=1.2 b=0.75; Margin cascade trigger tau=0.10")
BYTES_PER_POSTING = 8  # u32 doc id + 4 B tf/impact per exhaustive posting


def env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


def pct(xs, p):
    v = sorted(xs)
    return v[min(len(v) - 1, int(round(p * (len(v) - 1))))]


# ---------------------------------------------------------------- workloads
def gen(cfg, threads=0):
    from paper_2605_25092_b200 import synth
    kw = dict(n_records=cfg["n_records"], vocab_size=cfg["vocab_size"], min_doc_tokens=cfg["min_doc_tokens"],
              max_doc_tokens=cfg["max_doc_tokens"], threads=threads)
    if "time_span_ms" in cfg:
        kw["time_span_ms"] = cfg["time_span_ms"]
    corpus = synth.Corpus(**kw)
    queries = synth.Queries(corpus, n_queries=cfg["n_queries"], min_terms=cfg["min_terms"],
                            max_terms=cfg["max_terms"])
    return corpus, queries


def exhaustive_postings(hx, q_off, tids):
    """sum over queries of the distinct known terms' df (the reference's
    exhaustive postings_touched, csr_index.cpp:100-102)."""
    df = np.diff(hx.term_offsets.astype(np.int64))
    return np.array([int(df[np.unique(t[t != 0xFFFFFFFF])].sum()) for t in
                     (tids[q_off[i]:q_off[i + 1]] for i in range(len(q_off) - 1))], np.int64)


def golden(name):
    """The reference's answers on a sample of the config's queries
    (tests/golden/fullsize_<name>, oracle/make_fullsize_golden.py)."""
    p = os.path.join(ROOT, "tests", "golden", f"fullsize_{name}")
    if not os.path.exists(p + ".json"):
        return None, None
    with open(p + ".json") as f:
        meta = json.load(f)
    return meta, dict(np.load(p + ".npz"))


def ndcg10(ids, gold):
    """eval.cpp:14-61 with one relevant doc (rel 1): 1/log2(rank+1) or 0."""
    for r, d in enumerate(ids[:10]):
        if int(d) == int(gold):
            return 1.0 / np.log2(r + 2.0)
    return 0.0


def parity_vs_golden(got, name, tau=0.10):
    """north_star tolerances on the golden sample: ids, score bits, skip,
    nDCG@10 (qrels = the gold doc)."""
    meta, g = golden(name)
    if meta is None:
        return None
    sample = [int(x) for x in g[f"{name}_sample"]]
    ids, sc, n = g[f"{name}_ids"], g[f"{name}_scores"].view(np.float64), g[f"{name}_n"]
    ids_ok = skip_ok = True
    max_rel = 0.0
    nd_o, nd_r = [], []
    for j, i in enumerate(sample):
        m = int(n[j])
        mo = int(got["n"][i])
        ids_ok &= mo == m and got["ids"][i, :m].tolist() == ids[j, :m].tolist()
        if m and mo == m:
            max_rel = max(max_rel, float(np.max(np.abs(got["scores"][i, :m] - sc[j, :m]) / np.abs(sc[j, :m]))))
        conf = (sc[j, 0] - sc[j, 1]) / max(sc[j, 0], 1e-9) if m >= 2 and sc[j, 0] > 0 else 0.0
        skip_ok &= bool(got["skip"][i]) == (conf >= tau)
        nd_o.append(ndcg10(got["ids"][i, :mo], meta["gold"][j]))
        nd_r.append(ndcg10(ids[j, :m], meta["gold"][j]))
    return dict(sample=len(sample), reference="tests/golden/fullsize_%s (reference library answers)" % name,
                ids_identical=bool(ids_ok), max_rel_score_diff=max_rel, skip_identical=bool(skip_ok),
                ndcg10_ours=float(np.mean(nd_o)), ndcg10_reference=float(np.mean(nd_r)))


# ---------------------------------------------------------------- measurement helpers
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, gpu):
        self.gpu, self.samples, self.proc = gpu, [], None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,utilization.gpu")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        self.t.join(timeout=2)

        def f(x):
            try:
                return float(x)
            except ValueError:
                return None
        load = [s for s in self.samples if len(s) >= 8 and (f(s[7]) or 0) > 50] or self.samples
        sm = [f(s[0]) for s in load if f(s[0])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in load for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": f(load[0][1]) if load and len(load[0]) > 1 else None,
                "reasons": reasons, "samples": len(load)}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_summary(name):
    """Per-kernel ncu numbers of a committed capture (tools/ncu_summary.py)."""
    p = os.path.join(ROOT, "profiles", f"ncu_{name}.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return None


class DevBatch:
    """A query batch resident on the device + result buffers."""

    def __init__(self, torch, d, q_off, tids, k):
        self.nq = len(q_off) - 1
        self.k = k
        self.off = torch.from_numpy(np.ascontiguousarray(q_off, np.uint32).view(np.int32)).to(d)
        self.tid = torch.from_numpy(np.ascontiguousarray(tids, np.uint32).view(np.int32)).to(d)
        nq = self.nq
        self.out = dict(ids=torch.zeros((nq, k), dtype=torch.int64, device=d),
                        scores=torch.zeros((nq, k), dtype=torch.float64, device=d),
                        n=torch.zeros(nq, dtype=torch.int32, device=d),
                        conf=torch.zeros(nq, dtype=torch.float64, device=d),
                        skip=torch.zeros(nq, dtype=torch.uint8, device=d),
                        postings=torch.zeros(nq, dtype=torch.int64, device=d))

    def host(self):
        r = {key: v.cpu().numpy() for key, v in self.out.items()}
        r["ids"] = r["ids"].view(np.uint64)
        return r


def time_device_steps(torch, dev, batch, steps, warmup, flush, row_lo=0, row_hi=0, timing=True, extra=0):
    """Device time (CUDA events on torch's current stream, which the batch is
    enqueued on) of `steps` batches after `warmup`, L2 flushed before each."""
    from paper_2605_25092_b200 import search
    flags = (search.HM_FLAG_TIMING if timing else 0) | extra
    for _ in range(warmup):
        dev.search_batch_device(batch.off, batch.tid, batch.out, batch.k, row_lo=row_lo, row_hi=row_hi, flags=extra)
    ms, kern = [], []
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tm = dev.search_batch_device(batch.off, batch.tid, batch.out, batch.k, row_lo=row_lo, row_hi=row_hi,
                                     flags=flags)
        e1.record()
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        if timing:
            kern.append((tm, search.last_seed()))
    return ms, kern


# ---------------------------------------------------------------- CPU baselines (oracle/_ref)
def ref_index(hx):
    from oracle import ref
    return ref.RefIndex.from_arrays(hx.term_strings(), hx.term_offsets, hx.posting_rows,
                                    hx.posting_tf.astype(np.float64), hx.idf, hx.maxscore, hx.order_key,
                                    hx.doc_lens, hx.doc_ids, hx.avgdl)


def cpu_baseline_flat(hx, queries, name, n_sample, k, maxscore_also=True):
    """The reference library's CsrIndex::bm25_topk (and _maxscore) on the box's
    host cores (hybridmem's parallel_for shape), first n_sample queries."""
    from oracle import ref
    cores = os.cpu_count() or 1
    if not ref.available():
        return dict(value=None, unit="queries/s", cores=cores, kind="reference", sample="oracle/_ref not built")
    ri = ref_index(hx)
    qs = [queries.terms(i) for i in range(n_sample)]
    r = ri.search_batch(qs, k, workers=cores)
    out = dict(value=n_sample / (r["wall_ms"] / 1e3), unit="queries/s", cores=cores, kind="reference",
               sample=f"first {n_sample} {name} queries, exhaustive CsrIndex::bm25_topk, {cores} std::threads "
                      "(hybridmem parallel_for shape)", p50_ms=float(np.median(r["lat_ms"])))
    if maxscore_also:
        rm = ri.search_batch(qs, k, workers=cores, maxscore=True)
        out["maxscore_value"] = n_sample / (rm["wall_ms"] / 1e3)
        out["maxscore_p50_ms"] = float(np.median(rm["lat_ms"]))
    return out


def cpu_baseline_temporal(hx, part, t0, queries, n_sample, k):
    """The reference's TemporalIndex::topk (partitions cut from the same flat
    index, ref_temporal_from_flat) on the host cores."""
    from oracle import ref
    cores = os.cpu_count() or 1
    if not ref.available():
        return dict(value=None, unit="queries/s", cores=cores, kind="reference", sample="oracle/_ref not built")
    rt = ref.RefTemporal.from_flat(hx.term_strings(), hx.term_offsets, hx.posting_rows,
                                   hx.posting_tf.astype(np.float64), hx.idf, hx.order_key, hx.doc_lens,
                                   hx.doc_ids, hx.avgdl, part, t0)
    qs = [queries.terms(i) for i in range(n_sample)]
    r = rt.topk_batch(qs, k, workers=cores)
    return dict(value=n_sample / (r["wall_ms"] / 1e3), unit="queries/s", cores=cores, kind="reference",
                sample=f"first {n_sample} C3 queries, TemporalIndex::topk (MaxScore per partition, UB stop), "
                       f"{cores} std::threads")


# ---------------------------------------------------------------- configs 3 and 4
def measure_c4(torch, d, flush, args, peak):
    from paper_2605_25092_b200 import search, synth
    t0 = time.time()
    corpus, queries = gen(C4)
    hx = synth.HostIndex(corpus)
    del corpus
    dev = search.DeviceIndex.from_host(hx)
    q_off = queries.offsets.astype(np.uint32)
    tids = hx.resolve(queries.term_ranks)
    post = exhaustive_postings(hx, q_off, tids)
    b = DevBatch(torch, d, q_off, tids, C4["k"])
    build_s = time.time() - t0
    ms, kern = time_device_steps(torch, dev, b, max(3, args.steps // 2), 3, flush)
    got = b.host()
    t = statistics.mean(ms)
    bytes_algo = int(post.sum()) * BYTES_PER_POSTING
    nc = ncu_summary("c4") or {}
    dram = nc.get("step_dram_bytes")
    res = dict(workload="C4: 8,841,823 docs (V=1M, 40-80 tokens), 4,096 queries of 24-32 terms, top-100",
               qps=C4["n_queries"] / (t / 1e3), p50_batch_ms=pct(ms, 0.5), p99_batch_ms=pct(ms, 0.99),
               steps=len(ms), build_s=round(build_s, 1),
               kernel_ms=dict(plan=statistics.mean(x[0][0] for x in kern),
                              seeded=statistics.mean(x[1][0] for x in kern),
                              sweep=statistics.mean(x[0][1] for x in kern),
                              exact=statistics.mean(x[0][2] for x in kern)),
               handed_to_sweep=kern[-1][1][1],
               roofline=dict(bound="hbm", unit="GB/s", peak=peak, exhaustive_postings=int(post.sum()),
                             algorithmic_bytes=bytes_algo, effective_achieved=bytes_algo / (t / 1e3) / 1e9,
                             effective_frac=bytes_algo / (t / 1e3) / 1e9 / peak,
                             physical_dram_bytes=dram,
                             physical_frac=(dram / (nc["step_ms"] / 1e3) / 1e9 / peak) if dram else None,
                             physical_source="profiles/ncu_c4.json" if dram else None),
               parity=parity_vs_golden(got, "c4"),
               postings_identical_to_reference_count=bool((got["postings"] == post).all()))
    if not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline_flat(hx, queries, "C4", args.cpu_sample_c4, C4["k"])
    del dev, hx
    torch.cuda.empty_cache()
    return res


def measure_c1(torch, d, flush, args):
    """BASELINE configs[0] (the reference's CPU-runnable case): 100K docs,
    1,000 queries, top-10 -- L2-resident and launch-bound, so qps
    and latency, no roofline; parity on the reference's answers for the first
    40 queries (tests/golden/c1_sample.json, oracle/make_golden.py)."""
    from paper_2605_25092_b200 import search, synth
    corpus, queries = gen(C1)
    hx = synth.HostIndex(corpus)
    del corpus
    dev = search.DeviceIndex.from_host(hx)
    q_off = queries.offsets.astype(np.uint32)
    tids = hx.resolve(queries.term_ranks)
    post = exhaustive_postings(hx, q_off, tids)
    b = DevBatch(torch, d, q_off, tids, C1["k"])
    ms, _ = time_device_steps(torch, dev, b, max(5, args.steps), 3, flush, timing=False)
    got = b.host()
    t = statistics.mean(ms)
    with open(os.path.join(ROOT, "tests", "golden", "c1_sample.json")) as f:
        g = json.load(f)
    ids_ok = sc_ok = skip_ok = True
    nd_o, nd_r = [], []
    for i, qg in enumerate(g["queries"]):
        m = len(qg["ids"])
        ids_ok &= int(got["n"][i]) == m and got["ids"][i, :m].tolist() == qg["ids"]
        sc_ok &= [float(x).hex() for x in got["scores"][i, :m]] == qg["scores"]
        skip_ok &= bool(got["skip"][i]) == (float.fromhex(qg["margin"]) >= 0.10)
        nd_o.append(ndcg10(got["ids"][i, :int(got["n"][i])], qg["gold"]))
        nd_r.append(ndcg10(qg["ids"], qg["gold"]))
    res = dict(workload="C1: 100,000 docs (V=5,000, 5-30 tokens), 1,000 queries of 3-6 terms, top-10",
               qps=C1["n_queries"] / (t / 1e3), p50_batch_ms=pct(ms, 0.5), p99_batch_ms=pct(ms, 0.99),
               steps=len(ms), bound="latency / L2 (SURVEY §8d: the whole index is ~11 MB)",
               exhaustive_postings=int(post.sum()),
               parity=dict(sample=len(g["queries"]), reference="tests/golden/c1_sample.json (reference library answers)",
                           ids_identical=bool(ids_ok), scores_identical=bool(sc_ok), skip_identical=bool(skip_ok),
                           ndcg10_ours=float(np.mean(nd_o)), ndcg10_reference=float(np.mean(nd_r))),
               postings_identical_to_reference_count=all(int(got["postings"][i]) == qg["postings"]
                                                         for i, qg in enumerate(g["queries"])))
    if not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline_flat(hx, queries, "C1", C1["n_queries"], C1["k"])
    del dev, hx
    torch.cuda.empty_cache()
    return res


def measure_c3(torch, d, flush, args, peak):
    from paper_2605_25092_b200 import search, synth
    t0 = time.time()
    corpus, queries = gen(C3)
    K, order, part, tmin = corpus.partition(7 * DAY)
    hx = synth.HostIndex(corpus, row_order=order)
    del corpus
    dev = search.DeviceIndex.from_host(hx)
    tix = search.TemporalIndex(dev, part)
    lo, hi = tix.window()
    q_off = queries.offsets.astype(np.uint32)
    tids = hx.resolve(queries.term_ranks)
    b = DevBatch(torch, d, q_off, tids, C3["k"])
    build_s = time.time() - t0
    ms, kern = time_device_steps(torch, dev, b, args.steps, 3, flush, row_lo=lo, row_hi=hi)
    got = b.host()
    t = statistics.mean(ms)
    post = int(got["postings"].sum())
    res = dict(workload=f"C3: 5,000,000 records, constant arrival, {K} weekly partitions; newest "
                        f"{tix.budget()} searched ({hi - lo} docs); 10,000 queries, top-10, Margin + skip",
               qps=C3["n_queries"] / (t / 1e3), p50_batch_ms=pct(ms, 0.5), p99_batch_ms=pct(ms, 0.99),
               steps=len(ms), build_s=round(build_s, 1), partitions=K, window_rows=[int(lo), int(hi)],
               roofline=dict(bound="latency / L2 (SURVEY §8d: the window is ~2.8K docs)", unit="GB/s", peak=peak,
                             window_postings=post, algorithmic_bytes=post * BYTES_PER_POSTING,
                             effective_achieved=post * BYTES_PER_POSTING / (t / 1e3) / 1e9,
                             effective_frac=post * BYTES_PER_POSTING / (t / 1e3) / 1e9 / peak),
               skip_rate=float(got["skip"].mean()),
               parity=parity_vs_golden(got, "c3"))
    if not args.no_cpu_baseline:
        res["cpu_baseline"] = cpu_baseline_temporal(hx, part, tmin, queries, args.cpu_sample_c3, C3["k"])
    del dev, hx
    torch.cuda.empty_cache()
    return res


# ---------------------------------------------------------------- reference arm
def run_reference(args):
    """The reference's own CPU path, end to end: gen_corpus + build_index by the
    reference library (no framework code on this path), then MaxScore top-10
    (CsrIndex::bm25_topk_maxscore, the fastest reference path; output
    identical to bm25_topk) over a rotating sample of the same 10K queries,
    hybridmem's parallel_for over all host threads."""
    if env_int("RANK", 0) != 0:
        return 0
    try:
        from oracle import ref
        if not ref.available():
            print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
            return 0
    except Exception as e:  # pragma: no cover
        print(json.dumps({"impl": "reference", "unavailable": str(e)[:200]}))
        return 0
    cores = os.cpu_count() or 1
    t0 = time.time()
    corpus = ref.RefCorpus(C2["n_records"], vocab_size=C2["vocab_size"], min_tok=C2["min_doc_tokens"],
                           max_tok=C2["max_doc_tokens"])
    rq = ref.RefQueries(corpus, n_queries=C2["n_queries"], min_terms=C2["min_terms"], max_terms=C2["max_terms"])
    ri = ref.RefIndex.from_corpus(corpus)
    del corpus
    build_s = time.time() - t0
    S = args.ref_sample
    times, n_done = [], 0
    for step in range(args.warmup + args.steps):
        sub = [rq.terms[(step * S + j) % C2["n_queries"]] for j in range(S)]
        r = ri.search_batch(sub, C2["k"], workers=cores, maxscore=True)
        if step >= args.warmup:
            times.append(r["wall_ms"])
            n_done += S
    tot = sum(times) / 1e3
    qps = n_done / tot
    ex = ri.search_batch([rq.terms[j] for j in range(args.ref_sample_exhaustive)], C2["k"], workers=cores)
    ex_qps = args.ref_sample_exhaustive / (ex["wall_ms"] / 1e3)
    line = dict(metric=METRIC, value=qps, unit="queries/s", n_gpus=args.gpus, steps=args.steps,
                warmup=args.warmup, ms_per_step=tot * 1e3 / args.steps, higher_is_better=True,
                scaling="strong", vs_baseline=None, dtype="f64", data="synthetic (reference gen_corpus)",
                impl="reference",
                config=dict(workload=WORKLOAD, n_docs=C2["n_records"], n_queries=C2["n_queries"], k=C2["k"],
                            sample_queries_per_step=S,
                            path="reference gen_corpus + build_index, CsrIndex::bm25_topk_maxscore",
                            reference_build_s=round(build_s, 1)),
                p50_step_ms=pct(times, 0.5), p99_step_ms=pct(times, 0.99),
                exhaustive_value=ex_qps,
                cpu_baseline=dict(value=qps, unit="queries/s", cores=cores, kind="reference",
                                  sample=f"{S} C2 queries per step (rotating through the 10K) x {args.steps} "
                                         f"steps, bm25_topk_maxscore, {cores} std::threads; exhaustive "
                                         f"bm25_topk on {args.ref_sample_exhaustive}: {ex_qps:.1f} q/s"),
                e2e=dict(value=qps, unit="queries/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0),
                gpu_launches=0)
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-sample", type=int, default=200, help="queries per reference-arm step (MaxScore)")
    ap.add_argument("--ref-sample-exhaustive", type=int, default=32)
    ap.add_argument("--cpu-sample", type=int, default=96, help="C2 queries in the cpu_baseline leg")
    ap.add_argument("--cpu-sample-c4", type=int, default=16)
    ap.add_argument("--cpu-sample-c3", type=int, default=2000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--c2-only", action="store_true", help="skip configs 3 and 4")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch
    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    # test hook: HM_SHARE_GPU=1 puts every rank on cuda:0 with the gloo
    # transport (validates the sharded path on a one-GPU box; never a bench value)
    share = os.environ.get("HM_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # the log shows the ranks / transport NCCL used
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2605_25092_b200 import search, shard, synth
    d = torch.device("cuda", local)
    peak, peak_kind = peaks()

    t0 = time.time()
    corpus, queries = gen(C2)
    if world > 1:  # every rank builds and uploads only its own shard
        sh, hx = shard.ShardedIndex.from_corpus(corpus, rank, world, device=local)
        dev = sh.dev
    else:
        hx = synth.HostIndex(corpus)
        dev = search.DeviceIndex.from_host(hx, device=local)
        sh = None
    t_build = time.time() - t0
    nq, k = C2["n_queries"], C2["k"]
    q_off = queries.offsets.astype(np.uint32)
    tids = hx.resolve(queries.term_ranks)
    post_q = exhaustive_postings(hx, q_off, tids)  # this rank's shard (the flat counts at N=1)
    fmt = dev.format()
    b = DevBatch(torch, d, q_off, tids, k)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=d)

    def step(timing, extra=0):
        flags = (search.HM_FLAG_TIMING if timing else 0) | extra
        if world > 1:  # every shard's k best seed scores (seeded pass only), all-gathered: the
            # union's k-th-score bound, then the bounded search (shard.ShardedIndex.search_device)
            bound = shard.union_bound(sh.dev_bounds(b.off, b.tid, k, b.out, extra), k, world)
            tm = dev.search_batch_device(b.off, b.tid, b.out, k, flags=flags, ext_bound=bound)
        else:
            tm = dev.search_batch_device(b.off, b.tid, b.out, k, flags=flags)
        seed = search.last_seed() if timing else None
        res = b.out
        if world > 1:
            res = shard.gather_and_merge(b.out, k, world)
        return (tm, seed), res

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    # ---------------- headline: device-resident batches
    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    step_ms, k_ms = [], []
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tm, res = step(True)
        e1.record()
        torch.cuda.synchronize()
        barrier()
        step_ms.append(e0.elapsed_time(e1))
        k_ms.append(tm)
    clk = clocks.stop()
    n_exact, n_launch = search.last_stats()
    handed = search.last_handover(nq)  # the last timed step: queries the tile sweep served
    seed_ms = statistics.mean(x[1][0] for x in k_ms)
    sweep_ms = statistics.mean(x[0][1] for x in k_ms)
    plan_ms = statistics.mean(x[0][0] for x in k_ms)
    exact_ms = statistics.mean(x[0][2] for x in k_ms)
    tot_ms = sum(step_ms)
    if world > 1:  # max over ranks
        t = torch.tensor([tot_ms], dtype=torch.float64, device=d)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        tot_ms = float(t.item())
    qps = nq * args.steps / (tot_ms / 1e3)

    # ---------------- roofline of the headline step's kernels
    bytes_sweep = int(post_q[handed == 1].sum()) * BYTES_PER_POSTING
    bytes_seed = int(post_q[handed == 0].sum()) * BYTES_PER_POSTING
    bytes_all = int(post_q.sum()) * BYTES_PER_POSTING
    nc = ncu_summary("c2_headline") or {}
    kern = nc.get("kernels", {})

    def kroof(name, ms, algo):
        # ncu names the kernel by its demangled base name ("void search_seed_kernel")
        kn = next((v for kname, v in kern.items() if name in kname), {})
        dram = kn.get("dram_bytes")
        return dict(ms=ms, algorithmic_bytes=algo, effective_achieved=algo / (ms / 1e3) / 1e9,
                    effective_frac=algo / (ms / 1e3) / 1e9 / peak, dram_bytes=dram,
                    physical_frac=(dram / (kn["ms"] / 1e3) / 1e9 / peak) if dram else None,
                    binding=kn.get("binding"), binding_frac=kn.get("binding_frac"),
                    ncu_ms=kn.get("ms"))
    heads = dict(seeded_pass=kroof("search_seed_kernel", seed_ms, bytes_seed),
                 tile_sweep=kroof("search_fast_kernel", sweep_ms, bytes_sweep))
    dom = max(heads, key=lambda x: heads[x]["ms"])
    hd = heads[dom]
    roof = dict(bound="hbm", achieved=hd["effective_achieved"], peak=peak, unit="GB/s",
                frac=hd["effective_frac"], traffic=hd["dram_bytes"],
                kernel="search_seed_kernel" if dom == "seeded_pass" else "search_fast_kernel",
                peak_kind=peak_kind, bytes_per_posting=BYTES_PER_POSTING, effective=True,
                units_per_launch=("exhaustive postings of the queries this kernel served in the headline step "
                                  "(SURVEY §8d: 8 B per posting)"),
                physical_frac=hd["physical_frac"], binding=hd["binding"], binding_frac=hd["binding_frac"],
                kernel_share_of_step=hd["ms"] / statistics.mean(step_ms),
                headline=dict(step_ms=statistics.mean(step_ms), plan_ms=plan_ms, exact_ms=exact_ms,
                              exhaustive_equivalent_bytes=bytes_all,
                              exhaustive_equivalent_frac=bytes_all / (statistics.mean(step_ms) / 1e3) / 1e9 / peak,
                              step_dram_bytes=nc.get("step_dram_bytes"),
                              physical_frac=(nc["step_dram_bytes"] / (nc["step_ms"] / 1e3) / 1e9 / peak)
                              if nc.get("step_dram_bytes") else None,
                              ncu_source="profiles/ncu_c2_headline.json" if nc else None,
                              **heads))

    # ---------------- e2e through the host-buffer C ABI (H2D + D2H timed)
    api = sh if world > 1 else dev
    api.search_batch(q_off, tids, k)  # the host path's workspace is allocated on first use
    e2e_ms = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        t1 = time.perf_counter()
        api.search_batch(q_off, tids, k)
        e2e_ms.append((time.perf_counter() - t1) * 1e3)
    e2e_tot = sum(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e_tot], dtype=torch.float64, device=d)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_tot = float(t.item())
    e2e_qps = nq * len(e2e_ms) / (e2e_tot / 1e3)
    h2d = q_off.nbytes + tids.nbytes + 4 * 4096
    d2h = nq * k * 16 + nq * (4 + 8 + 1 + 8) + 16

    # ---------------- e2e from query strings: vocabulary resolution in native threads (N > 1:
    # every rank resolves the batch against the global vocabulary its shard carries, then the
    # doc-sharded search; max over ranks)
    vocab = search.Vocab(hx.term_strings())
    qtext = [" ".join(queries.terms(i)) for i in range(nq)]
    enc = [s.encode() for s in qtext]
    text = b"".join(enc)
    toff = np.zeros(nq + 1, np.uint64)
    toff[1:] = np.cumsum([len(e) for e in enc])
    vocab.resolve_text(text, toff)
    s_ms, r_ms = [], []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        t1 = time.perf_counter()
        o2, t2 = vocab.resolve_text(text, toff)
        t_res = time.perf_counter()
        api.search_batch(o2, t2, k)
        t3 = time.perf_counter()
        s_ms.append((t3 - t1) * 1e3)
        r_ms.append((t_res - t1) * 1e3)
    assert (o2 == q_off).all() and (t2 == tids).all(), "string resolution differs from the term ids"
    s_tot = sum(s_ms)
    if world > 1:
        t = torch.tensor([s_tot], dtype=torch.float64, device=d)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        s_tot = float(t.item())
    strings = dict(value=nq * len(s_ms) / (s_tot / 1e3), unit="queries/s", p50_ms=pct(s_ms, 0.5),
                   p99_ms=pct(s_ms, 0.99), resolve_ms_p50=pct(r_ms, 0.5),
                   h2d_bytes_per_step=int(h2d), d2h_bytes_per_step=int(d2h),
                   path="query strings (host) -> hm_vocab_resolve (native threads) -> hm_search_batch"
                        + (" on every rank's shard, NCCL merge" if world > 1 else ""),
                   text_bytes=len(text))

    # ---------------- small-batch latency (N=1; device time of 1- and 10-query batches)
    small_lat = None
    if world == 1:
        small_lat = {}
        for B in (1, 10):
            ms = []
            for r in range(23):
                s0 = (r * B) % (nq - B)
                o = (q_off[s0:s0 + B + 1] - q_off[s0]).astype(np.int32)
                tt = np.ascontiguousarray(tids[q_off[s0]:q_off[s0 + B]], np.uint32).view(np.int32)
                so, st_ = torch.from_numpy(o).to(d), torch.from_numpy(tt).to(d)
                sout = {key: v[:B] for key, v in b.out.items()}
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                dev.search_batch_device(so, st_, sout, k)
                e1.record()
                torch.cuda.synchronize()
                if r >= 3:
                    ms.append(e0.elapsed_time(e1))
            small_lat[f"batch_{B}"] = dict(p50_ms=pct(ms, 0.5), p99_ms=max(ms), reps=len(ms))

    # ---------------- parity: the full batch vs the reference's answers (N > 1: the merged
    # answer of the doc-sharded search, bound exchange included, on rank 0)
    parity = None
    cpu = None
    configs = None
    if world > 1:
        _, res = step(False)
        torch.cuda.synchronize()
        if rank == 0:
            got = {key: v.cpu().numpy() for key, v in res.items()}
            got["ids"] = got["ids"].view(np.uint64)
            parity = parity_vs_golden(got, "c2")
    if rank == 0 and world == 1:
        dev.search_batch_device(b.off, b.tid, b.out, k)
        torch.cuda.synchronize()
        got = b.host()
        parity = parity_vs_golden(got, "c2")
        if parity is not None:
            parity["postings_identical_to_reference_count"] = bool((got["postings"] == post_q).all())
        if not args.no_cpu_baseline:
            try:
                cpu = cpu_baseline_flat(hx, queries, "C2", args.cpu_sample, k)
            except Exception as e:  # report, never fall back
                cpu = dict(value=None, unit="queries/s", cores=os.cpu_count(), kind="reference",
                           sample=f"failed: {str(e)[:160]}")
        if not args.c2_only:
            del dev
            torch.cuda.empty_cache()
            configs = dict(c4=measure_c4(torch, d, flush, args, peak), c3=measure_c3(torch, d, flush, args, peak),
                           c1=measure_c1(torch, d, flush, args))

    if rank == 0:
        line = dict(metric=METRIC, value=qps, unit="queries/s", n_gpus=world, steps=args.steps,
                    warmup=args.warmup, ms_per_step=tot_ms / args.steps, higher_is_better=True,
                    scaling="strong", vs_baseline=None, dtype="f32 select + f64 exact rescore",
                    data="synthetic (reference generator, bit-identical native port)",
                    config=dict(workload=WORKLOAD, n_docs=C2["n_records"], n_postings_this_rank=int(len(hx.posting_rows)),
                                n_queries=nq, k=k, exhaustive_postings_per_batch_this_rank=int(post_q.sum()),
                                parallelism=f"doc-sharded x{world} (NCCL all-gather of every shard's k best seed scores -> the "
                                            f"union's k-th-score bound; NCCL all-gather of k candidates, merge)"
                                if world > 1 else "1 GPU",
                                l2="flushed between timed steps (256 MB write)",
                                index_format=fmt, build_s=round(t_build, 1), exact_fallback_queries=n_exact,
                                path="seeded MaxScore pre-pass (search_seed_kernel) + exhaustive tile sweep "
                                     "(search_fast_kernel) for the queries it hands over",
                                seeded_pass_ms=seed_ms, tile_sweep_ms=sweep_ms,
                                handed_to_sweep=int(handed.sum())),
                    p50_step_ms=pct(step_ms, 0.5), p99_step_ms=pct(step_ms, 0.99),
                    small_batch_latency=small_lat,
                    roofline=roof, clocks=clk,
                    e2e=dict(value=e2e_qps, unit="queries/s", h2d_bytes_per_step=int(h2d),
                             d2h_bytes_per_step=int(d2h), ms_per_step=e2e_tot / len(e2e_ms),
                             p50_ms=pct(e2e_ms, 0.5), p99_ms=pct(e2e_ms, 0.99), reps=len(e2e_ms)),
                    e2e_from_strings=strings,
                    gpu_launches=n_launch * args.steps,
                    cpu_baseline=cpu, parity=parity, configs=configs)
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
