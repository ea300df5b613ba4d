"""Doc-sharded multi-GPU search: one process per GPU.

The corpus rows are split into G contiguous ranges; rank g holds the sub-CSR
of rows [lo_g, hi_g) with rows renumbered from 0 and the GLOBAL statistics
(idf, avgdl, order keys) -- the same device as the reference's SharedStats
(proj/include/hybrid/csr_index.hpp:28-35) that makes partition-local scoring
bit-identical to flat scoring (src/temporal_index.cpp:136-142).  Each rank
computes an exact local top-k (ids are global DocIds), the k candidates per
query are exchanged with one all-gather (NCCL over NVLink/NVSwitch; gloo in the
CPU tests), and every rank merges the G*k candidates on device with
hm_merge_shards_device (score desc, DocId asc) and recomputes the Margin
confidence / skip decision on the merged list.  Every doc lives on exactly one
shard, so the merged list equals the single-GPU and CPU answer.
"""
import numpy as np

from . import search


def shard_bounds(n_docs, world):
    """Contiguous, balanced row ranges [lo, hi) for `world` shards."""
    return [(n_docs * g // world, n_docs * (g + 1) // world) for g in range(world)]


def shard_arrays(term_offsets, posting_rows, posting_tf, doc_lens, doc_ids, lo, hi):
    """Sub-CSR of rows [lo, hi): rows renumbered from 0, term ids unchanged."""
    rows = np.asarray(posting_rows)
    mask = (rows >= lo) & (rows < hi)
    cm = np.zeros(len(rows) + 1, np.int64)
    np.cumsum(mask, out=cm[1:])
    off = cm[np.asarray(term_offsets, np.int64)].astype(np.uint64)
    return dict(term_offsets=off, posting_rows=(rows[mask] - lo).astype(np.uint32),
                posting_tf=np.asarray(posting_tf)[mask].astype(np.uint32),
                doc_lens=np.asarray(doc_lens)[lo:hi], doc_ids=np.asarray(doc_ids)[lo:hi])


def shard_host_index(hx, rank, world):
    """Shard `rank` of a synth.HostIndex, keeping the global statistics."""
    lo, hi = shard_bounds(hx.n_docs, world)[rank]
    d = shard_arrays(hx.term_offsets, hx.posting_rows, hx.posting_tf, hx.doc_lens, hx.doc_ids,
                     lo, hi)
    d.update(idf=hx.idf, order_key=hx.order_key, avgdl=hx.avgdl)
    return d


def _allreduce(x, op, group=None):
    """In-place all-reduce of a CPU numpy array over the default group (NCCL
    needs device tensors: the array travels through this rank's GPU)."""
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(x)
    if dist.get_backend(group) == "nccl":
        d = t.cuda()
        dist.all_reduce(d, op=op, group=group)
        t.copy_(d.cpu())
    else:
        dist.all_reduce(t, op=op, group=group)
    return x


def build_shard(corpus, rank, world, group=None, k1=1.2, b=0.75, threads=0):
    """Rank `rank`'s shard built by this rank alone (no rank builds the whole
    index): its document frequencies and length sum are summed over the ranks
    (all-reduce), the shard's postings are built with the resulting GLOBAL
    idf / avgdl, and the order keys are the global per-term maxima (a MAX
    all-reduce of the shards' maxscores) -- bit-identical to shard_host_index
    of the flat build (tests/test_multi.py)."""
    import torch.distributed as dist
    from . import synth
    n = corpus.n
    lo, hi = shard_bounds(n, world)[rank]
    df, ls = synth.shard_counts(corpus, lo, hi, threads)
    if world > 1:
        df = _allreduce(df.view(np.int64), dist.ReduceOp.SUM, group).view(np.uint64)
        ls = int(_allreduce(np.array([ls], np.int64), dist.ReduceOp.SUM, group)[0])
    hx = synth.HostIndex.shard(corpus, lo, hi, df, n, ls, k1=k1, b=b, threads=threads)
    ms = np.ascontiguousarray(hx.maxscore, np.float64)
    if world > 1:
        ms = _allreduce(ms, dist.ReduceOp.MAX, group)
    hx.maxscore = ms
    hx.order_key = ms.copy()
    hx.row_range = (lo, hi)
    return hx


def gather_and_merge(local, k, world, group=None, tau=None, tau_default=0.10,
                     epsilon_guard=1e-9):
    """All-gather per-shard top-k (torch tensors on this rank's device) and merge.

    local: dict(ids[nq,k] int64, scores[nq,k] f64, n[nq] int32) on the device.
    Returns the merged dict (ids, scores, n, conf, skip) on the device.
    """
    import torch
    import torch.distributed as dist
    nq = local["n"].shape[0]
    dev = local["n"].device
    if world > 1:
        g_ids = torch.empty((world, nq, k), dtype=torch.int64, device=dev)
        g_sc = torch.empty((world, nq, k), dtype=torch.float64, device=dev)
        g_n = torch.empty((world, nq), dtype=torch.int32, device=dev)
        if dist.get_backend(group) == "gloo":  # CPU transport (tests: ranks sharing one GPU)
            for g, x in ((g_ids, local["ids"]), (g_sc, local["scores"]), (g_n, local["n"])):
                parts = [torch.empty_like(x, device="cpu") for _ in range(world)]
                dist.all_gather(parts, x.contiguous().cpu(), group=group)
                g.copy_(torch.stack(parts))
        else:  # NCCL over NVLink: one all-gather per field, device to device
            dist.all_gather_into_tensor(g_ids, local["ids"].contiguous(), group=group)
            dist.all_gather_into_tensor(g_sc, local["scores"].contiguous(), group=group)
            dist.all_gather_into_tensor(g_n, local["n"].contiguous(), group=group)
    else:
        g_ids, g_sc, g_n = local["ids"][None], local["scores"][None], local["n"][None]
    out = dict(ids=torch.zeros((nq, k), dtype=torch.int64, device=dev),
               scores=torch.zeros((nq, k), dtype=torch.float64, device=dev),
               n=torch.zeros(nq, dtype=torch.int32, device=dev),
               conf=torch.zeros(nq, dtype=torch.float64, device=dev),
               skip=torch.zeros(nq, dtype=torch.uint8, device=dev))
    search.merge_shards_device(g_ids.contiguous(), g_sc.contiguous(), g_n.contiguous(), out, k,
                               tau=tau, tau_default=tau_default, epsilon_guard=epsilon_guard)
    return out


def union_bound(seeds, k, world, group=None):
    """All-gather every rank's k best seed scores per query (float32[nq, k])
    and take the k-th largest of the world * k values: a k-th score of real
    documents of the whole corpus, hence a lower bound on its k-th score."""
    import torch
    import torch.distributed as dist
    nq = seeds.shape[0]
    if world <= 1:
        allv = seeds
    else:
        g = torch.empty((world, nq, k), dtype=seeds.dtype, device=seeds.device)
        if dist.get_backend(group) == "gloo":
            parts = [torch.empty((nq, k), dtype=seeds.dtype) for _ in range(world)]
            dist.all_gather(parts, seeds.cpu(), group=group)
            g.copy_(torch.stack(parts))
        else:
            dist.all_gather_into_tensor(g, seeds.contiguous(), group=group)
        allv = g.permute(1, 0, 2).reshape(nq, world * k)
    return torch.topk(allv, k, dim=1).values[:, k - 1].contiguous()


def allreduce_postings(local_post, world, group=None):
    """postings_touched of the merged result: the shards' counts summed."""
    import torch.distributed as dist
    tot = local_post.clone()
    if world > 1:
        if dist.get_backend(group) == "gloo":
            t = tot.cpu()
            dist.all_reduce(t, group=group)
            tot.copy_(t)
        else:
            dist.all_reduce(tot, group=group)
    return tot


def merge_host(shard_ids, shard_scores, shard_n, k, tau_default=0.10, eps=1e-9):
    """Host restatement of the merge (used by the gloo CPU tests of the exchange
    protocol; the product merge is merge_kernel on the device)."""
    G, nq = shard_n.shape
    ids = np.zeros((nq, k), np.uint64)
    sc = np.zeros((nq, k), np.float64)
    n = np.zeros(nq, np.uint32)
    conf = np.zeros(nq)
    for q in range(nq):
        cand = [(float(shard_scores[g, q, r]), int(shard_ids[g, q, r]))
                for g in range(G) for r in range(int(shard_n[g, q]))]
        cand.sort(key=lambda x: (-x[0], x[1]))
        cand = [c for c in cand if c[0] > 0][:k]
        n[q] = len(cand)
        for r, (s, d) in enumerate(cand):
            ids[q, r] = d
            sc[q, r] = s
        conf[q] = search.margin(sc[q, :n[q]], eps) if n[q] else 0.0
    return ids, sc, n, conf, (conf >= tau_default).astype(np.uint8)


class ShardedIndex:
    """This rank's shard on its GPU plus the exchange; the public multi-GPU API."""

    def __init__(self, hx, rank, world, device=0):
        d = shard_host_index(hx, rank, world)
        self.rank, self.world = rank, world
        self.dev = search.DeviceIndex(d["term_offsets"], d["posting_rows"], d["idf"],
                                      d["order_key"], d["doc_lens"], d["doc_ids"], d["avgdl"],
                                      posting_tf=d["posting_tf"], device=device)

    @classmethod
    def from_corpus(cls, corpus, rank, world, device=0, group=None, threads=0):
        """Each rank builds and uploads only its own shard (build_shard).
        -> (ShardedIndex, the shard's HostIndex: term ids / resolve are global)."""
        hx = build_shard(corpus, rank, world, group=group, threads=threads)
        self = cls.__new__(cls)
        self.rank, self.world = rank, world
        self.dev = search.DeviceIndex(hx.term_offsets, hx.posting_rows, hx.idf, hx.order_key, hx.doc_lens,
                                      hx.doc_ids, hx.avgdl, posting_tf=hx.posting_tf, device=device)
        return self, hx

    def search_device(self, q_off, q_tid, k, local_out, **kw):
        """Device-resident batch: shard bounds, local top-k, all-gather, merge.

        With world > 1 every rank first runs the seeded pass's bound only
        (HM_FLAG_BOUND_ONLY: a lower bound on each query's k-th score in its
        shard), the bounds are all-reduced with MAX -- a lower bound on the
        k-th score of the whole corpus -- and the search proper prunes against
        it: a shard's list keeps only documents that can be in the global
        top-k, so the merge of the lists is the exact answer while each shard
        works against the global threshold instead of its own (weaker) one.
        The merged skip decision uses the caller's per-query tau /
        tau_default / epsilon_guard; postings_touched is summed over the
        shards (every posting lives on exactly one shard)."""
        if self.world > 1 and 0 < k <= 256:
            flags = kw.pop("flags", 0)
            nq = q_off.numel() - 1
            seeds = self.dev_bounds(q_off, q_tid, k, local_out, flags,
                                    **{x: v for x, v in kw.items() if x not in ("tau",)})
            bound = union_bound(seeds, k, self.world)
            self.dev.search_batch_device(q_off, q_tid, local_out, k, flags=flags, ext_bound=bound, **kw)
        else:
            self.dev.search_batch_device(q_off, q_tid, local_out, k, **kw)
        out = gather_and_merge(local_out, k, self.world, tau=kw.get("tau"),
                               tau_default=kw.get("tau_default", 0.10),
                               epsilon_guard=kw.get("epsilon_guard", 1e-9))
        out["postings"] = allreduce_postings(local_out["postings"], self.world)
        return out

    def dev_bounds(self, q_off, q_tid, k, scratch_out, flags=0, **kw):
        """This shard's bound pass: float32[nq, k], the k best complete seed
        scores of every query (HM_FLAG_BOUND_ONLY)."""
        import torch
        nq = q_off.numel() - 1
        seeds = torch.zeros((nq, k), dtype=torch.float32, device=q_off.device)
        self.dev.search_batch_device(q_off, q_tid, scratch_out, k, flags=flags | search.HM_FLAG_BOUND_ONLY,
                                     out_bound=seeds, **kw)
        return seeds

    def search_batch(self, q_off, q_tid, k, **kw):
        """Host buffers in, host results out (H2D, search, all-gather, merge, D2H)."""
        import torch
        dev = torch.device("cuda", self.dev.device)
        d_off = torch.from_numpy(np.ascontiguousarray(q_off, np.uint32).view(np.int32)).to(dev)
        d_tid = torch.from_numpy(np.ascontiguousarray(q_tid, np.uint32).view(np.int32)).to(dev)
        nq = len(q_off) - 1
        loc = dict(ids=torch.zeros((nq, k), dtype=torch.int64, device=dev),
                   scores=torch.zeros((nq, k), dtype=torch.float64, device=dev),
                   n=torch.zeros(nq, dtype=torch.int32, device=dev),
                   conf=torch.zeros(nq, dtype=torch.float64, device=dev),
                   skip=torch.zeros(nq, dtype=torch.uint8, device=dev),
                   postings=torch.zeros(nq, dtype=torch.int64, device=dev))
        out = self.search_device(d_off, d_tid, k, loc, **kw)
        return {key: v.cpu().numpy() for key, v in out.items()}
