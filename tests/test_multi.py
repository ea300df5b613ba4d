"""Doc-sharded multi-GPU path.

CPU (gloo, world_size 2): shard splitting with global statistics, the
all-gather of k candidates per query, and the merge restate the unsharded
answer exactly (scores per shard come from the oracle restatement, since the
CPU box has no GPU).  GPU: G simulated shards on one device, device merge
(hm_merge_shards_device) == unsharded GPU results.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from _util import check_batch, restate, search, synth, synth_setup
from paper_2605_25092_b200 import shard

K = 10


def _worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    _, _, hx, tids = synth_setup(30000, 5000, 5, 30, 64)
    d = shard.shard_host_index(hx, rank, world)
    orc = restate.OracleIndex(d["term_offsets"], d["posting_rows"],
                              d["posting_tf"].astype(np.float64), d["idf"], d["order_key"],
                              d["doc_lens"], d["doc_ids"], d["avgdl"])
    ids, sc, n, post = orc.topk(tids, K)
    g_ids = [torch.zeros((len(tids), K), dtype=torch.int64) for _ in range(world)]
    g_sc = [torch.zeros((len(tids), K), dtype=torch.float64) for _ in range(world)]
    g_n = [torch.zeros(len(tids), dtype=torch.int32) for _ in range(world)]
    dist.all_gather(g_ids, torch.from_numpy(ids.view(np.int64)))
    dist.all_gather(g_sc, torch.from_numpy(sc))
    dist.all_gather(g_n, torch.from_numpy(n.astype(np.int32)))
    mi, ms, mn, mc, mk = shard.merge_host(torch.stack(g_ids).numpy().view(np.uint64),
                                          torch.stack(g_sc).numpy(), torch.stack(g_n).numpy(), K)
    p = torch.tensor([int(post.sum())], dtype=torch.int64)
    dist.all_reduce(p)
    if rank == 0:
        out_q.put((mi, ms, mn, mc, mk, int(p.item())))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_bounds_cover_rows():
    for n, w in [(10, 3), (8841823, 8), (1, 2), (0, 4)]:
        b = shard.shard_bounds(n, w)
        assert b[0][0] == 0 and b[-1][1] == n
        assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))


def test_shard_arrays_partition_postings():
    _, _, hx, _ = synth_setup(5000, 500, 5, 30, 4)
    parts = [shard.shard_host_index(hx, g, 3) for g in range(3)]
    assert sum(len(p["posting_rows"]) for p in parts) == len(hx.posting_rows)
    for p in parts:
        off = p["term_offsets"].astype(np.int64)
        assert off[0] == 0 and off[-1] == len(p["posting_rows"])
        for t in range(0, len(off) - 1, 37):
            r = p["posting_rows"][off[t]:off[t + 1]]
            assert (np.diff(r.astype(np.int64)) > 0).all() and (r < len(p["doc_ids"])).all()


def test_gloo_world2_shard_exchange_merge_equals_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    mi, ms, mn, mc, mk, post = res
    _, _, hx, tids = synth_setup(30000, 5000, 5, 30, 64)
    ids, sc, n, p_all = restate.OracleIndex.from_host(hx).topk(tids, K)
    assert (mn == n).all() and post == int(p_all.sum())
    for i in range(len(n)):
        assert (mi[i, :n[i]] == ids[i, :n[i]]).all()
        assert (ms[i, :n[i]].view(np.uint64) == sc[i, :n[i]].view(np.uint64)).all()
        assert mc[i] == restate.margin(sc[i, :n[i]])


def _build_worker(rank, world, port, out_q):
    """A rank builds only its own shard (shard.build_shard: df / length sums
    and maxscores all-reduced over gloo)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    corpus = synth.Corpus(n_records=20000, vocab_size=3000, min_doc_tokens=5, max_doc_tokens=30)
    hx = shard.build_shard(corpus, rank, world, threads=2)
    out_q.put((rank, dict(term_offsets=hx.term_offsets, posting_rows=hx.posting_rows, posting_tf=hx.posting_tf,
                          idf=hx.idf, order_key=hx.order_key, doc_lens=hx.doc_lens, doc_ids=hx.doc_ids,
                          avgdl=hx.avgdl, rank_to_tid=hx.rank_to_tid)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_per_rank_shard_build_equals_flat_shard(world):
    """Each rank builds only its rows, with the global statistics from
    all-reduces: identical to slicing the flat build (shard_host_index) --
    rows, tf, idf, avgdl, order keys (global maxima), DocIds, term ids."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + world * 11 + (os.getpid() % 500)
    procs = [ctx.Process(target=_build_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    corpus = synth.Corpus(n_records=20000, vocab_size=3000, min_doc_tokens=5, max_doc_tokens=30)
    full = synth.HostIndex(corpus)
    for r in range(world):
        want = shard.shard_host_index(full, r, world)
        g = got[r]
        assert (g["rank_to_tid"] == full.rank_to_tid).all()
        for key in ("term_offsets", "posting_rows", "posting_tf", "doc_lens", "doc_ids"):
            assert (np.asarray(g[key]) == np.asarray(want[key])).all(), key
        for key in ("idf", "order_key"):
            assert (np.asarray(g[key]).view(np.uint64) == np.asarray(want[key]).view(np.uint64)).all(), key
        assert float(g["avgdl"]).hex() == float(want["avgdl"]).hex()


@pytest.mark.gpu
@pytest.mark.parametrize("G", [2, 4, 8])
def test_device_merge_of_simulated_shards(gpu, G):
    _, _, hx, tids = synth_setup(100000, 5000, 5, 30, 300)
    full = search.DeviceIndex.from_host(hx).search_lists(tids, K)
    nq = len(tids)
    ids = torch.zeros((G, nq, K), dtype=torch.int64)
    sc = torch.zeros((G, nq, K), dtype=torch.float64)
    nn = torch.zeros((G, nq), dtype=torch.int32)
    post = np.zeros(nq, np.uint64)
    for g in range(G):
        d = shard.shard_host_index(hx, g, G)
        dev = search.DeviceIndex(d["term_offsets"], d["posting_rows"], d["idf"], d["order_key"],
                                 d["doc_lens"], d["doc_ids"], d["avgdl"], posting_tf=d["posting_tf"])
        r = dev.search_lists(tids, K)
        ids[g] = torch.from_numpy(r["ids"].view(np.int64))
        sc[g] = torch.from_numpy(r["scores"])
        nn[g] = torch.from_numpy(r["n"].astype(np.int32))
        post += r["postings"]
    out = shard.gather_and_merge(dict(ids=ids[0].cuda(), scores=sc[0].cuda(), n=nn[0].cuda()), K, 1)
    dev_out = dict(ids=torch.zeros((nq, K), dtype=torch.int64, device="cuda"),
                   scores=torch.zeros((nq, K), dtype=torch.float64, device="cuda"),
                   n=torch.zeros(nq, dtype=torch.int32, device="cuda"),
                   conf=torch.zeros(nq, dtype=torch.float64, device="cuda"),
                   skip=torch.zeros(nq, dtype=torch.uint8, device="cuda"))
    search.merge_shards_device(ids.cuda(), sc.cuda(), nn.cuda(), dev_out, K)
    torch.cuda.synchronize()
    got = {k: v.cpu().numpy() for k, v in dev_out.items()}
    got["ids"] = got["ids"].view(np.uint64)
    got["postings"] = post
    check_batch(got, full["ids"], full["scores"], full["n"], full["postings"], what=f"G={G}")
    assert out["n"].shape[0] == nq


def _gpu_worker(rank, world, port, out_q):
    """One rank of the sharded path on a shared GPU: ShardedIndex (this rank's
    shard, global statistics), device search, all-gather (gloo transport),
    device merge."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    corpus, _, hx, tids = synth_setup(60000, 5000, 5, 30, 200)
    sh, _ = shard.ShardedIndex.from_corpus(corpus, rank, world, device=0, threads=2)
    off = np.zeros(len(tids) + 1, np.uint32)
    off[1:] = np.cumsum([len(t) for t in tids])
    flat = np.concatenate([np.asarray(t, np.uint32) for t in tids])
    tau = np.linspace(0.0, 0.4, len(tids))
    # HM_FLAG_SEED_ALL: the seeded pass (and with it the shards' bound exchange) runs on these small shards
    res = sh.search_batch(off, flat, K, tau=torch.from_numpy(tau).cuda(), flags=search.HM_FLAG_SEED_ALL)
    if rank == 0:
        out_q.put({k: v for k, v in res.items()})
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_index_ranks_on_one_gpu_equal_unsharded(gpu, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + world * 7 + (os.getpid() % 500)
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    _, _, hx, tids = synth_setup(60000, 5000, 5, 30, 200)
    ids, sc, n, post = restate.OracleIndex.from_host(hx).topk(tids, K)
    tau = np.linspace(0.0, 0.4, len(tids))
    assert (res["n"].astype(np.uint32) == n).all()
    assert (res["postings"].astype(np.uint64) == post).all()  # summed over the shards
    for i in range(len(n)):
        assert (res["ids"][i, :n[i]].view(np.uint64) == ids[i, :n[i]]).all()
        assert (res["scores"][i, :n[i]].view(np.uint64) == sc[i, :n[i]].view(np.uint64)).all()
        assert res["conf"][i] == restate.margin(sc[i, :n[i]])
        assert bool(res["skip"][i]) == (res["conf"][i] >= tau[i])  # the caller's per-query tau
