"""Doc-sharded search behind the C ABI (hm_sharded_*): G shards on listed
devices (the same device may be listed more than once -- the one-GPU box runs
G shards on cuda:0, the merge then reads local memory; on a multi-GPU box it
reads peer memory over NVLink), results bit-identical to the unsharded index
and to the reference restatement; plus the NCCL one-rank-per-GPU path when
the box has two GPUs."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from _util import check_batch, restate, search, synth_setup

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _flat(tids):
    off = np.zeros(len(tids) + 1, np.uint32)
    off[1:] = np.cumsum([len(t) for t in tids])
    flat = np.concatenate([np.asarray(t, np.uint32) for t in tids]) if off[-1] else np.zeros(0, np.uint32)
    return off, flat


@pytest.fixture(scope="module")
def c1ish():
    _, _, hx, tids = synth_setup(100000, 5000, 5, 30, 400)
    return hx, tids


@pytest.mark.gpu
@pytest.mark.parametrize("G", [1, 2, 3, 8])
def test_sharded_equals_unsharded_and_oracle(gpu, c1ish, G):
    hx, tids = c1ish
    off, flat = _flat(tids)
    sh = search.ShardedDeviceIndex.from_host(hx, [0] * G)
    info = sh.info()
    assert info["n_shards"] == G and info["shard_row"][-1] == hx.n_docs
    assert info["p2p"].all()  # same device: the merge reads the shards in place
    tau = np.linspace(0.0, 0.5, len(tids))
    got = sh.search_batch(off, flat, 10, tau=tau)
    ids, sc, n, post = restate.OracleIndex.from_host(hx).topk(tids, 10)
    assert (got["n"] == n).all()
    assert (got["postings"] == post).all()  # postings_touched summed over the shards
    for i in range(len(n)):
        m = n[i]
        assert (got["ids"][i, :m] == ids[i, :m]).all(), f"G={G} query {i}"
        assert (got["scores"][i, :m].view(np.uint64) == sc[i, :m].view(np.uint64)).all()
        conf = restate.margin(sc[i, :m])
        assert got["conf"][i] == conf and bool(got["skip"][i]) == (conf >= tau[i])


@pytest.mark.gpu
@pytest.mark.parametrize("k", [0, 1, 100, 300])
def test_sharded_any_k(gpu, c1ish, k):
    hx, tids = c1ish
    tids = tids[:64]
    off, flat = _flat(tids)
    sh = search.ShardedDeviceIndex.from_host(hx, [0, 0, 0, 0])
    got = sh.search_batch(off, flat, k)
    want = search.DeviceIndex.from_host(hx).search_batch(off, flat, k)
    assert (got["n"] == want["n"]).all()
    assert (got["ids"] == want["ids"]).all() and (got["scores"].view(np.uint64) == want["scores"].view(np.uint64)).all()
    assert (got["conf"] == want["conf"]).all() and (got["skip"] == want["skip"]).all()
    assert (got["postings"] == want["postings"]).all()


@pytest.mark.gpu
def test_sharded_row_window(gpu, c1ish):
    hx, tids = c1ish
    off, flat = _flat(tids[:128])
    sh = search.ShardedDeviceIndex.from_host(hx, [0, 0, 0])
    dev = search.DeviceIndex.from_host(hx)
    n = hx.n_docs
    for lo, hi in [(0, n // 5), (n // 3 - 7, n // 3 + 11), (n // 2, 0), (n - 1, n)]:
        got = sh.search_batch(off, flat, 10, row_lo=lo, row_hi=hi)
        want = dev.search_batch(off, flat, 10, row_lo=lo, row_hi=hi)
        for key in ("n", "ids", "conf", "skip", "postings"):
            assert (got[key] == want[key]).all(), (lo, hi, key)
        assert (got["scores"].view(np.uint64) == want["scores"].view(np.uint64)).all()


@pytest.mark.gpu
@pytest.mark.parametrize("k", [1, 10, 100])
@pytest.mark.parametrize("flags", [0, 32])
def test_sharded_bounded_any_k_and_windows(gpu, c1ish, k, flags):
    """Batches of 256+ queries exchange the shards' k best seed scores first
    (each shard then keeps only documents that can be in the union's top-k):
    still the unsharded answer, with and without a row window.  flags 32 =
    HM_FLAG_SEED_ALL: the seeded pass runs on these small shards too, so the
    bounds are real and the shards' seeded passes run without their seed
    phase."""
    hx, tids = c1ish
    off, flat = _flat(tids[:300])
    sh = search.ShardedDeviceIndex.from_host(hx, [0, 0, 0, 0])
    dev = search.DeviceIndex.from_host(hx)
    n = hx.n_docs
    for lo, hi in [(0, 0), (n // 7, n - n // 5)]:
        got = sh.search_batch(off, flat, k, row_lo=lo, row_hi=hi, flags=flags)
        want = dev.search_batch(off, flat, k, row_lo=lo, row_hi=hi)
        for key in ("n", "ids", "conf", "skip", "postings"):
            assert (got[key] == want[key]).all(), (k, lo, hi, key)
        assert (got["scores"].view(np.uint64) == want["scores"].view(np.uint64)).all()


@pytest.mark.gpu
def test_bound_pass_and_external_bound(gpu, c1ish):
    """HM_FLAG_BOUND_ONLY reports a lower bound on every query's k-th score
    (selection domain, score * 2^-61); searching with that bound -- or any
    bound at or below the k-th score -- as ext_bound returns the same top-k."""
    hx, tids = c1ish
    off, flat = _flat(tids)
    dev = search.DeviceIndex.from_host(hx)
    nq, k = len(tids), 10
    d_off = torch.from_numpy(off.view(np.int32)).cuda()
    d_tid = torch.from_numpy(flat.view(np.int32)).cuda()

    def outbuf():
        return dict(ids=torch.zeros((nq, k), dtype=torch.int64, device="cuda"),
                    scores=torch.zeros((nq, k), dtype=torch.float64, device="cuda"),
                    n=torch.zeros(nq, dtype=torch.int32, device="cuda"),
                    conf=torch.zeros(nq, dtype=torch.float64, device="cuda"),
                    skip=torch.zeros(nq, dtype=torch.uint8, device="cuda"),
                    postings=torch.zeros(nq, dtype=torch.int64, device="cuda"))
    ref = outbuf()
    dev.search_batch_device(d_off, d_tid, ref, k)
    seeds = torch.zeros((nq, k), dtype=torch.float32, device="cuda")
    # (HM_FLAG_SEED_ALL: the seeded pass also runs on this small index)
    dev.search_batch_device(d_off, d_tid, outbuf(), k, flags=search.HM_FLAG_BOUND_ONLY | search.HM_FLAG_SEED_ALL,
                            out_bound=seeds)
    torch.cuda.synchronize()
    sc = ref["scores"].cpu().numpy()
    nn = ref["n"].cpu().numpy()
    sel = sc * 2.0 ** -61
    sv = -np.sort(-seeds.cpu().numpy().astype(np.float64), axis=1)  # the k best seed scores, descending
    for i in range(nq):  # the j-th best seed score never exceeds the j-th best score (1e-4: the domains)
        m = int(nn[i])
        assert (sv[i, :m] <= sel[i, :m] * (1 + 1e-4)).all(), f"query {i}: a seed score above the top-k"
        assert (sv[i, m:] == 0).all()
    bound = seeds.min(dim=1).values.contiguous()  # one shard: the k-th largest of its k values
    kth = np.where(nn >= k, sc[:, k - 1], 0.0) * 2.0 ** -61
    assert (bound.cpu().numpy() > 0).sum() > nq // 4, "the seeded pass reported almost no bounds"
    for ext in (bound, torch.from_numpy((kth * (1 - 1e-4)).astype(np.float32)).cuda()):
        for flags in (0, search.HM_FLAG_SEED_ALL):  # the sweep alone / the seeded pass without its seed phase
            got = outbuf()
            dev.search_batch_device(d_off, d_tid, got, k, ext_bound=ext, flags=flags)
            torch.cuda.synchronize()
            for key in ("n", "ids", "scores", "postings"):
                assert torch.equal(got[key], ref[key]), (flags, key)


@pytest.mark.gpu
def test_sharded_errors(gpu, c1ish):
    hx, tids = c1ish
    sh = search.ShardedDeviceIndex.from_host(hx, [0, 0])
    with pytest.raises(IndexError, match="term id out of range"):
        sh.search_batch(np.array([0, 1], np.uint32), np.array([hx.n_terms + 5], np.uint32), 10)
    with pytest.raises(ValueError, match="n_shards"):
        search.ShardedDeviceIndex.from_host(hx, [0] * 17)


def test_sharded_symbols_exported():
    L = search.lib()
    for name in ("hm_sharded_create", "hm_sharded_destroy", "hm_sharded_info", "hm_sharded_search_batch"):
        assert hasattr(L, name)


@pytest.mark.gpu
@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2,
                    reason="needs two GPUs (the NCCL all-gather over NVLink)")
def test_nccl_two_ranks_equal_unsharded(gpu, tmp_path):
    """One process per GPU over NCCL: each rank builds only its shard, searches
    on its own GPU, all-gathers k candidates per query over NVLink and merges
    (paper_2605_25092_b200/shard.py); rank 0's answer equals the oracle."""
    script = tmp_path / "nccl_run.py"
    out = tmp_path / "res.npz"
    script.write_text(f"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, {ROOT!r}); sys.path.insert(0, {os.path.join(ROOT, 'tests')!r})
from _util import synth_setup
from paper_2605_25092_b200 import shard
rank = int(os.environ["RANK"]); world = int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl")
corpus, _, hx, tids = synth_setup(60000, 5000, 5, 30, 200)
sh, _ = shard.ShardedIndex.from_corpus(corpus, rank, world, device=rank, threads=2)
off = np.zeros(len(tids) + 1, np.uint32); off[1:] = np.cumsum([len(t) for t in tids])
res = sh.search_batch(off, np.concatenate(tids).astype(np.uint32), 10)
if rank == 0:
    np.savez({str(out)!r}, **{{k: np.asarray(v) for k, v in res.items()}})
dist.barrier(); dist.destroy_process_group()
""")
    env = dict(os.environ, NCCL_DEBUG="INFO")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", str(29700 + os.getpid() % 200),
                        str(script)], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    res = np.load(out)
    _, _, hx, tids = synth_setup(60000, 5000, 5, 30, 200)
    ids, sc, n, post = restate.OracleIndex.from_host(hx).topk(tids, 10)
    got = dict(ids=res["ids"].view(np.uint64), scores=res["scores"], n=res["n"].astype(np.uint32),
               conf=res["conf"], skip=res["skip"], postings=res["postings"].astype(np.uint64))
    check_batch(got, ids, sc, n, post, what="nccl world 2")
