"""GPU parity of the essential-term variant of the tile sweep (MaxScore inside
the sweep, the reference's lossless pruning of CsrIndex::bm25_topk_maxscore,
src/csr_index.cpp:106-207, whose output equals the exhaustive bm25_topk,
acceptance.cpp:144-171).

The variant serves plans of >= 8 terms by default (C4's 24-32-term agent
queries) and every query with HM_FLAG_NE_ALL; HM_FLAG_NO_NESKIP turns it off.
All three must give the oracle's bits: ids, score bits, counts, Margin
confidence, skip and postings_touched.
"""
import numpy as np
import pytest

from _util import check_batch, restate, search, synth_setup

pytestmark = pytest.mark.gpu

FLAGS = (0, search.HM_FLAG_NE_ALL, search.HM_FLAG_NO_NESKIP,
         search.HM_FLAG_NE_ALL | search.HM_FLAG_EXHAUSTIVE)


@pytest.fixture(scope="module")
def long_plans(gpu):
    """100K Zipf docs with 24-32-term queries sampled from 40-80-token gold
    documents (the C4 shape at C1 size): the low-bound head terms hold most
    postings, so the variant leaves them out of the stream."""
    corpus, queries, hx, tids = synth_setup(100000, 5000, 40, 80, 600, min_terms=24, max_terms=32)
    dev = search.DeviceIndex.from_host(hx)
    orc = restate.OracleIndex.from_host(hx)
    return dict(hx=hx, tids=tids, dev=dev, orc=orc)


@pytest.mark.parametrize("k", [1, 10, 100])
@pytest.mark.parametrize("flags", FLAGS)
def test_long_plans_bit_identical(long_plans, k, flags):
    got = long_plans["dev"].search_lists(long_plans["tids"], k, flags=flags)
    ids, sc, n, post = long_plans["orc"].topk(long_plans["tids"], k)
    check_batch(got, ids, sc, n, post, what=f"long plans k={k} flags={flags}")


def test_long_plans_window_and_params(long_plans):
    """A row window (recency / doc shard) and other (k1, b): the left-out
    bounds come from the re-baked impacts."""
    n_docs = len(long_plans["hx"].doc_ids)
    lo, hi = 5011, n_docs - 20000
    for k1, b in ((0.9, 0.4), (2.0, 1.0)):
        got = long_plans["dev"].search_lists(long_plans["tids"], 20, row_lo=lo, row_hi=hi, k1=k1, b=b)
        w = long_plans["orc"].topk(long_plans["tids"], 20, row_lo=lo, row_hi=hi, k1=k1, b=b)
        check_batch(got, *w, what=f"long plans window k1={k1} b={b}")


def test_short_plans_through_the_variant(gpu):
    """C1-shaped short queries forced through the variant (HM_FLAG_NE_ALL),
    with and without the seeded pass's starting bound."""
    corpus, queries, hx, tids = synth_setup(100000, 5000, 5, 30, 1000)
    dev = search.DeviceIndex.from_host(hx)
    orc = restate.OracleIndex.from_host(hx)
    ids, sc, n, post = orc.topk(tids, 10)
    for flags in (search.HM_FLAG_NE_ALL, search.HM_FLAG_NE_ALL | search.HM_FLAG_SEED_ALL,
                  search.HM_FLAG_NE_ALL | search.HM_FLAG_EXHAUSTIVE):
        got = dev.search_lists(tids, 10, flags=flags)
        check_batch(got, ids, sc, n, post, what=f"C1 flags={flags}")


def test_mixed_batch_routes_by_plan_length(long_plans):
    """One batch mixing 3-term, 8-32-term and > 32-term plans: each goes to its
    kernel (plain sweep / essential-term variant / exact fp64) and the
    results are the oracle's."""
    rng = np.random.default_rng(11)
    V = len(long_plans["hx"].idf)
    tids = list(long_plans["tids"][:40])
    tids += [t[:3] for t in long_plans["tids"][40:80]]
    tids += [rng.choice(V, size=n, replace=False).astype(np.uint32) for n in (33, 40, 64, 200, 300)]
    rng.shuffle(tids)
    got = long_plans["dev"].search_lists(tids, 10)
    ids, sc, n, post = long_plans["orc"].topk(tids, 10)
    check_batch(got, ids, sc, n, post, what="mixed plan lengths")
