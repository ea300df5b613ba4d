// Drop-in for the learned-sparse bridge's search functions
// (proj/include/hybrid/bridge.hpp:31-40, compiled against the reference's own
// header in place): bridge_topk and bridge_topk_maxscore run on the GPU
// through the C ABI (hm_bridge_*, include/hm_b200.h), bit-identical to
// src/bridge.cpp:112-204.  There is no CPU scoring path.
//
// Only the two search symbols are replaced.  SparseVector::validate,
// bridge_ingest and bridge_export (host-side data-format work,
// bridge.cpp:10-90) stay the reference's object code: a maintainer links
// proj's bridge.o with bridge_topk / bridge_topk_maxscore weakened
// (objcopy --weaken-symbol, tests/cpp/Makefile).
#include <algorithm>
#include <string>
#include <vector>

#include "dropin_common.hpp"
#include "hm_b200.h"
#include "hybrid/bridge.hpp"

namespace {

using hm_dropin::throw_on;

struct BridgeEntry {
    const void* key = nullptr;
    uint64_t fp = 0;
    hm_bridge* h = nullptr;
    ~BridgeEntry() {
        if (h) hm_bridge_destroy(h);
    }
};
using Cache = hm_dropin::LruCache<BridgeEntry>;

Cache::Ptr device_bridge(const hybrid::CsrIndex& x) {
    static Cache cache(4);
    uint64_t fp = hm_dropin::mix(7, x.terms.size());
    fp = hm_dropin::sample(fp, x.term_offsets);
    fp = hm_dropin::sample(fp, x.posting_rows);
    fp = hm_dropin::sample(fp, x.posting_weights);
    fp = hm_dropin::sample(fp, x.doc_ids);
    return cache.get(&x, fp, [&](BridgeEntry& e) {
        static const uint64_t zero_off = 0;
        hm_bridge_view v{};
        v.n_terms = static_cast<uint32_t>(x.terms.size());
        v.term_offsets = x.term_offsets.empty() ? &zero_off : x.term_offsets.data();
        v.posting_rows = x.posting_rows.data();
        v.posting_weights = x.posting_weights.data();
        v.n_docs = x.num_docs();
        v.doc_ids = x.doc_ids.data();
        throw_on(hm_bridge_create(&v, 0, &e.h));
    });
}

hybrid::RankedList gpu_bridge_topk(const hybrid::CsrIndex& idx, const hybrid::SparseVector& q, std::size_t k,
                                   hybrid::SearchStats* stats) {
    if (idx.mode != hybrid::IndexMode::Bridge)
        throw std::runtime_error("bridge scoring requires a bridge-mode index");
    q.validate();
    hybrid::RankedList out;
    if (idx.terms.empty() || idx.doc_ids.empty()) return out;  // every term unknown: nothing touched
    const std::size_t kk = std::min<std::size_t>(k, idx.doc_ids.size());  // k > N: the same list
    const uint64_t off[2] = {0, q.nnz()};
    hm_bridge_batch b{};
    b.n_queries = 1;
    b.q_off = off;
    b.q_idx = q.indices.data();
    b.q_val = q.values.data();
    b.k = static_cast<uint32_t>(std::min<std::size_t>(kk, 0xFFFFFFFFu));
    std::vector<uint64_t> ids(std::max<std::size_t>(kk, 1));
    std::vector<double> sc(ids.size());
    uint32_t n = 0;
    uint64_t post = 0;
    hm_results r{ids.data(), sc.data(), &n, nullptr, nullptr, &post};
    auto e = device_bridge(idx);
    throw_on(hm_bridge_search_batch(e->h, &b, &r));
    if (stats) stats->postings_touched += post;  // accumulates (bridge.cpp:135)
    out.entries.reserve(n);
    for (uint32_t i = 0; i < n; ++i) out.entries.emplace_back(ids[i], sc[i]);
    return out;
}

}  // namespace

namespace hybrid {

RankedList bridge_topk(const CsrIndex& idx, const SparseVector& query_vec, std::size_t k, SearchStats* stats) {
    return gpu_bridge_topk(idx, query_vec, k, stats);
}

// MaxScore pruning only narrows which documents the CPU keeps accumulating;
// its output is bridge_topk's (test_bridge.cpp:108-109), computed directly.
RankedList bridge_topk_maxscore(const CsrIndex& idx, const SparseVector& query_vec, std::size_t k,
                                SearchStats* stats) {
    return gpu_bridge_topk(idx, query_vec, k, stats);
}

}  // namespace hybrid
