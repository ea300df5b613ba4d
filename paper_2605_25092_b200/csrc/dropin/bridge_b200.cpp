// Drop-in implementation of the reference's learned-sparse bridge API
// (proj/include/hybrid/bridge.hpp, compiled against the reference's own
// header in place) on the B200 path: it replaces proj/src/bridge.cpp at link
// time.  Ingest / export / validate are host-side data-format work (the CSC
// transpose of per-doc vectors, bridge.cpp:22-90); every bridge_topk and
// bridge_topk_maxscore runs on the GPU through the C ABI (hm_bridge_*,
// include/hm_b200.h), bit-identical to the reference.  There is no CPU
// scoring path.
//
// Interfaces (file:line in proj/include/hybrid/bridge.hpp):
//   SparseVector::validate          :18        (bridge.cpp:10-20)
//   bridge_ingest                   :21-25     (bridge.cpp:22-73)
//   bridge_export                   :27-29     (bridge.cpp:75-90)
//   bridge_topk / _maxscore         :31-40     -> hm_bridge_search_batch
#include <algorithm>
#include <mutex>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "hm_b200.h"
#include "hybrid/bridge.hpp"

namespace hybrid {

namespace {

void throw_on(int rc) {
    if (rc == HM_OK) return;
    const std::string msg = hm_last_error();
    if (rc == HM_ERR_INVALID) throw std::invalid_argument(msg);
    if (rc == HM_ERR_RANGE) throw std::out_of_range(msg);
    throw std::runtime_error(msg);
}

// One device copy per bridge-mode CsrIndex, uploaded on first search; the
// fingerprint catches an index destroyed and re-created at the same address.
struct BridgeEntry {
    hm_bridge* h = nullptr;
    const void* rows = nullptr;
    const void* w = nullptr;
    const void* ids = nullptr;
    std::size_t n_post = 0, n_docs = 0, n_terms = 0;
};

struct BridgeCache {
    std::mutex mu;
    std::unordered_map<const CsrIndex*, BridgeEntry> map;
    ~BridgeCache() {
        for (auto& kv : map) hm_bridge_destroy(kv.second.h);
    }
};

hm_bridge* device_bridge(const CsrIndex& x) {
    static BridgeCache c;
    std::lock_guard<std::mutex> lk(c.mu);
    BridgeEntry& e = c.map[&x];
    if (e.h && e.rows == x.posting_rows.data() && e.w == x.posting_weights.data() &&
        e.ids == x.doc_ids.data() && e.n_post == x.posting_rows.size() && e.n_docs == x.doc_ids.size() &&
        e.n_terms == x.terms.size())
        return e.h;
    if (e.h) {
        hm_bridge_destroy(e.h);
        e.h = nullptr;
    }
    hm_bridge_view v{};
    v.n_terms = static_cast<uint32_t>(x.terms.size());
    v.term_offsets = x.term_offsets.data();
    v.posting_rows = x.posting_rows.data();
    v.posting_weights = x.posting_weights.data();
    v.n_docs = x.num_docs();
    v.doc_ids = x.doc_ids.data();
    hm_bridge* h = nullptr;
    throw_on(hm_bridge_create(&v, 0, &h));
    e = BridgeEntry{h, x.posting_rows.data(), x.posting_weights.data(), x.doc_ids.data(),
                    x.posting_rows.size(), x.doc_ids.size(), x.terms.size()};
    return h;
}

void check_bridge(const CsrIndex& idx) {
    if (idx.mode != IndexMode::Bridge) throw std::runtime_error("bridge scoring requires a bridge-mode index");
}

RankedList gpu_bridge_topk(const CsrIndex& idx, const SparseVector& q, std::size_t k, SearchStats* stats) {
    check_bridge(idx);
    q.validate();
    RankedList out;
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
    throw_on(hm_bridge_search_batch(device_bridge(idx), &b, &r));
    if (stats) stats->postings_touched += post;  // accumulates (bridge.cpp:135)
    out.entries.reserve(n);
    for (uint32_t i = 0; i < n; ++i) out.entries.emplace_back(ids[i], sc[i]);
    return out;
}

}  // namespace

void SparseVector::validate() const {
    if (indices.size() != values.size()) throw std::invalid_argument("indices/values length mismatch");
    for (std::size_t i = 0; i < indices.size(); ++i) {
        if (i > 0 && indices[i] <= indices[i - 1])
            throw std::invalid_argument("sparse vector indices must be strictly increasing");
        if (!(values[i] > 0.0)) throw std::invalid_argument("sparse vector values must be > 0");
    }
}

// Counting-sort transpose: one pass sizes every term's list, a second pass
// (docs in row order) fills it, so rows ascend within each term.
CsrIndex bridge_ingest(const std::vector<std::pair<DocId, SparseVector>>& doc_vectors) {
    CsrIndex idx;
    idx.mode = IndexMode::Bridge;
    std::unordered_set<DocId> seen;
    seen.reserve(doc_vectors.size());
    std::uint32_t dim = 0;
    for (const auto& [id, vec] : doc_vectors) {
        if (!seen.insert(id).second) throw std::runtime_error("duplicate doc id: " + std::to_string(id));
        vec.validate();
        if (!vec.indices.empty()) dim = std::max(dim, vec.indices.back() + 1);
    }
    idx.term_offsets.assign(dim + 1ull, 0);
    for (const auto& dv : doc_vectors)
        for (std::uint32_t t : dv.second.indices) ++idx.term_offsets[t + 1ull];
    for (std::uint32_t t = 0; t < dim; ++t) idx.term_offsets[t + 1ull] += idx.term_offsets[t];
    const std::uint64_t P = idx.term_offsets[dim];
    idx.posting_rows.resize(P);
    idx.posting_weights.resize(P);
    std::vector<std::uint64_t> fill(idx.term_offsets.begin(), idx.term_offsets.end() - 1);
    idx.doc_ids.reserve(doc_vectors.size());
    idx.doc_lens.reserve(doc_vectors.size());
    double len_sum = 0.0;
    for (const auto& [id, vec] : doc_vectors) {
        const auto row = static_cast<std::uint32_t>(idx.doc_ids.size());
        for (std::size_t i = 0; i < vec.nnz(); ++i) {
            const std::uint64_t at = fill[vec.indices[i]]++;
            idx.posting_rows[at] = row;
            idx.posting_weights[at] = vec.values[i];
        }
        idx.doc_ids.push_back(id);
        idx.doc_lens.push_back(static_cast<std::uint32_t>(vec.nnz()));
        len_sum += static_cast<double>(vec.nnz());
    }
    idx.avgdl = idx.doc_ids.empty() ? 0.0 : len_sum / static_cast<double>(idx.doc_ids.size());
    idx.terms.reserve(dim);
    idx.term_idfs.assign(dim, 0.0);
    idx.term_maxscores.assign(dim, 0.0);
    for (std::uint32_t t = 0; t < dim; ++t) {
        idx.terms.push_back(std::to_string(t));
        idx.vocab.emplace(idx.terms.back(), t);
        for (std::uint64_t i = idx.term_offsets[t]; i < idx.term_offsets[t + 1]; ++i)
            idx.term_maxscores[t] = std::max(idx.term_maxscores[t], idx.posting_weights[i]);
    }
    idx.term_order_keys = idx.term_maxscores;
    return idx;
}

std::vector<std::pair<DocId, SparseVector>> bridge_export(const CsrIndex& idx) {
    if (idx.mode != IndexMode::Bridge) throw std::runtime_error("bridge export requires a bridge-mode index");
    std::vector<std::pair<DocId, SparseVector>> out(idx.doc_ids.size());
    for (std::size_t r = 0; r < idx.doc_ids.size(); ++r) out[r].first = idx.doc_ids[r];
    for (std::uint32_t t = 0; t < idx.terms.size(); ++t)
        for (std::uint64_t i = idx.term_offsets[t]; i < idx.term_offsets[t + 1]; ++i) {
            SparseVector& v = out[idx.posting_rows[i]].second;
            v.indices.push_back(t);
            v.values.push_back(idx.posting_weights[i]);
        }
    return out;
}

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
