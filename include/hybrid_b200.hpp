// include/hybrid_b200.hpp -- batch extension of the reference's C++ search
// API (proj/include/hybrid/, used in place, never copied).
//
// The reference has no batch entry: its batch path is hybridmem's cmd_search
// calling CsrIndex::bm25_topk(_maxscore) / TemporalIndex::topk once per query
// under parallel_for (tools/hybridmem.cpp:227-313).  These functions take the
// whole batch in one call and run it as ONE GPU batch through the C ABI
// (include/hm_b200.h); result i equals the reference's per-query call on
// queries[i], bit for bit, at any batch size or composition.  The per-query
// reference entry points are implemented on top of them by
// csrc/dropin/hybrid_b200.cpp (link recipe: INTEGRATION.md).
#pragma once
#include <cstddef>
#include <string>
#include <vector>

#include "hybrid/csr_index.hpp"
#include "hybrid/temporal_index.hpp"

namespace hybrid_b200 {

/// Per-query cascade trigger of the batch (src/cascade.cpp:10-21, 79-84):
/// Margin confidence of the top-k scores and conf >= tau.
struct Decision {
    double conf = 0.0;
    bool skip = false;
};

/// CsrIndex::bm25_topk / bm25_topk_maxscore (csr_index.hpp:72-79) for every
/// query of the batch.  stats[i].postings_touched += the reference's
/// exhaustive count (sum of df over the distinct known terms,
/// csr_index.cpp:100-102) -- also for the MaxScore entry, whose CPU path
/// counts its own probe cost instead (csr_index.cpp:152-183).  decisions
/// (optional): Margin + skip at threshold tau, computed on the device.
std::vector<hybrid::RankedList> bm25_topk_batch(const hybrid::CsrIndex& index,
                                                const std::vector<std::vector<std::string>>& queries,
                                                std::size_t k, const hybrid::Bm25Params& p,
                                                std::vector<hybrid::SearchStats>* stats = nullptr,
                                                std::vector<Decision>* decisions = nullptr, double tau = 0.10);

/// TemporalIndex::topk (temporal_index.hpp:56-66) for every query: the
/// partitions are assembled once into one partition-ordered flat device index
/// (they share the corpus statistics, so its scores are the partitions'
/// bits), every partition of the budget min(k*, k_max, K) is searched for
/// every query in one GPU batch (hm_search_batch_parts), and the lists are
/// merged newest first with the reference's admissible upper-bound stop, so
/// results, partitions_searched and early_stopped are the reference's.
/// postings_touched sums the searched partitions' exhaustive counts (the CPU
/// path sums its MaxScore probe cost).
std::vector<hybrid::RankedList> temporal_topk_batch(const hybrid::TemporalIndex& index,
                                                    const std::vector<std::vector<std::string>>& queries,
                                                    std::size_t k, const hybrid::Bm25Params& p,
                                                    std::vector<hybrid::TemporalStats>* stats = nullptr,
                                                    bool use_ub_stop = true);

/// Device copies held by the drop-in's cache (LRU, at most 4 flat and 2
/// temporal indexes); release_device_copies() frees them all.
std::size_t cached_device_indexes();
void release_device_copies();

}  // namespace hybrid_b200
