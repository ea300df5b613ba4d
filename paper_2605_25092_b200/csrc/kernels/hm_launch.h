// Host-visible launchers of the sm_100a search kernels (kernels/bm25_search.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "hm_types.h"

namespace hm {

// one thread per query: make_plan (src/csr_index.cpp:31-48) + LPT cost
cudaError_t launch_plan(const DevIndex& ix, const BatchArgs& a, uint32_t* order_in,
                        cudaStream_t st);
// LPT order: queries sorted by descending posting cost (CUB radix sort)
cudaError_t lpt_sort_bytes(uint32_t nq, size_t* bytes);
cudaError_t launch_lpt_sort(void* temp, size_t bytes, const BatchArgs& a,
                            uint64_t* cost_sorted, const uint32_t* order_in,
                            int key_bits, cudaStream_t st);
// the seeded pass's own LPT order (cost_seed descending) into order_seed
// (key_bits: the costs' significant bits -- radix passes over those only)
cudaError_t launch_seed_sort(void* temp, size_t bytes, const BatchArgs& a, uint64_t* cost_sorted,
                             const uint32_t* order_in, uint32_t* order_seed, int key_bits, cudaStream_t st);
// small batches split each query into row slabs (BatchArgs::split): slab
// queries in the real LPT order, and their postings summed per real query
cudaError_t launch_expand_order(uint32_t nq_real, uint32_t split, const uint32_t* order_real, uint32_t* order,
                                cudaStream_t st);
cudaError_t launch_sum_slab_postings(uint32_t nq_real, uint32_t split, const uint64_t* v_post, uint64_t* out_post,
                                     cudaStream_t st);
// persistent fused kernel: TAAT scoring + selection + exact rescoring + margin
cudaError_t launch_search(const DevIndex& ix, const BatchArgs& a, int grid, cudaStream_t st);
// launch_search also runs the essential-term variant first (one more launch)
bool sweep_ne_launched(const BatchArgs& a);
// seeded MaxScore pre-pass (kernels/search_seed.cu); hands the queries it
// does not serve to the exhaustive kernel through a.fb_list
cudaError_t launch_search_seed(const DevIndex& ix, const BatchArgs& a, int grid, cudaStream_t st);
// persistent exact fp64 kernel for the queries in a.exact_list
cudaError_t launch_exact(const DevIndex& ix, const BatchArgs& a, int grid, cudaStream_t st);
// merge of per-shard exact top-k lists (after the all-gather)
cudaError_t launch_merge(uint32_t n_shards, uint32_t nq, uint32_t k, const uint64_t* ids,
                         const double* scores, const uint32_t* n, const double* tau,
                         double tau_default, double eps, uint64_t* out_ids,
                         double* out_scores, uint32_t* out_n, double* out_conf,
                         uint8_t* out_skip, cudaStream_t st);
// doc-sharded search: all-gather of the shards' lists over peer memory fused
// with the k-way merge (rank by binary search), Margin, skip, postings sum
cudaError_t launch_gather_merge(const ShardLists& lists, uint32_t nq, uint32_t k, const double* tau,
                                double tau_default, double eps, uint64_t* out_ids, double* out_scores,
                                uint32_t* out_n, double* out_conf, uint8_t* out_skip, uint64_t* out_post,
                                cudaStream_t st);
// doc shards: per query the k-th largest of the shards' k best seed scores
cudaError_t launch_bound_kth(const BoundLists& lists, uint32_t nq, uint32_t k, float* out, cudaStream_t st);
// K0: bake the long-term postings into bk[] for (k1, b); *err |= 1 when an
// impact falls outside the 7 representable binades (kernels/bake.cu)
uint32_t bake_ks(double k1);
cudaError_t launch_bake(const DevIndex& ix, const uint32_t* long_terms, uint32_t n_long, double k1,
                        double b, uint32_t ks, uint32_t* bk, uint32_t* err, cudaStream_t st);
// the wide path (wide.cu): one group of w.G queries, any k and plan length;
// plan arrays of `a` must be filled (launch_plan)
size_t wide_sort_bytes(uint64_t n_items);
cudaError_t launch_wide_group(const DevIndex& ix, const BatchArgs& a, const WideArgs& w, void* sort_tmp,
                              size_t sort_bytes, cudaStream_t st);
// resident CTAs per SM of the two persistent kernels
cudaError_t search_occupancy(int* search_blocks_per_sm, int* exact_blocks_per_sm);
cudaError_t search_occupancy_fast(int* blocks);
size_t search_smem_bytes();

}  // namespace hm
