// Device layout and launchers of the learned-sparse bridge path
// (kernels/bridge.cu; C ABI in host/hm_bridge.cpp).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hm {

// A Bridge-mode CsrIndex (proj/include/hybrid/csr_index.hpp:44-60 with
// mode == IndexMode::Bridge, built by bridge_ingest, src/bridge.cpp:22-73),
// HBM-resident in the reference's own layout: 12 B per posting.
struct BridgeDev {
    const uint64_t* term_off;  // [n_terms + 1]
    const uint32_t* rows;      // [P], strictly increasing per term
    const double* w;           // [P] learned weights
    const uint64_t* doc_ids;   // [n_docs]
    uint32_t n_terms, n_docs;
};

struct BridgeArgs {
    uint32_t nq;
    const uint64_t* q_off;     // [nq + 1]
    const uint32_t* q_idx;     // validated sparse vectors (ascending term ids)
    const double* q_val;
    uint32_t k;
    uint32_t row_lo, row_hi;
    uint32_t split, nq_real;   // split > 1: query q = slab q / nq_real of real query q % nq_real
    uint32_t m_max;            // >= every query's nnz (scratch stride)
    uint64_t* scratch;         // [grid][(3 + 2 * 8) * m_max]
    uint32_t* counters;        // [0] query cursor
    uint64_t* out_ids;         // [nq * k]
    double* out_scores;        // [nq * k]
    uint32_t* out_n;           // [nq]
    uint64_t* out_post;        // [nq] or null
};

uint32_t bridge_max_k();
// CTAs a launch for this k uses (the scratch is sized per CTA)
uint32_t bridge_grid(uint32_t k, int sms);
cudaError_t launch_bridge(const BridgeDev& ix, const BridgeArgs& a, int sms, cudaStream_t st);

}  // namespace hm
