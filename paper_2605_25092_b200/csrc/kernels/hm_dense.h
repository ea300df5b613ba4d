// Device layout and launcher of the dense escalate channel (kernels/dense.cu;
// C ABI in host/hm_dense.cpp).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace hm {

// hybrid::EmbeddingMatrix (include/hybrid/dense.hpp:13-22) in HBM, the
// reference's own layout: row-major fp32 [n x dim] plus the DocIds.
struct DenseDev {
    const float* E;
    const uint64_t* ids;
    uint32_t n, dim;
};

struct DenseArgs {
    uint32_t nq;
    const float* q_in;     // [nq x dim] fp32 queries
    double* q64;           // [nq x dim] scratch: the queries widened once
    uint32_t k;
    uint32_t n_slabs;      // document slabs (grid.y); partial lists per slab
    uint64_t* part_ids;    // [n_slabs][nq][k]
    double* part_scores;   // [n_slabs][nq][k]
    uint32_t* part_n;      // [n_slabs][nq]
    uint64_t* out_ids;     // [nq * k]
    double* out_scores;    // [nq * k]
    uint32_t* out_n;       // [nq]
};

// tensor-core candidate path (kernels/dense_tc.cu)
struct DenseTcArgs {
    uint32_t nq, dim, n_rows, k, n_slabs;
    const float* q;          // [nq x dim] fp32 queries (device)
    float err_scale;         // 1.25 (2^-9 + 2^-20 + dim 2^-22) max_r ||r||
    uint32_t* cand_n;        // [nq] (zeroed before the launch)
    int* thr_key;            // [nq] shared selection bound, order-preserving int (0x80808080 = -huge)
    uint32_t* cand_rows;     // [nq x cand_cap]
    uint32_t cand_cap;
    uint64_t* out_ids;       // [nq * k]
    double* out_scores;
    uint32_t* out_n;
};
uint32_t dense_tc_max_k();
uint32_t dense_tc_tile_rows();  // rows per B tile (the E map's box)
uint32_t dense_tc_slabs(uint32_t nq, uint32_t n_rows, int sms);
// map_q / map_e: CUtensorMap (fp32, K-major, 32 x {128, 256} boxes, 128B swizzle)
cudaError_t launch_dense_tc(const DenseDev& ix, const void* map_q, const void* map_e, const DenseTcArgs& a, int sms,
                            cudaStream_t st);

uint32_t dense_max_k();
uint32_t dense_slabs(uint32_t nq, uint32_t n_rows, int sms);
cudaError_t launch_dense(const DenseDev& ix, const DenseArgs& a, cudaStream_t st);
// k > dense_max_k(): one query, every row scored, two stable radix sorts
size_t dense_large_k_bytes(uint32_t n_rows);
cudaError_t launch_dense_widen(const float* q, double* q64, uint32_t dim, cudaStream_t st);
cudaError_t launch_dense_large_k(const DenseDev& ix, const double* q64, uint32_t k, void* scratch, size_t bytes,
                                 uint64_t* out_ids, double* out_scores, uint32_t* out_n, cudaStream_t st);

}  // namespace hm
