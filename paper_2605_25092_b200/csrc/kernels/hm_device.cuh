// Device-side layout and helpers shared by the BM25 search kernels.
//
// HBM layout of an index (built once by hm_index_create, host/hm_index.cpp):
//   post[P]      u32  packed posting: (row << code_bits) | code.  Posting lists
//                     are term-major, rows strictly increasing per term, so the
//                     packed words are sorted and binary-searchable by row.
//                     code < n_codes names a (tf, doc_len) pair of the code
//                     table; code == esc means "look tf up in tf[] and doc_len
//                     in doc_lens[]".  4 B per posting.
//   tf[P]        u32  raw term frequency (escapes and exact rescoring only)
//   term_off[V+1] u64, idf[V] f64 (exact), idf32[V] f32 (selection),
//   order_key[V] f64 (plan order), long_slot[V] i32,
//   tile_tab[n_long][n_tiles+1] u32: for "long" terms (df > 32 * n_tiles)
//                     the offset, relative to the term start, of the first
//                     posting of every kTile-row tile.
//   doc_lens[N] u32, doc_ids[N] u64.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "hm_types.h"

namespace hm {


// ---------------------------------------------------------------------------
// exact BM25 in the reference's operation order (src/csr_index.cpp:10-15):
//   norm = avgdl > 0 ? len / avgdl : 1;  denom = tf + k1 * ((1 - b) + b * norm)
//   s = ((idf * tf) * (k1 + 1)) / denom
// Explicit round-to-nearest intrinsics: never contracted into FMAs.
__device__ __forceinline__ double bm25_exact(double tf, double idf, double dl,
                                             double avgdl, double k1, double b) {
    double norm = avgdl > 0.0 ? __ddiv_rn(dl, avgdl) : 1.0;
    double denom = __dadd_rn(tf, __dmul_rn(k1, __dadd_rn(__dsub_rn(1.0, b), __dmul_rn(b, norm))));
    return __ddiv_rn(__dmul_rn(__dmul_rn(idf, tf), __dadd_rn(k1, 1.0)), denom);
}

// idf-free impact tf*(k1+1)/(tf + K_len) evaluated in fp64, rounded once.
__device__ __forceinline__ float impact32(double tf, double dl, double avgdl,
                                          double k1, double b) {
    double norm = avgdl > 0.0 ? dl / avgdl : 1.0;
    double denom = tf + k1 * (1.0 - b + b * norm);
    return static_cast<float>(tf * (k1 + 1.0) / denom);
}

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t ldg_stream(const uint32_t* p) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

// first index in [lo, hi) whose packed word is >= key
__device__ __forceinline__ uint64_t lower_bound_packed(const uint32_t* post, uint64_t lo,
                                                       uint64_t hi, uint32_t key) {
    while (lo < hi) {
        uint64_t mid = lo + ((hi - lo) >> 1);
        if (__ldg(post + mid) < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
// first posting of term [lo, hi) with row >= row (rows may be >= 2^(32-cb))
__device__ __forceinline__ uint64_t lower_bound_row(const uint32_t* post, uint64_t lo,
                                                    uint64_t hi, uint32_t row, uint32_t cb) {
    while (lo < hi) {
        uint64_t mid = lo + ((hi - lo) >> 1);
        if ((__ldg(post + mid) >> cb) < row) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// canonical ranking (include/hybrid/types.hpp:21-25): score desc, DocId asc
__device__ __forceinline__ bool better(double sa, uint64_t ia, double sb, uint64_t ib) {
    if (sa != sb) return sa > sb;
    return ia < ib;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

}  // namespace hm
