// Dense escalate channel on sm_100a: brute-force inner-product top-k over an
// EmbeddingMatrix, bit-identical to hybrid::dense_topk (src/dense.cpp:86-101).
//
// The reference scores every row as dot = sum_j double(r_j) * q_j in fp64,
// j ascending, then ranks ALL rows by (score desc, DocId asc) (no score
// filter: RankedList::sort_and_truncate, include/hybrid/types.hpp:21-30).
// double(float) * double(float) is exact in fp64 (24 + 24 < 53 significant
// bits), so fma(r_j, q_j, acc) rounds exactly like acc + r_j * q_j: the
// kernel evaluates each dot as the same sequential fp64 chain, with DFMA.
//
//   dense_q64_kernel     queries -> fp64 once per batch
//   dense_exact_kernel   grid (query tile of 8, document slab); a thread owns
//                        one row of a 256-row tile and carries 8 dot chains
//                        (row loads float4, query values broadcast); the
//                        8 queries' candidate lists live in shared memory:
//                        a row joins when it reaches the list's k-th score,
//                        full lists are bitonic-sorted to their best k
//   dense_merge_kernel   per query: the slabs' sorted lists merged by rank
//   large k (> 256: the lists would not fit shared memory): every row's
//   exact score, then two stable radix sorts -- by DocId, then by score
//   descending -- which is exactly the (score desc, DocId asc) order
#include <cstdint>

#include <cub/cub.cuh>

#include "hm_dense.h"

namespace hm {
namespace {

constexpr int kDT = 256;       // threads = rows per tile
constexpr int kQT = 8;         // queries per CTA
constexpr int kDW = 512;       // list capacity (>= k + kDT, a power of two)
constexpr uint32_t kDenseMaxK = kDW - kDT;

__device__ __forceinline__ bool better(double sa, uint64_t ia, double sb, uint64_t ib) {
    return sa > sb || (sa == sb && ia < ib);
}

struct DenseSmem {
    double s[kQT][kDW];
    uint64_t id[kQT][kDW];
    uint32_t n[kQT];
    double L[kQT];  // admission bound: the list's k-th score once it holds k
};

__global__ void dense_q64_kernel(const float* q, double* q64, uint64_t n) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        q64[i] = static_cast<double>(q[i]);
}

// sort list (s, id)[0..W) in place by rank (warp-cooperative bitonic network;
// entries past n are padded with -inf sentinels)
__device__ void sort_list(double* s, uint64_t* id, uint32_t n, int lane) {
    for (uint32_t i = n + lane; i < static_cast<uint32_t>(kDW); i += 32) {
        s[i] = -__longlong_as_double(0x7ff0000000000000ll);
        id[i] = ~0ull;
    }
    __syncwarp();
    for (uint32_t size = 2; size <= static_cast<uint32_t>(kDW); size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t t = lane; t < static_cast<uint32_t>(kDW) / 2; t += 32) {
                const uint32_t i = 2 * t - (t & (stride - 1)), j = i + stride;
                const double si = s[i], sj = s[j];
                const uint64_t ii = id[i], ij = id[j];
                if ((i & size) == 0 ? better(sj, ij, si, ii) : better(si, ii, sj, ij)) {
                    s[i] = sj;
                    s[j] = si;
                    id[i] = ij;
                    id[j] = ii;
                }
            }
            __syncwarp();
        }
}

__global__ void __launch_bounds__(kDT) dense_exact_kernel(DenseDev ix, DenseArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    DenseSmem& S = *reinterpret_cast<DenseSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t q0 = blockIdx.x * kQT;
    const uint32_t nqt = min(static_cast<uint32_t>(kQT), a.nq - q0);
    const uint32_t slab = blockIdx.y;
    const uint32_t r_lo = static_cast<uint32_t>((static_cast<uint64_t>(ix.n) * slab) / a.n_slabs);
    const uint32_t r_hi = static_cast<uint32_t>((static_cast<uint64_t>(ix.n) * (slab + 1)) / a.n_slabs);
    const uint32_t k = a.k, dim = ix.dim;
    if (tid < kQT) {
        S.n[tid] = 0;
        S.L[tid] = -__longlong_as_double(0x7ff0000000000000ll);
    }
    __syncthreads();
    const double* qb = a.q64 + static_cast<uint64_t>(q0) * dim;
    uint32_t qu[kQT];  // the tile's query rows (a short last tile repeats its last query)
#pragma unroll
    for (int u = 0; u < kQT; ++u) qu[u] = static_cast<uint32_t>(u) < nqt ? u : nqt - 1;
    for (uint32_t t0 = r_lo; t0 < r_hi; t0 += kDT) {
        const uint32_t row = t0 + tid;
        double acc[kQT];
#pragma unroll
        for (int u = 0; u < kQT; ++u) acc[u] = 0.0;
        if (row < r_hi) {
            const float* r = ix.E + static_cast<uint64_t>(row) * dim;
            if ((dim & 3u) == 0) {
                const float4* r4 = reinterpret_cast<const float4*>(r);
                for (uint32_t j4 = 0; j4 < dim / 4; ++j4) {
                    const float4 x = __ldg(r4 + j4);
                    const float xv[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const double rd = static_cast<double>(xv[h]);
                        const uint32_t j = 4 * j4 + h;
#pragma unroll
                        for (int u = 0; u < kQT; ++u)
                            acc[u] = __fma_rn(rd, __ldg(qb + static_cast<uint64_t>(qu[u]) * dim + j), acc[u]);
                    }
                }
            } else {
                for (uint32_t j = 0; j < dim; ++j) {
                    const double rd = static_cast<double>(__ldg(r + j));
#pragma unroll
                    for (int u = 0; u < kQT; ++u)
                        acc[u] = __fma_rn(rd, __ldg(qb + static_cast<uint64_t>(qu[u]) * dim + j), acc[u]);
                }
            }
        }
        // admission: every row is ranked (no score filter), so a row joins
        // list u while the list holds fewer than k or it reaches the k-th score
        if (row < r_hi) {
            const uint64_t id = __ldg(ix.ids + row);
#pragma unroll
            for (int u = 0; u < kQT; ++u)
                if (static_cast<uint32_t>(u) < nqt && acc[u] >= S.L[u]) {
                    const uint32_t p = atomicAdd(&S.n[u], 1u);
                    S.s[u][p] = acc[u];
                    S.id[u][p] = id;
                }
        }
        __syncthreads();
        // lists that cannot take another full tile: sort, keep the best k
        for (uint32_t u = warp; u < nqt; u += kDT / 32) {
            const uint32_t n = S.n[u];
            if (n + kDT > static_cast<uint32_t>(kDW) || t0 + kDT >= r_hi) {
                sort_list(S.s[u], S.id[u], n, lane);
                if (lane == 0) {
                    S.n[u] = min(n, k);
                    if (n >= k) S.L[u] = S.s[u][k - 1];
                }
            }
        }
        __syncthreads();
    }
    // this slab's sorted best k per query
    for (uint32_t u = 0; u < nqt; ++u) {
        const uint32_t n = S.n[u];
        const uint64_t o = (static_cast<uint64_t>(slab) * a.nq + q0 + u) * k;
        for (uint32_t i = tid; i < n; i += kDT) {
            a.part_ids[o + i] = S.id[u][i];
            a.part_scores[o + i] = S.s[u][i];
        }
        if (tid == 0) a.part_n[static_cast<uint64_t>(slab) * a.nq + q0 + u] = n;
    }
}

__global__ void __launch_bounds__(256) dense_merge_kernel(DenseArgs a) {
    const uint32_t q = blockIdx.x, k = a.k, G = a.n_slabs;
    auto at = [&](uint32_t g, uint32_t i) { return (static_cast<uint64_t>(g) * a.nq + q) * k + i; };
    uint32_t total = 0;
    for (uint32_t g = 0; g < G; ++g) total += a.part_n[static_cast<uint64_t>(g) * a.nq + q];
    for (uint32_t g = 0; g < G; ++g) {
        const uint32_t ng = a.part_n[static_cast<uint64_t>(g) * a.nq + q];
        for (uint32_t i = threadIdx.x; i < ng; i += blockDim.x) {
            const double s = a.part_scores[at(g, i)];
            const uint64_t id = a.part_ids[at(g, i)];
            uint32_t rank = i;
            for (uint32_t h = 0; h < G; ++h) {
                if (h == g) continue;
                uint32_t lo = 0, hi = a.part_n[static_cast<uint64_t>(h) * a.nq + q];
                while (lo < hi) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (better(a.part_scores[at(h, mid)], a.part_ids[at(h, mid)], s, id)) lo = mid + 1;
                    else hi = mid;
                }
                rank += lo;
            }
            if (rank < k) {
                a.out_ids[static_cast<uint64_t>(q) * k + rank] = id;
                a.out_scores[static_cast<uint64_t>(q) * k + rank] = s;
            }
        }
    }
    if (threadIdx.x == 0) a.out_n[q] = min(total, k);
}


// ------------------------------------------------------------ large k
__global__ void dense_scores_kernel(DenseDev ix, const double* q64, uint64_t* skey, uint32_t* rows) {
    const uint32_t row = blockIdx.x * blockDim.x + threadIdx.x;
    if (row >= ix.n) return;
    const float* r = ix.E + static_cast<uint64_t>(row) * ix.dim;
    double acc = 0.0;
    for (uint32_t j = 0; j < ix.dim; ++j) acc = __fma_rn(static_cast<double>(__ldg(r + j)), q64[j], acc);
    // order-preserving map to u64, complemented: ascending key = descending score
    const uint64_t b = static_cast<uint64_t>(__double_as_longlong(acc));
    const uint64_t ord = (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    skey[row] = ~ord;
    rows[row] = row;
}

__global__ void dense_gather_kernel(uint32_t n, const uint64_t* skey, const uint32_t* rows_by_id, uint64_t* key2) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) key2[i] = skey[rows_by_id[i]];
}

__global__ void dense_emit_kernel(DenseDev ix, uint32_t k, const uint32_t* rows, const uint64_t* key_sorted,
                                  uint64_t* out_ids, double* out_scores, uint32_t* out_n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < k) {
        const uint64_t ord = ~key_sorted[i];
        const uint64_t b = (ord >> 63) ? (ord & 0x7fffffffffffffffull) : ~ord;
        out_ids[i] = ix.ids[rows[i]];
        out_scores[i] = __longlong_as_double(static_cast<long long>(b));
    }
    if (i == 0) *out_n = k;
}

}  // namespace

uint32_t dense_max_k() { return kDenseMaxK; }

uint32_t dense_slabs(uint32_t nq, uint32_t n_rows, int sms) {
    // enough CTAs for every SM twice, slabs of at least a few tiles
    const uint32_t qtiles = (nq + kQT - 1) / kQT;
    uint32_t s = (2u * static_cast<uint32_t>(sms) + qtiles - 1) / qtiles;
    s = min(s, max(1u, n_rows / (4u * kDT)));
    return max(1u, min(s, 64u));
}

cudaError_t launch_dense(const DenseDev& ix, const DenseArgs& a, cudaStream_t st) {
    if (a.nq == 0) return cudaSuccess;
    const uint64_t nq_el = static_cast<uint64_t>(a.nq) * ix.dim;
    const uint64_t blocks = (nq_el + 255) / 256 < 4096 ? (nq_el + 255) / 256 : 4096;
    dense_q64_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(a.q_in, a.q64, nq_el);
    const size_t smem = sizeof(DenseSmem);
    cudaError_t e = cudaFuncSetAttribute(dense_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const dim3 grid((a.nq + kQT - 1) / kQT, a.n_slabs);
    dense_exact_kernel<<<grid, kDT, smem, st>>>(ix, a);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    dense_merge_kernel<<<a.nq, 256, 0, st>>>(a);
    return cudaGetLastError();
}

}  // namespace hm

namespace hm {

size_t dense_large_k_bytes(uint32_t n) {
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint64_t*)nullptr, (uint64_t*)nullptr, (const uint32_t*)nullptr,
                                    (uint32_t*)nullptr, static_cast<int>(n));
    b = a;
    const size_t el = static_cast<size_t>(n);
    return b + el * (8 + 8 + 8 + 4 + 4 + 4) + 6 * 256;
}

cudaError_t launch_dense_large_k(const DenseDev& ix, const double* q64, uint32_t k, void* scratch, size_t bytes,
                                 uint64_t* out_ids, double* out_scores, uint32_t* out_n, cudaStream_t st) {
    const uint32_t n = ix.n;
    auto carve = [&](size_t sz) {
        void* p = scratch;
        const size_t a = (sz + 255) & ~size_t(255);
        scratch = static_cast<char*>(scratch) + a;
        bytes -= a;
        return p;
    };
    uint64_t* skey = static_cast<uint64_t*>(carve(8ull * n));
    uint64_t* ids_sorted = static_cast<uint64_t*>(carve(8ull * n));
    uint64_t* key2 = static_cast<uint64_t*>(carve(8ull * n));
    uint32_t* rows = static_cast<uint32_t*>(carve(4ull * n));
    uint32_t* rows_by_id = static_cast<uint32_t*>(carve(4ull * n));
    uint32_t* rows_final = static_cast<uint32_t*>(carve(4ull * n));
    uint64_t* key_final = skey;  // reused after the gather
    size_t temp = bytes;
    const unsigned blocks = (n + 255) / 256;
    dense_scores_kernel<<<blocks, 256, 0, st>>>(ix, q64, skey, rows);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    e = cub::DeviceRadixSort::SortPairs(scratch, temp, ix.ids, ids_sorted, rows, rows_by_id, static_cast<int>(n), 0, 64,
                                        st);
    if (e != cudaSuccess) return e;
    dense_gather_kernel<<<blocks, 256, 0, st>>>(n, skey, rows_by_id, key2);
    temp = bytes;
    e = cub::DeviceRadixSort::SortPairs(scratch, temp, key2, key_final, rows_by_id, rows_final, static_cast<int>(n), 0,
                                        64, st);
    if (e != cudaSuccess) return e;
    dense_emit_kernel<<<(k + 255) / 256, 256, 0, st>>>(ix, k, rows_final, key_final, out_ids, out_scores, out_n);
    return cudaGetLastError();
}

__global__ void dense_q64_one(const float* q, double* q64, uint32_t n) {
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) q64[i] = static_cast<double>(q[i]);
}

cudaError_t launch_dense_widen(const float* q, double* q64, uint32_t n, cudaStream_t st) {
    dense_q64_one<<<1, 256, 0, st>>>(q, q64, n);
    return cudaGetLastError();
}

}  // namespace hm
