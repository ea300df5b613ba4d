// gather_merge_kernel: the all-gather + k-way merge of doc-sharded search
// (hm_sharded_*, host/hm_shard.cpp) fused into one kernel over peer memory.
//
// Every shard g left its exact local top-k lists in its own HBM
// (ids/scores [nq][k], n [nq], postings [nq]); with peer access enabled the
// root device's kernel reads them straight over NVLink (P2P loads through
// NVSwitch), so there is no separate gather copy.  One CTA per query:
//   1. the G lists of the query are staged into shared memory (coalesced
//      16-byte-per-entry reads from each peer) when G*k fits, else read in
//      place;
//   2. every entry's rank in the merged order is its own index plus, for each
//      other list, the number of that list's entries ranked before it (binary
//      search -- lists are sorted by (score desc, DocId asc),
//      include/hybrid/types.hpp:21-25).  A DocId lives in exactly one shard,
//      so ranks are distinct and the entries with rank < k ARE the global
//      top-k, in order: each is written to its slot, no sort;
//   3. Margin confidence from ranks 0 and 1 (src/cascade.cpp:15-21) and the
//      skip decision (src/cascade.cpp:79-84), postings_touched summed over the
//      shards (SearchStats accumulates, src/csr_index.cpp:102).
// Any k (no capacity limit: the in-place variant covers G*k beyond shared
// memory), any G <= kMaxShards.  The shards' scores are the flat index's bits
// (global idf / avgdl / order keys, SharedStats, csr_index.hpp:28-35), so the
// merged lists equal the single-device and reference answers.
#include <cstdint>

#include "hm_device.cuh"
#include "hm_launch.h"

namespace hm {

constexpr int kGMThreads = 256;
constexpr uint32_t kGMStageMax = 4096;  // staged entries: 64 KB of shared memory

// number of entries of list (s, d, n) ranked before (sa, ia)
// (with_equal: also the entries equal to it -- a DocId repeated across shards)
template <class S, class D>
__device__ __forceinline__ uint32_t count_before(const S* s, const D* d, uint32_t n, double sa, uint64_t ia,
                                                 bool with_equal) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (with_equal ? !better(sa, ia, s[mid], d[mid]) : better(s[mid], d[mid], sa, ia)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(kGMThreads) gather_merge_kernel(ShardLists L, uint32_t nq, uint32_t k, bool staged,
                                                                  const double* tau, double tau_default, double eps,
                                                                  uint64_t* out_ids, double* out_scores,
                                                                  uint32_t* out_n, double* out_conf,
                                                                  uint8_t* out_skip, uint64_t* out_post) {
    extern __shared__ __align__(16) unsigned char gm_smem[];
    __shared__ uint32_t s_n[kMaxShards + 1], s_base[kMaxShards + 1];
    __shared__ double s_top[2];
    const uint32_t G = L.G;
    for (uint32_t q = blockIdx.x; q < nq; q += gridDim.x) {
        if (threadIdx.x == 0) {
            uint32_t tot = 0;
            uint64_t post = 0;
            for (uint32_t g = 0; g < G; ++g) {
                const uint32_t n = min(L.n[g][q], k);
                s_n[g] = n;
                s_base[g] = tot;
                tot += n;
                if (L.post[g]) post += L.post[g][q];
            }
            s_base[G] = tot;
            s_top[0] = s_top[1] = 0.0;
            if (out_post) out_post[q] = post;
        }
        __syncthreads();
        const uint32_t tot = s_base[G];
        const uint64_t row = static_cast<uint64_t>(q) * k;
        double* st_sc = reinterpret_cast<double*>(gm_smem);
        uint64_t* st_id = reinterpret_cast<uint64_t*>(gm_smem + 8ull * kGMStageMax);
        if (staged) {  // the query's G lists -> shared memory, shard after shard
            for (uint32_t g = 0; g < G; ++g)
                for (uint32_t r = threadIdx.x; r < s_n[g]; r += kGMThreads) {
                    st_sc[s_base[g] + r] = L.scores[g][row + r];
                    st_id[s_base[g] + r] = L.ids[g][row + r];
                }
            __syncthreads();
        }
        for (uint32_t e = threadIdx.x; e < tot; e += kGMThreads) {
            uint32_t g = 0;
            while (e >= s_base[g + 1]) ++g;
            const uint32_t r = e - s_base[g];
            const double sa = staged ? st_sc[e] : L.scores[g][row + r];
            const uint64_t ia = staged ? st_id[e] : L.ids[g][row + r];
            uint32_t rank = r;
            for (uint32_t h = 0; h < G && rank < k; ++h) {
                if (h == g) continue;
                rank += staged ? count_before(st_sc + s_base[h], st_id + s_base[h], s_n[h], sa, ia, h < g)
                               : count_before(L.scores[h] + row, L.ids[h] + row, s_n[h], sa, ia, h < g);
            }
            if (rank < k) {
                out_ids[row + rank] = ia;
                out_scores[row + rank] = sa;
                if (rank < 2) s_top[rank] = sa;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const uint32_t nout = min(tot, k);
            out_n[q] = nout;
            double conf = 0.0;  // Margin (cascade.cpp:15-21): 0 with < 2 scores or s0 <= 0
            if (nout >= 2 && s_top[0] > 0.0) conf = __ddiv_rn(__dsub_rn(s_top[0], s_top[1]), fmax(s_top[0], eps));
            if (out_conf) out_conf[q] = conf;
            if (out_skip) out_skip[q] = conf >= (tau ? tau[q] : tau_default) ? 1 : 0;
        }
        __syncthreads();
    }
}

// Doc shards' bound exchange: per query the k-th largest of the G shards' k
// best seed scores ([G] pointers to [nq][k], read over peer memory) -- a k-th
// score of real documents of the union, hence a lower bound on its k-th score.
constexpr int kBKThreads = 128;
__global__ void __launch_bounds__(kBKThreads) bound_kth_kernel(BoundLists L, uint32_t nq, uint32_t k, float* out) {
    __shared__ float v[kMaxShards * kMaxK];
    __shared__ uint32_t hist[256], sel[2];
    for (uint32_t q = blockIdx.x; q < nq; q += gridDim.x) {
        const uint32_t n = L.G * k;
        for (uint32_t i = threadIdx.x; i < n; i += kBKThreads) v[i] = L.b[i / k][static_cast<uint64_t>(q) * k + i % k];
        __syncthreads();
        const float x = block_kth_largest<kBKThreads>(v, n, k, hist, sel, [] { __syncthreads(); });
        if (threadIdx.x == 0) out[q] = x;
        __syncthreads();
    }
}

cudaError_t launch_bound_kth(const BoundLists& L, uint32_t nq, uint32_t k, float* out, cudaStream_t st) {
    if (nq == 0) return cudaSuccess;
    if (L.G == 0 || L.G > static_cast<uint32_t>(kMaxShards) || k == 0 || k > static_cast<uint32_t>(kMaxK))
        return cudaErrorInvalidValue;
    bound_kth_kernel<<<nq < 4096u ? nq : 4096u, kBKThreads, 0, st>>>(L, nq, k, out);
    return cudaGetLastError();
}

cudaError_t launch_gather_merge(const ShardLists& L, uint32_t nq, uint32_t k, const double* tau, double tau_default,
                                double eps, uint64_t* out_ids, double* out_scores, uint32_t* out_n,
                                double* out_conf, uint8_t* out_skip, uint64_t* out_post, cudaStream_t st) {
    if (nq == 0) return cudaSuccess;
    if (L.G == 0 || L.G > static_cast<uint32_t>(kMaxShards)) return cudaErrorInvalidValue;
    const bool staged = static_cast<uint64_t>(L.G) * k <= kGMStageMax;
    const size_t smem = staged ? 16ull * kGMStageMax : 0;
    static bool attr = false;
    if (staged && !attr) {
        const cudaError_t e = cudaFuncSetAttribute(gather_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                   static_cast<int>(16 * kGMStageMax));
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const uint32_t grid = nq < 4096u ? nq : 4096u;
    gather_merge_kernel<<<grid, kGMThreads, smem, st>>>(L, nq, k, staged, tau, tau_default, eps, out_ids, out_scores,
                                                         out_n, out_conf, out_skip, out_post);
    return cudaGetLastError();
}

}  // namespace hm
