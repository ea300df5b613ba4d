// sm_100a kernels of the batched BM25 search path (besides the fused
// selection kernel in search_pipe.cu):
//
//   plan_kernel    make_plan (src/csr_index.cpp:31-48) per query, on device,
//                  plus the LPT cost (sum of df) used to order the batch
//   exact_kernel   fp64 accumulation strictly in plan order for queries that
//                  cannot use the fp32 selection (candidate flood,
//                  non-positive idf, b outside [0,1], HM_FLAG_FORCE_EXACT)
//   merge_kernel   k-way merge of per-shard top-k lists (multi-GPU)
//
// Exactness argument of the fp32 selection used by search_pipe.cu.
// With positive contributions, every fp32 score A(d) is within relative
// delta = (m+10)*2^-24 of the fp64 score E(d).  L is always the k-th largest A
// over a set of real documents, so L <= a_k, the final k-th largest A.  A tile
// emits every doc with A >= L*(1-2.5*delta), a superset of
// {A >= a_k*(1-2.5*delta)}.  Any doc of the exact top-k (exact ties included)
// has  A >= (1-delta) e_k >= a_k (1-delta)/(1+delta) >= a_k (1-2.5*delta),
// so the survivors {A >= a_k (1-2.5 delta)} contain the exact top-k, and
// rescoring them in fp64 in the reference's order makes ids and scores
// bit-identical to the reference.
#include <cub/cub.cuh>

#include "hm_device.cuh"
#include "hm_launch.h"

namespace hm {

// ============================================================ planner
__global__ void plan_kernel(DevIndex ix, BatchArgs a, uint32_t* order_in) {
    uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= a.nq) return;
    const uint32_t lo = a.q_off[q], hi = a.q_off[q + 1];
    uint32_t* pt = a.plan_tid + lo;
    uint32_t* pm = a.plan_mult + lo;
    uint32_t m = 0;
    for (uint32_t i = lo; i < hi; ++i) {
        uint32_t t = a.q_tid[i];
        if (t == kNoTerm || t >= ix.n_terms) continue;  // unknown: dropped (:35-36)
        uint32_t j = 0;
        while (j < m && pt[j] != t) ++j;
        if (j == m) {
            pt[m] = t;
            pm[m] = 1;
            ++m;
        } else {
            ++pm[j];
        }
    }
    // canonical order: order key descending, ties by ascending tid (:40-46)
    for (uint32_t i = 1; i < m; ++i) {
        uint32_t t = pt[i], mu = pm[i];
        double kt = ix.order_key[t];
        int j = static_cast<int>(i) - 1;
        while (j >= 0) {
            uint32_t u = pt[j];
            double ku = ix.order_key[u];
            bool u_first = (ku != kt) ? (ku > kt) : (u < t);
            if (u_first) break;
            pt[j + 1] = u;
            pm[j + 1] = pm[j];
            --j;
        }
        pt[j + 1] = t;
        pm[j + 1] = mu;
    }
    uint64_t c = 0, cs = 0;
    for (uint32_t i = 0; i < m; ++i) {
        const uint64_t df = ix.term_off[pt[i] + 1] - ix.term_off[pt[i]];
        c += df;
        if (df <= kSeedScratch / 2) cs += df;
    }
    a.plan_len[q] = m;
    a.cost[q] = c;
    if (a.cost_seed) a.cost_seed[q] = cs;
    if (m >= kNeMinTerms && m <= 32) atomicAdd(&a.counters[8], 1u);  // the essential-term sweep has work
    order_in[q] = q;
}

// ============================================================ exact kernel
// One CTA per SM.  fp64 accumulators for one kTile-row tile (128 KB); every
// plan term is applied in plan order with a barrier in between, each doc's
// contributions are added `mult` times in sequence (src/csr_index.cpp:87-101),
// so every accumulated score is the reference's bit pattern.  Candidates are
// ranked by the composite key (score desc, DocId asc) -- a strict total order,
// so no slack is needed; the list keeps the best k.
constexpr int kExactThreads = 512;

struct __align__(16) ExactSmem {
    double acc[kTile];
    double cand_E[kExactCap];
    uint64_t cand_id[kExactCap];
    uint32_t cand_row[kExactCap];
    uint64_t t_start[kMaxTerms], t_wlo[kMaxTerms], t_end[kMaxTerms], t_cur[kMaxTerms],
        t_cur0[kMaxTerms], t_seg[kMaxTerms];
    double t_idf[kMaxTerms];
    uint32_t t_mult[kMaxTerms];
    int32_t t_slot[kMaxTerms];
    uint32_t code_tf[kMaxCodes], code_len[kMaxCodes];
    uint64_t post;
    double LE;
    uint64_t Lid;
    uint32_t q, n_c, ovf, haveL;
};

__device__ __forceinline__ void exact_sync() { __syncthreads(); }

// sort the exact list, keep the best `keep` entries, set L to the last kept
__device__ void exact_sort_keep(ExactSmem& S, uint32_t keep) {
    const uint32_t nc = min(S.n_c, static_cast<uint32_t>(kExactCap));
    const uint32_t n2 = pow2_ceil(nc);
    for (uint32_t i = nc + threadIdx.x; i < n2; i += kExactThreads) {
        S.cand_E[i] = -INFINITY;
        S.cand_id[i] = ~0ull;
        S.cand_row[i] = 0;
    }
    __syncthreads();
    block_bitonic<kExactThreads>(S.cand_E, S.cand_id, S.cand_row, n2, exact_sync);
    if (threadIdx.x == 0) {
        const uint32_t nk = min(nc, keep);
        S.n_c = nk;
        if (nk == keep && keep > 0) {
            S.haveL = 1;
            S.LE = S.cand_E[nk - 1];
            S.Lid = S.cand_id[nk - 1];
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kExactThreads, 1) exact_kernel(DevIndex ix, BatchArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ExactSmem& S = *reinterpret_cast<ExactSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31;
    const uint32_t cb = ix.code_bits;
    const double k1 = a.k1, bb = a.b;
    for (int i = tid; i < kTile; i += kExactThreads) S.acc[i] = 0.0;
    for (int i = tid; i < kMaxCodes; i += kExactThreads) {
        S.code_tf[i] = ix.code_tf[i];
        S.code_len[i] = ix.code_len[i];
    }
    for (;;) {
        __syncthreads();
        if (tid == 0) {
            const uint32_t w = atomicAdd(&a.counters[2], 1u);
            S.q = w < a.counters[1] ? a.exact_list[w] : kNoTerm;
        }
        __syncthreads();
        const uint32_t q = S.q;
        if (q == kNoTerm) break;
        uint32_t qr, row_lo, row_hi;  // the real query and this (slab) query's rows
        query_window(a, q, qr, row_lo, row_hi);
        const uint32_t poff = a.q_off[qr];
        const uint32_t m = a.plan_len[qr];
        const uint32_t k = a.k;
        if (tid < static_cast<int>(m)) {
            const uint32_t t = a.plan_tid[poff + tid];
            const int32_t slot = ix.long_slot[t];
            const uint64_t s0 = ix.term_off[t], s1 = ix.term_off[t + 1];
            const uint64_t w0 = row_lo > 0 ? first_at_or_after(ix, slot, s0, s1, row_lo) : s0;
            const uint64_t w1 = row_hi < ix.n_docs ? first_at_or_after(ix, slot, s0, s1, row_hi) : s1;
            S.t_start[tid] = s0;
            S.t_wlo[tid] = w0;
            S.t_end[tid] = w1;
            S.t_cur[tid] = w0;
            S.t_slot[tid] = slot;
            S.t_idf[tid] = ix.idf[t];
            S.t_mult[tid] = a.plan_mult[poff + tid];
        }
        __syncthreads();
        if (tid == 0) {
            uint64_t post = 0;
            for (uint32_t i = 0; i < m; ++i) post += S.t_end[i] - S.t_wlo[i];
            S.post = post;
            S.n_c = 0;
            S.haveL = 0;
            S.ovf = 0;
        }
        __syncthreads();
        if (m > 0 && k > 0 && row_hi > row_lo) {
            const uint32_t j0 = row_lo >> kTileShift, j1 = (row_hi - 1) >> kTileShift;
            for (uint32_t j = j0; j <= j1; ++j) {
                const uint32_t base = j << kTileShift;
                const uint32_t R0 = max(base, row_lo);
                const uint32_t R1 = min(base + kTile, row_hi);
                const uint32_t rlo = R0 - base, rn = R1 - R0;
                if (tid < static_cast<int>(m)) {
                    if (S.t_slot[tid] >= 0) {
                        const uint32_t* tb = tile_row(ix, S.t_slot[tid]);
                        S.t_cur0[tid] = S.t_start[tid] + __ldg(tb + j * kSubPerTile);
                        S.t_seg[tid] = S.t_start[tid] + __ldg(tb + (j + 1) * kSubPerTile);
                    } else {
                        const uint64_t c = S.t_cur[tid];
                        S.t_cur0[tid] = c;
                        const uint64_t lim = min(S.t_end[tid], c + static_cast<uint64_t>(rn));
                        S.t_seg[tid] = lower_bound_row(ix.post, c, lim, R1, cb);
                    }
                }
                for (int attempt = 0;; ++attempt) {
                    __syncthreads();
                    for (uint32_t i = 0; i < m; ++i) {  // plan order (:87-101)
                        const uint64_t b = S.t_cur0[i], e = S.t_seg[i];
                        const double idf = S.t_idf[i];
                        const uint32_t mu = S.t_mult[i];
                        const bool lng = S.t_slot[i] >= 0;
                        for (uint64_t x = b + tid; x < e; x += kExactThreads) {
                            const uint32_t p = __ldg(ix.post + x);
                            uint32_t local, code;
                            bool esc;
                            if (lng) {
                                local = p >> kCodeBitsLong;
                                if (local - rlo >= rn) continue;
                                code = p & kEscLong;
                                esc = code >= ix.n_codes;
                            } else {
                                local = (p >> cb) - base;
                                code = p & ix.esc_short;
                                esc = code >= ix.n_codes_short;
                            }
                            double tf, dl;
                            if (!esc) {
                                tf = S.code_tf[code];
                                dl = S.code_len[code];
                            } else {
                                tf = __ldg(ix.tf + x);
                                dl = __ldg(ix.doc_lens + base + local);
                            }
                            const double s = bm25_exact(tf, idf, dl, ix.avgdl, k1, bb);
                            double v = S.acc[local];
                            for (uint32_t r = 0; r < mu; ++r) v = __dadd_rn(v, s);
                            S.acc[local] = v;
                        }
                        __syncthreads();
                    }
                    // scan: docs not worse than L (composite key) join the list
                    const bool haveL = S.haveL;
                    const double LE = S.LE;
                    const uint64_t Lid = S.Lid;
                    for (uint32_t rb = rlo; rb < rlo + rn; rb += kExactThreads) {
                        const uint32_t r = rb + tid;
                        double E = 0.0;
                        if (r < rlo + rn) {
                            E = S.acc[r];
                            S.acc[r] = 0.0;
                        }
                        bool qual = false;
                        uint64_t id = 0;
                        if (E > 0.0) {
                            id = __ldg(ix.doc_ids + base + r);
                            qual = !haveL || !better(LE, Lid, E, id);
                        }
                        const uint32_t bal = __ballot_sync(0xffffffffu, qual);
                        if (bal) {
                            uint32_t bse = 0;
                            if (lane == 0) bse = atomicAdd(&S.n_c, __popc(bal));
                            bse = __shfl_sync(0xffffffffu, bse, 0);
                            if (lane == 0 && bse + __popc(bal) > kExactCap) S.ovf = 1;
                            const uint32_t slot = bse + __popc(bal & ((1u << lane) - 1));
                            if (qual && slot < kExactCap) {
                                S.cand_E[slot] = E;
                                S.cand_id[slot] = id;
                                S.cand_row[slot] = base + r;
                            }
                        }
                    }
                    __syncthreads();
                    if (!S.ovf) break;
                    // overflow: tighten L on the partial list, drop this tile's
                    // entries, redo the tile
                    exact_sort_keep(S, k);
                    if (tid == 0) {
                        uint32_t w = 0;
                        for (uint32_t i = 0; i < S.n_c; ++i) {
                            const uint32_t row = S.cand_row[i];
                            if (row >= R0 && row < R1) continue;
                            S.cand_E[w] = S.cand_E[i];
                            S.cand_id[w] = S.cand_id[i];
                            S.cand_row[w] = row;
                            ++w;
                        }
                        S.n_c = w;
                        S.ovf = 0;
                        if (attempt > 64) atomicOr(&a.counters[3], kErrNoConverge);
                    }
                    if (attempt > 64) break;
                }
                if (tid < static_cast<int>(m) && S.t_slot[tid] < 0) S.t_cur[tid] = S.t_seg[tid];
                __syncthreads();
                if (S.n_c > kExactCap / 2) exact_sort_keep(S, k);
            }
            exact_sort_keep(S, k);
        }
        if (tid == 0) {
            uint32_t nout = 0;
            for (uint32_t i = 0; i < S.n_c && nout < k; ++i) {
                if (!(S.cand_E[i] > 0.0)) break;
                a.out_ids[static_cast<uint64_t>(q) * k + nout] = S.cand_id[i];
                a.out_scores[static_cast<uint64_t>(q) * k + nout] = S.cand_E[i];
                ++nout;
            }
            a.out_n[q] = nout;
            if (a.out_post) a.out_post[q] = S.post;
            write_decision(a, q, S.cand_E, nout);
        }
    }
}

// ============================================================ shard merge
constexpr int kMergeThreads = 256;
constexpr int kMergeMax = 2048;

// number of entries of the sorted list (s, d, n) ranked before (sa, ia)
// (with_equal: also the entries equal to it)
__device__ __forceinline__ uint32_t merge_count_before(const double* s, const uint64_t* d, uint32_t n, double sa,
                                                       uint64_t ia, bool with_equal) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (with_equal ? !better(sa, ia, s[mid], d[mid]) : better(s[mid], d[mid], sa, ia)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// The G sorted lists of a query (slabs of a split batch: disjoint row ranges,
// so every DocId appears once) staged in shared memory; every entry's rank in
// the merged order is its index plus, per other list, the entries ranked
// before it (binary search) -- the entries of rank < k are the top k, each
// written straight to its slot (no sort; as gather_merge_kernel, shard_merge.cu).
__global__ void __launch_bounds__(kMergeThreads) merge_kernel(
    uint32_t G, uint32_t nq, uint32_t k, const uint64_t* ids, const double* scores,
    const uint32_t* n, const double* tau, double tau_default, double eps, uint64_t* out_ids,
    double* out_scores, uint32_t* out_n, double* out_conf, uint8_t* out_skip) {
    __shared__ double sc[kMergeMax];
    __shared__ uint64_t id[kMergeMax];
    __shared__ uint16_t s_n[kMergeMax + 1], s_base[kMergeMax + 2];  // G <= G * k <= kMergeMax
    __shared__ double s_top[2];
    const uint32_t q = blockIdx.x;
    if (threadIdx.x == 0) {
        uint32_t tot = 0;
        for (uint32_t g = 0; g < G; ++g) {
            const uint32_t m = min(n[static_cast<uint64_t>(g) * nq + q], k);
            s_n[g] = static_cast<uint16_t>(m);
            s_base[g] = static_cast<uint16_t>(tot);
            tot += m;
        }
        s_base[G] = static_cast<uint16_t>(tot);
        s_top[0] = s_top[1] = 0.0;
    }
    __syncthreads();
    const uint32_t tot = s_base[G];
    for (uint32_t e = threadIdx.x; e < G * k; e += kMergeThreads) {
        const uint32_t g = e / k, r = e % k;
        if (r < s_n[g]) {
            const uint64_t o = (static_cast<uint64_t>(g) * nq + q) * k + r;
            sc[s_base[g] + r] = scores[o];
            id[s_base[g] + r] = ids[o];
        }
    }
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < tot; e += kMergeThreads) {
        uint32_t g = 0, hi = G;  // the list holding e: largest g with s_base[g] <= e (and a nonempty list)
        while (hi - g > 1) {
            const uint32_t mid = (g + hi) >> 1;
            if (s_base[mid] <= e) g = mid;
            else hi = mid;
        }
        const uint32_t r = e - s_base[g];
        const double sa = sc[e];
        const uint64_t ia = id[e];
        uint32_t rank = r;
        for (uint32_t h = 0; h < G && rank < k; ++h)  // (equal pairs -- a repeated DocId -- by list)
            if (h != g) rank += merge_count_before(sc + s_base[h], id + s_base[h], s_n[h], sa, ia, h < g);
        if (rank < k) {
            out_ids[static_cast<uint64_t>(q) * k + rank] = ia;
            out_scores[static_cast<uint64_t>(q) * k + rank] = sa;
            if (rank < 2) s_top[rank] = sa;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t nout = min(tot, k);  // (the lists hold positive scores only)
        out_n[q] = nout;
        double conf = 0.0;
        if (nout >= 2 && s_top[0] > 0.0) conf = __ddiv_rn(__dsub_rn(s_top[0], s_top[1]), fmax(s_top[0], eps));
        const double t = tau ? tau[q] : tau_default;
        if (out_conf) out_conf[q] = conf;
        if (out_skip) out_skip[q] = conf >= t ? 1 : 0;
    }
}

// ============================================================ split batches
// LPT order of slab queries: every slab of the i-th most expensive real query
__global__ void expand_order_kernel(uint32_t nq_real, uint32_t split, const uint32_t* order_real, uint32_t* order) {
    const uint32_t v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= nq_real * split) return;
    const uint32_t i = v / split, s = v % split;
    order[v] = s * nq_real + order_real[i];
}

// postings_touched of a real query = the sum over its slab queries
__global__ void sum_slab_postings_kernel(uint32_t nq_real, uint32_t split, const uint64_t* v_post,
                                         uint64_t* out_post) {
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq_real) return;
    uint64_t t = 0;
    for (uint32_t s = 0; s < split; ++s) t += v_post[static_cast<uint64_t>(s) * nq_real + q];
    out_post[q] = t;
}

// ============================================================ launchers
cudaError_t launch_plan(const DevIndex& ix, const BatchArgs& a, uint32_t* order_in,
                        cudaStream_t st) {
    if (a.nq == 0) return cudaSuccess;
    plan_kernel<<<(a.nq + 127) / 128, 128, 0, st>>>(ix, a, order_in);
    return cudaGetLastError();
}

cudaError_t launch_expand_order(uint32_t nq_real, uint32_t split, const uint32_t* order_real, uint32_t* order,
                                cudaStream_t st) {
    const uint32_t n = nq_real * split;
    if (n == 0) return cudaSuccess;
    expand_order_kernel<<<(n + 255) / 256, 256, 0, st>>>(nq_real, split, order_real, order);
    return cudaGetLastError();
}

cudaError_t launch_sum_slab_postings(uint32_t nq_real, uint32_t split, const uint64_t* v_post, uint64_t* out_post,
                                     cudaStream_t st) {
    if (nq_real == 0 || !out_post) return cudaSuccess;
    sum_slab_postings_kernel<<<(nq_real + 255) / 256, 256, 0, st>>>(nq_real, split, v_post, out_post);
    return cudaGetLastError();
}

cudaError_t lpt_sort_bytes(uint32_t nq, size_t* bytes) {
    *bytes = 0;
    return cub::DeviceRadixSort::SortPairsDescending(nullptr, *bytes, (const uint64_t*)nullptr,
                                                     (uint64_t*)nullptr, (const uint32_t*)nullptr,
                                                     (uint32_t*)nullptr, static_cast<int>(nq));
}

cudaError_t launch_lpt_sort(void* temp, size_t bytes, const BatchArgs& a, uint64_t* cost_sorted,
                            const uint32_t* order_in, int key_bits, cudaStream_t st) {
    if (a.nq == 0) return cudaSuccess;
    return cub::DeviceRadixSort::SortPairsDescending(temp, bytes, a.cost, cost_sorted, order_in,
                                                     a.order, static_cast<int>(a.nq), 0, key_bits, st);
}

cudaError_t launch_seed_sort(void* temp, size_t bytes, const BatchArgs& a, uint64_t* cost_sorted,
                             const uint32_t* order_in, uint32_t* order_seed, int key_bits, cudaStream_t st) {
    if (a.nq == 0) return cudaSuccess;
    return cub::DeviceRadixSort::SortPairsDescending(temp, bytes, a.cost_seed, cost_sorted, order_in, order_seed,
                                                     static_cast<int>(a.nq), 0, key_bits, st);
}

static bool g_exact_attr = false;

cudaError_t launch_exact(const DevIndex& ix, const BatchArgs& a, int grid, cudaStream_t st) {
    if (!g_exact_attr) {
        cudaError_t e = cudaFuncSetAttribute(exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(sizeof(ExactSmem)));
        if (e != cudaSuccess) return e;
        g_exact_attr = true;
    }
    exact_kernel<<<grid, kExactThreads, sizeof(ExactSmem), st>>>(ix, a);
    return cudaGetLastError();
}

cudaError_t launch_merge(uint32_t G, uint32_t nq, uint32_t k, const uint64_t* ids,
                         const double* scores, const uint32_t* n, const double* tau,
                         double tau_default, double eps, uint64_t* out_ids, double* out_scores,
                         uint32_t* out_n, double* out_conf, uint8_t* out_skip, cudaStream_t st) {
    if (nq == 0) return cudaSuccess;
    if (static_cast<uint64_t>(G) * k > kMergeMax) return cudaErrorInvalidValue;
    merge_kernel<<<nq, kMergeThreads, 0, st>>>(G, nq, k, ids, scores, n, tau, tau_default, eps,
                                               out_ids, out_scores, out_n, out_conf, out_skip);
    return cudaGetLastError();
}

cudaError_t search_occupancy(int* sb, int* eb) {
    cudaError_t e = search_occupancy_fast(sb);
    if (e != cudaSuccess) return e;
    if (!g_exact_attr) {
        e = cudaFuncSetAttribute(exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(sizeof(ExactSmem)));
        if (e != cudaSuccess) return e;
        g_exact_attr = true;
    }
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(eb, exact_kernel, kExactThreads, sizeof(ExactSmem));
}

}  // namespace hm
