// bridge_kernel: learned-sparse ("bridge") top-k on sm_100a.
//
// The reference's bridge scoring (src/bridge.cpp:112-137) accumulates
// S[doc] += w_q * W_t per posting, in ascending query term-id order, in fp64,
// and that order is a bit-exactness contract (bridge.hpp:30-33, the
// brute-force oracle of test_bridge.cpp:31-51 and acceptance criterion 5,
// acceptance.cpp:232-278).  Unlike BM25 there is no (tf, len) structure to
// bake, so this kernel scores EXACTLY in fp64 and needs no rescoring pass:
//
//   * persistent CTAs of 8 warps; a CTA owns one query at a time;
//   * the query's row window is split into 8 contiguous spans, one per warp;
//     a warp sweeps its span in 1,024-row units with a private fp64
//     accumulator slice in shared memory (8 KB), so no other thread ever
//     touches its rows: no atomics and no barriers inside the sweep;
//   * per unit the warp walks the query's terms in ascending term-id order
//     (the contract): lane j keeps term j's posting cursor in a register,
//     one ballot finds the terms with postings in the unit, and each such
//     term's postings are applied by the 32 lanes (rows ascend within a term,
//     so the unit's postings are a prefix from the cursor) with
//     acc = acc + (w_q * W) rounded separately (__dmul_rn/__dadd_rn, no FMA:
//     the reference is built without contraction);
//   * after a unit the warp scans its 1,024 accumulators, zeroes them, and
//     appends rows with S > 0 and S >= the running threshold to its candidate
//     list (collect keeps S > 0 only, bridge.cpp:100-108).  A full list is
//     pruned to its best k by (score desc, DocId asc) (RankedList::better,
//     include/hybrid/types.hpp:21-25); the k-th score becomes the warp's bound
//     and, through an atomicMax, the CTA's;
//   * at the end of the query the 8 sorted lists are merged by rank.
// Scores are exact, so the bound needs no slack: a document of the final
// top-k always has S >= any list's k-th score.
#include <cstdint>

#include "hm_bridge.h"

namespace hm {
namespace {

constexpr int kBrWarps = 8;
constexpr int kBrThreads = kBrWarps * 32;
constexpr uint32_t kBrUnit = 1024;  // rows per warp unit (8 KB of fp64)
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr int kRegGroups = 4;       // cursors of the first 128 terms live in registers
#ifndef HM_BR_BATCH
#define HM_BR_BATCH 6  // terms whose first chunk is loaded together
#endif
#ifndef HM_BR_RUN
#define HM_BR_RUN 8    // chunks in flight in a dense run
#endif

__device__ __forceinline__ bool better(double sa, uint64_t ia, double sb, uint64_t ib) {
    return sa > sb || (sa == sb && ia < ib);
}

template <int W>
struct BridgeSmem {
    double acc[kBrWarps][kBrUnit];
    double cs[kBrWarps][W];     // candidate scores
    uint64_t ci[kBrWarps][W];   // candidate DocIds
    uint32_t nw[kBrWarps];
    unsigned long long Lg;      // CTA bound: max over warps of their k-th score (bits)
    uint32_t q, m;
    unsigned long long post;
};

// Keep the best min(n, k) entries of warp list (s, id), sorted by
// (score desc, DocId asc): an in-place bitonic sort of the W slots (the n
// live entries padded with -inf sentinels), 32 lanes per compare-exchange
// stage, no scratch and no register arrays.
template <int W>
__device__ uint32_t prune_list(double* s, uint64_t* id, uint32_t n, uint32_t k, int lane) {
    static_assert((W & (W - 1)) == 0, "bitonic lists are a power of two");
    for (uint32_t i = n + lane; i < static_cast<uint32_t>(W); i += 32) {
        s[i] = -__longlong_as_double(0x7ff0000000000000ll);
        id[i] = ~0ull;
    }
    __syncwarp();
    for (uint32_t size = 2; size <= static_cast<uint32_t>(W); size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t t = lane; t < static_cast<uint32_t>(W) / 2; t += 32) {
                const uint32_t i = 2 * t - (t & (stride - 1)), j = i + stride;
                const double si = s[i], sj = s[j];
                const uint64_t ii = id[i], ij = id[j];
                const bool first = (i & size) == 0;  // this block ascends in rank
                if (first ? better(sj, ij, si, ii) : better(si, ii, sj, ij)) {
                    s[i] = sj;
                    s[j] = si;
                    id[i] = ij;
                    id[j] = ii;
                }
            }
            __syncwarp();
        }
    return n < k ? n : k;
}

template <int W>
__global__ void __launch_bounds__(kBrThreads) bridge_kernel(BridgeDev ix, BridgeArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    BridgeSmem<W>& S = *reinterpret_cast<BridgeSmem<W>*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t k = a.k;
    const uint32_t mstride = a.m_max;
    // per-CTA scratch: t_beg, t_end, t_wq [m_max], cursors [8][m_max], peeks [8][m_max]
    // (cursors/peeks of terms beyond the first 128 of a query; the rest live in registers)
    uint64_t* const t_beg = a.scratch + static_cast<uint64_t>(blockIdx.x) * (3 + 2 * kBrWarps) * mstride;
    uint64_t* const t_end = t_beg + mstride;
    double* const t_wq = reinterpret_cast<double*>(t_end + mstride);
    uint64_t* const cur_g = t_end + 2 * mstride + static_cast<uint64_t>(warp) * mstride;
    uint64_t* const pk_g = cur_g + static_cast<uint64_t>(kBrWarps) * mstride;
    double* const acc = S.acc[warp];

    for (uint32_t i = lane; i < kBrUnit; i += 32) acc[i] = 0.0;
    if (tid < kBrWarps) S.nw[tid] = 0;
    if (tid == 0) S.Lg = 0ull;

    for (;;) {
        __syncthreads();
        if (tid == 0) S.q = atomicAdd(&a.counters[0], 1u);
        __syncthreads();
        const uint32_t q = S.q;
        if (q >= a.nq) break;
        // small batches: query q is the (q / nq_real)-th row slab of real
        // query q % nq_real (merged afterwards like doc shards)
        const uint32_t qr = a.split > 1 ? q % a.nq_real : q;
        uint32_t row_lo = a.row_lo, row_hi = a.row_hi;
        if (a.split > 1) {
            const uint64_t sp = a.row_hi - a.row_lo, s = q / a.nq_real;
            row_lo = a.row_lo + static_cast<uint32_t>(sp * s / a.split);
            row_hi = a.row_lo + static_cast<uint32_t>(sp * (s + 1) / a.split);
        }
        // ---- the query's known terms, in its (ascending) order (bridge.cpp:120-123)
        if (warp == 0) {
            const uint64_t o0 = a.q_off[qr], o1 = a.q_off[qr + 1];
            uint32_t cnt = 0;
            // (device batches: a query longer than m_max is refused, n = 0 and
            // postings = ~0; the host entry point sizes m_max itself)
            for (uint64_t b0 = o0; b0 < o1 && o1 - o0 <= mstride; b0 += 32) {
                const uint64_t i = b0 + lane;
                const uint32_t t = i < o1 ? a.q_idx[i] : kNone;
                const bool ok = t < ix.n_terms;
                const uint32_t bal = __ballot_sync(0xffffffffu, ok);
                if (ok) {
                    const uint32_t pos = cnt + __popc(bal & ((1u << lane) - 1u));
                    t_beg[pos] = ix.term_off[t];
                    t_end[pos] = ix.term_off[t + 1];
                    t_wq[pos] = a.q_val[i];
                }
                cnt += __popc(bal);
            }
            if (lane == 0) {
                S.m = o1 - o0 <= mstride ? cnt : kNone;
                S.post = 0ull;
            }
        }
        __syncthreads();
        const uint32_t m = S.m;
        if (m == 0 || m == kNone || row_hi <= row_lo) {
            if (tid == 0) {
                a.out_n[q] = 0;
                if (a.out_post) a.out_post[q] = m == kNone ? ~0ull : 0ull;
            }
            continue;
        }
        // ---- my span of the window, and each term's cursor at its start
        const uint32_t span = row_hi - row_lo;
        const uint32_t lo_w = row_lo + static_cast<uint32_t>((static_cast<uint64_t>(span) * warp) / kBrWarps);
        const uint32_t hi_w = row_lo + static_cast<uint32_t>((static_cast<uint64_t>(span) * (warp + 1)) / kBrWarps);
        auto lower_bound = [&](uint64_t lo, uint64_t hi, uint32_t row) {
            while (lo < hi) {
                const uint64_t mid = (lo + hi) >> 1;
                if (ix.rows[mid] < row) lo = mid + 1;
                else hi = mid;
            }
            return lo;
        };
        // lane j of group g: term 32g + j's cursor (first posting at or after the
        // current unit), the end of its postings in my span, and the row at the
        // cursor ("peek", kNone when exhausted) -- carried across units, so a
        // unit costs no load for the terms without postings in it
        uint64_t creg[kRegGroups], ereg[kRegGroups];
        uint32_t preg[kRegGroups];
        unsigned long long post = 0;  // postings of my span (SearchStats, bridge.cpp:133)
#pragma unroll
        for (int g = 0; g < kRegGroups; ++g) {
            creg[g] = ereg[g] = 0;
            preg[g] = kNone;
        }
        for (uint32_t g = 0; g * 32 < m; ++g) {
            const uint32_t j = g * 32 + lane;
            if (j < m) {
                const uint64_t b = t_beg[j], e = t_end[j];
                const uint64_t c = lo_w == 0 ? b : lower_bound(b, e, lo_w);
                const uint64_t d = hi_w >= ix.n_docs ? e : lower_bound(c, e, hi_w);
                const uint32_t pk = c < d ? __ldg(ix.rows + c) : kNone;
                post += d - c;
                if (g < kRegGroups) {
#pragma unroll
                    for (int u = 0; u < kRegGroups; ++u)
                        if (u == static_cast<int>(g)) {
                            creg[u] = c;
                            ereg[u] = d;
                            preg[u] = pk;
                        }
                } else {
                    cur_g[j] = c;
                    pk_g[j] = pk;
                }
            }
        }
        if (post) atomicAdd(&S.post, post);
        if (k == 0) {  // nothing to rank; SearchStats still counts (bridge.cpp:133)
            __syncthreads();
            if (tid == 0) {
                a.out_n[q] = 0;
                if (a.out_post) a.out_post[q] = S.post;
            }
            continue;
        }
        // a term group's walk over one unit: apply every term with postings in
        // [ub, uhi), in ascending order
        uint32_t nw = S.nw[warp];
        double Lw = 0.0;
        // Terms are applied in ascending order, but their loads are not
        // serialised: the first 32 postings of up to kBatch active terms are
        // loaded together, and a term with more postings in the unit continues
        // 4 chunks (128 postings) at a time.  The row that ends a term's run
        // is its next peek.
        auto walk_group = [&](uint32_t g, uint64_t& c, uint32_t& pk, uint64_t e, uint32_t ub, uint32_t uhi) {
            constexpr int kBatch = HM_BR_BATCH;
            constexpr int kRun = HM_BR_RUN;
            uint32_t act = __ballot_sync(0xffffffffu, pk < uhi);
            while (act) {
                int ti[kBatch];
                uint64_t cb[kBatch], eb[kBatch];
                uint32_t rr[kBatch];
                double ww[kBatch];
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    ti[u] = -1;
                    if (act) {
                        ti[u] = __ffs(act) - 1;
                        act &= act - 1;
                    }
                    const int src = ti[u] < 0 ? 0 : ti[u];
                    cb[u] = __shfl_sync(0xffffffffu, c, src);
                    eb[u] = __shfl_sync(0xffffffffu, e, src);
                    rr[u] = kNone;
                    ww[u] = 0.0;
                    const uint64_t p = cb[u] + lane;
                    if (ti[u] >= 0 && p < eb[u]) {
                        rr[u] = __ldg(ix.rows + p);
                        ww[u] = __ldg(ix.w + p);
                    }
                }
#pragma unroll
                for (int u = 0; u < kBatch; ++u) {
                    if (ti[u] < 0) break;  // warp-uniform
                    const double wq = t_wq[g * 32 + ti[u]];
                    uint64_t c0 = cb[u];
                    uint32_t npk;
                    // first chunk (already loaded)
                    bool v = rr[u] < uhi;
                    if (v) acc[rr[u] - ub] = __dadd_rn(acc[rr[u] - ub], __dmul_rn(wq, ww[u]));
                    uint32_t n = __popc(__ballot_sync(0xffffffffu, v));
                    c0 += n;
                    npk = __shfl_sync(0xffffffffu, rr[u], n & 31);
                    while (n == 32) {  // a dense run: kRun chunks in flight
                        uint32_t r4[kRun];
                        double w4[kRun];
#pragma unroll
                        for (int h = 0; h < kRun; ++h) {
                            const uint64_t p = c0 + 32 * h + lane;
                            r4[h] = kNone;
                            w4[h] = 0.0;
                            if (p < eb[u]) {
                                r4[h] = __ldg(ix.rows + p);
                                w4[h] = __ldg(ix.w + p);
                            }
                        }
#pragma unroll
                        for (int h = 0; h < kRun; ++h) {
                            if (n != 32) break;  // warp-uniform
                            v = r4[h] < uhi;
                            if (v) acc[r4[h] - ub] = __dadd_rn(acc[r4[h] - ub], __dmul_rn(wq, w4[h]));
                            n = __popc(__ballot_sync(0xffffffffu, v));
                            c0 += n;
                            npk = __shfl_sync(0xffffffffu, r4[h], n & 31);
                        }
                    }
                    __syncwarp();
                    if (lane == ti[u]) {
                        c = c0;
                        pk = npk;
                    }
                }
            }
        };
        for (uint32_t ub = lo_w; ub < hi_w; ub += kBrUnit) {
            const uint32_t uhi = min(ub + kBrUnit, hi_w);
#pragma unroll
            for (int g = 0; g < kRegGroups; ++g)
                if (static_cast<uint32_t>(g) * 32 < m) walk_group(g, creg[g], preg[g], ereg[g], ub, uhi);
            for (uint32_t g = kRegGroups; g * 32 < m; ++g) {
                const uint32_t j = g * 32 + lane;
                uint64_t c = j < m ? cur_g[j] : 0;
                uint32_t pk = j < m ? static_cast<uint32_t>(pk_g[j]) : kNone;
                const uint64_t e = j < m ? t_end[j] : 0;
                walk_group(g, c, pk, e, ub, uhi);
                if (j < m) {
                    cur_g[j] = c;
                    pk_g[j] = pk;
                }
            }
            // ---- scan the unit: zero it, admit S > 0 and S >= bound
            const uint32_t nrow = uhi - ub;
            for (uint32_t r0 = 0; r0 < nrow; r0 += 32) {
                const uint32_t r = r0 + lane;
                double x = 0.0;
                if (r < nrow) {
                    x = acc[r];
                    if (x != 0.0) acc[r] = 0.0;
                }
                const double thr = fmax(Lw, __longlong_as_double(static_cast<long long>(S.Lg)));
                const bool c = x > 0.0 && x >= thr;
                const uint32_t bal = __ballot_sync(0xffffffffu, c);
                if (!bal) continue;
                if (nw + 32 > static_cast<uint32_t>(W)) {
                    nw = prune_list<W>(S.cs[warp], S.ci[warp], nw, k, lane);
                    if (nw == k) {
                        Lw = S.cs[warp][k - 1];
                        if (lane == 0) atomicMax(&S.Lg, static_cast<unsigned long long>(__double_as_longlong(Lw)));
                    }
                }
                const double thr2 = fmax(Lw, __longlong_as_double(static_cast<long long>(S.Lg)));
                const bool c2 = c && x >= thr2;
                const uint32_t bal2 = __ballot_sync(0xffffffffu, c2);
                if (c2) {
                    const uint32_t pos = nw + __popc(bal2 & ((1u << lane) - 1u));
                    S.cs[warp][pos] = x;
                    S.ci[warp][pos] = __ldg(ix.doc_ids + ub + r);
                }
                nw += __popc(bal2);
                __syncwarp();
            }
        }
        // ---- end of the query: every list pruned to its best k (sorted), then
        // merged by rank: an entry's global rank is its own index plus, per
        // other list, the entries that rank before it (binary search)
        nw = prune_list<W>(S.cs[warp], S.ci[warp], nw, k, lane);
        if (lane == 0) S.nw[warp] = nw;
        __syncthreads();
        uint32_t total = 0;
#pragma unroll
        for (int w = 0; w < kBrWarps; ++w) total += S.nw[w];
        for (int w = 0; w < kBrWarps; ++w) {
            const uint32_t n_own = S.nw[w];
            for (uint32_t i = tid; i < n_own; i += kBrThreads) {
                const double s = S.cs[w][i];
                const uint64_t id = S.ci[w][i];
                uint32_t rank = i;
                for (int v = 0; v < kBrWarps; ++v) {
                    if (v == w) continue;
                    uint32_t lo = 0, hi = S.nw[v];
                    while (lo < hi) {  // entries of list v that rank before (s, id)
                        const uint32_t mid = (lo + hi) >> 1;
                        if (better(S.cs[v][mid], S.ci[v][mid], s, id)) lo = mid + 1;
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
        if (tid == 0) {
            a.out_n[q] = total < k ? total : k;
            if (a.out_post) a.out_post[q] = S.post;
        }
        __syncthreads();
        if (tid < kBrWarps) S.nw[tid] = 0;
        if (tid == 0) S.Lg = 0ull;
    }
}

template <int W>
cudaError_t launch_w(const BridgeDev& ix, const BridgeArgs& a, int sms, cudaStream_t st) {
    const size_t smem = sizeof(BridgeSmem<W>);
    cudaError_t e = cudaFuncSetAttribute(bridge_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bridge_kernel<W>, kBrThreads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    bridge_kernel<W><<<sms * per_sm, kBrThreads, smem, st>>>(ix, a);
    return cudaGetLastError();
}

}  // namespace

uint32_t bridge_max_k() { return 512; }

uint32_t bridge_grid(uint32_t k, int sms) {
    // CTAs of the launch for this k (scratch is sized per CTA)
    int per_sm = 1;
    auto occ = [&](auto kern, size_t smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kBrThreads, smem);
    };
    if (k <= 32) occ(bridge_kernel<64>, sizeof(BridgeSmem<64>));
    else if (k <= 128) occ(bridge_kernel<256>, sizeof(BridgeSmem<256>));
    else occ(bridge_kernel<1024>, sizeof(BridgeSmem<1024>));
    return static_cast<uint32_t>(sms * (per_sm < 1 ? 1 : per_sm));
}

cudaError_t launch_bridge(const BridgeDev& ix, const BridgeArgs& a, int sms, cudaStream_t st) {
    // list capacity W >= k + 32 (a scan step appends up to 32 entries)
    if (a.k <= 32) return launch_w<64>(ix, a, sms, st);
    if (a.k <= 128) return launch_w<256>(ix, a, sms, st);
    return launch_w<1024>(ix, a, sms, st);
}

}  // namespace hm
