// sm_100a kernels of the batched BM25 search path.
//
//   plan_kernel    make_plan (src/csr_index.cpp:31-48) per query, on device
//   search_kernel  persistent; one CTA owns one query at a time and sweeps the
//                  query's row window tile by tile (kTile rows).  Per tile it
//                  streams every plan term's posting segment (128-bit
//                  ld.global.nc loads) into fp32 shared-memory accumulators,
//                  then scans the tile once: docs whose fp32 score can still
//                  reach the top-k are appended to a candidate list, the
//                  accumulators are zeroed (the pitfall-3 sentinel reset,
//                  src/twophase.cpp:24-27, happens per tile and per query).
//                  At the end the surviving candidates are RESCORED EXACTLY in
//                  fp64 in the reference's operation and accumulation order,
//                  ranked by (score desc, DocId asc), and the Margin
//                  confidence + skip decision are computed in the epilogue
//                  (src/cascade.cpp:15-21, 79-84).
//   exact_kernel   fp64 accumulation in plan order for queries that cannot
//                  use the fp32 selection (candidate flood, non-positive idf,
//                  b outside [0,1], or HM_FLAG_FORCE_EXACT).
//   merge_kernel   k-way merge of per-shard top-k lists (multi-GPU).
//
// Exactness argument of the selection.  With positive
// contributions, every fp32 score A(d) is within relative delta = (m+10)*2^-24
// of the fp64 score E(d).  L is always the k-th largest A over a set of real
// documents, so L <= a_k, the final k-th largest A.  A tile emits every doc
// with A >= L*(1-2.5*delta), a superset of {A >= a_k*(1-2.5*delta)}.  Any doc
// of the exact top-k (exact ties included) has
//   A >= (1-delta) e_k >= a_k (1-delta)/(1+delta) >= a_k (1-2.5*delta),
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
    uint64_t c = 0;
    for (uint32_t i = 0; i < m; ++i) c += ix.term_off[pt[i] + 1] - ix.term_off[pt[i]];
    a.plan_len[q] = m;
    a.cost[q] = c;
    order_in[q] = q;
}

// ============================================================ block helpers
// k-th largest of n >= k non-negative floats (radix select on the bits).
__device__ float block_kth_largest(const float* v, uint32_t n, uint32_t k, uint32_t* hist,
                                   uint32_t* sh) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t prefix = 0, pmask = 0, kk = k;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int i = tid; i < 256; i += kThreads) hist[i] = 0;
        __syncthreads();
        for (uint32_t i = tid; i < n; i += kThreads) {
            uint32_t u = __float_as_uint(v[i]);
            if ((u & pmask) == prefix) atomicAdd(&hist[(u >> shift) & 255u], 1u);
        }
        __syncthreads();
        if (warp == 0) {
            uint32_t loc[8], s = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                loc[j] = hist[lane * 8 + j];
                s += loc[j];
            }
            uint32_t incl = s;  // sum over lanes >= lane
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                uint32_t nb = __shfl_down_sync(0xffffffffu, incl, o);
                if (lane + o < 32) incl += nb;
            }
            uint32_t above = incl - s;
            if (above < kk && kk <= incl) {
                uint32_t cum = above;
                for (int j = 7; j >= 0; --j) {
                    if (cum + loc[j] >= kk) {
                        sh[0] = prefix | (static_cast<uint32_t>(lane * 8 + j) << shift);
                        sh[1] = kk - cum;
                        break;
                    }
                    cum += loc[j];
                }
            }
        }
        __syncthreads();
        prefix = sh[0];
        kk = sh[1];
        pmask |= 255u << shift;
    }
    __syncthreads();
    return __uint_as_float(prefix);
}

// In-place bitonic sort, "better" (score desc, id asc) first.  n is a power of
// two; entries past the live count must hold the (-inf, ~0) sentinel.
template <typename Row>
__device__ void block_bitonic(double* sc, uint64_t* id, Row* row, uint32_t n) {
    for (uint32_t k = 2; k <= n; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < n; i += kThreads) {
                uint32_t p = i ^ j;
                if (p > i) {
                    bool up = (i & k) == 0;
                    bool sw = up ? better(sc[p], id[p], sc[i], id[i])
                                 : better(sc[i], id[i], sc[p], id[p]);
                    if (sw) {
                        double ts = sc[i];
                        sc[i] = sc[p];
                        sc[p] = ts;
                        uint64_t ti = id[i];
                        id[i] = id[p];
                        id[p] = ti;
                        if (row) {
                            Row tr = row[i];
                            row[i] = row[p];
                            row[p] = tr;
                        }
                    }
                }
            }
            __syncthreads();
        }
    }
}

__device__ __forceinline__ uint32_t pow2_ceil(uint32_t x) {
    return x <= 1 ? 1 : 1u << (32 - __clz(x - 1));
}

// Margin confidence (src/cascade.cpp:15-21) and skip (:79-84), fp64.
__device__ __forceinline__ void write_decision(const BatchArgs& a, uint32_t q, const double* s,
                                               uint32_t n) {
    double conf = 0.0;
    if (n >= 2 && s[0] > 0.0) conf = __ddiv_rn(__dsub_rn(s[0], s[1]), fmax(s[0], a.eps));
    double tau = a.tau ? a.tau[q] : a.tau_default;
    if (a.out_conf) a.out_conf[q] = conf;
    if (a.out_skip) a.out_skip[q] = conf >= tau ? 1 : 0;
}

// ============================================================ shared state
struct __align__(16) SearchSmem {
    float acc[kTile];              // fp32 per-doc accumulators of one tile
    uint32_t cand_row[kCap];       // candidate list (row, fp32 score)
    float cand_a[kCap];
    // plan of the current query
    uint64_t t_start[kMaxTerms];   // term list start
    uint64_t t_wlo[kMaxTerms];     // first posting inside the row window
    uint64_t t_end[kMaxTerms];     // end of the window's postings
    uint64_t t_cur[kMaxTerms];     // short terms: cursor
    uint64_t t_cur0[kMaxTerms];    // short terms: cursor at tile start
    double t_idf[kMaxTerms];
    uint32_t t_tid[kMaxTerms];
    uint32_t t_mult[kMaxTerms];
    float t_c32[kMaxTerms];
    int32_t t_slot[kMaxTerms];
    uint32_t seg_b[kMaxTerms], seg_e[kMaxTerms];
    uint16_t long_list[kMaxTerms], short_list[kMaxTerms];
    float w32[kMaxCodes];
    uint32_t code_tf[kMaxCodes], code_len[kMaxCodes];
    uint32_t hist[256];
    uint32_t sel[2];
    uint64_t post;
    uint32_t q, n_long, n_short, n_c, ovf, bad, n_surv;
    float L;
};

// survivors live in the (zero, idle) accumulator array during the epilogue
struct SurvView {
    double* E;
    uint64_t* id;
    uint32_t* row;
};
__device__ __forceinline__ SurvView surv_view(SearchSmem& S) {
    char* p = reinterpret_cast<char*>(S.acc);
    return {reinterpret_cast<double*>(p), reinterpret_cast<uint64_t*>(p + 8 * kSurvCap),
            reinterpret_cast<uint32_t*>(p + 16 * kSurvCap)};
}
constexpr int kSurvBytes = 20 * kSurvCap;
static_assert(kSurvBytes <= static_cast<int>(sizeof(float)) * kTile, "survivors fit in acc");

__device__ __forceinline__ float posting_w(const DevIndex& ix, const SearchSmem& S, uint32_t p,
                                           uint64_t i, uint32_t row, double k1, double b) {
    uint32_t code = p & ix.esc;
    if (code < ix.n_codes) return S.w32[code];
    return impact32(static_cast<double>(__ldg(ix.tf + i)),
                    static_cast<double>(__ldg(ix.doc_lens + row)), ix.avgdl, k1, b);
}

// ============================================================ fused kernel
__global__ void __launch_bounds__(kThreads, 2) search_kernel(DevIndex ix, BatchArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    SearchSmem& S = *reinterpret_cast<SearchSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t cb = ix.code_bits;
    const uint32_t row_lo = a.row_lo, row_hi = a.row_hi;
    const double k1 = a.k1, bb = a.b;

    for (int i = tid; i < kTile; i += kThreads) S.acc[i] = 0.f;
    for (int i = tid; i < kMaxCodes; i += kThreads) {
        S.w32[i] = a.w32[i];
        S.code_tf[i] = ix.code_tf[i];
        S.code_len[i] = ix.code_len[i];
    }
    if (tid == 0) {
        S.n_c = 0;
        S.L = 0.f;
    }

    for (;;) {
        __syncthreads();
        if (tid == 0) {
            uint32_t w = atomicAdd(&a.counters[0], 1u);
            S.q = w < a.nq ? a.order[w] : kNoTerm;
        }
        __syncthreads();
        const uint32_t q = S.q;
        if (q == kNoTerm) break;
        const uint32_t poff = a.q_off[q];
        const uint32_t m = a.plan_len[q];
        const uint32_t k = a.k;

        // ---------------- prologue: plan + window cursors
        if (m > kMaxTerms) {
            if (tid == 0) {
                atomicOr(&a.counters[3], kErrTooManyTerms);
                a.out_n[q] = 0;
                if (a.out_post) a.out_post[q] = 0;
                write_decision(a, q, nullptr, 0);
            }
            continue;
        }
        if (tid < static_cast<int>(m)) {
            uint32_t t = a.plan_tid[poff + tid];
            uint32_t mult = a.plan_mult[poff + tid];
            double idf = ix.idf[t];
            uint64_t s0 = ix.term_off[t], s1 = ix.term_off[t + 1];
            uint64_t w0 = s0, w1 = s1;
            if (row_lo > 0) w0 = lower_bound_row(ix.post, s0, s1, row_lo, cb);
            if (row_hi < ix.n_docs) w1 = lower_bound_row(ix.post, w0, s1, row_hi, cb);
            S.t_tid[tid] = t;
            S.t_mult[tid] = mult;
            S.t_idf[tid] = idf;
            S.t_c32[tid] = static_cast<float>(static_cast<double>(mult) * idf);
            S.t_start[tid] = s0;
            S.t_wlo[tid] = w0;
            S.t_end[tid] = w1;
            S.t_cur[tid] = w0;
            S.t_slot[tid] = ix.long_slot[t];
        }
        __syncthreads();
        if (tid == 0) {
            uint64_t post = 0;
            uint32_t nl = 0, ns = 0, bad = 0;
            for (uint32_t i = 0; i < m; ++i) {
                post += S.t_end[i] - S.t_wlo[i];
                double idf = S.t_idf[i];
                if (!(idf > 0.0) || !isfinite(idf)) bad = 1;
                if (S.t_slot[i] >= 0) S.long_list[nl++] = static_cast<uint16_t>(i);
                else S.short_list[ns++] = static_cast<uint16_t>(i);
            }
            S.post = post;
            S.n_long = nl;
            S.n_short = ns;
            S.bad = bad;
            S.ovf = 0;
            if (!(a.flags & 2u)) {  // HM_FLAG_DEBUG_NO_RESET skips the sentinel reset
                S.n_c = 0;
                S.L = 0.f;
            }
        }
        __syncthreads();
        if (S.bad || (a.flags & 1u)) {  // exact kernel takes this query
            if (tid == 0) {
                a.exact_list[atomicAdd(&a.counters[1], 1u)] = q;
                if (a.out_post) a.out_post[q] = S.post;
            }
            continue;
        }
        if (m == 0 || k == 0 || row_hi <= row_lo) {
            if (tid == 0) {
                a.out_n[q] = 0;
                if (a.out_post) a.out_post[q] = S.post;
                write_decision(a, q, nullptr, 0);
            }
            continue;
        }
        const uint32_t n_long = S.n_long, n_short = S.n_short;
        const float delta = static_cast<float>(m + 10) * 5.9604645e-08f;  // 2^-24
        const float f_slack = 1.0f - 2.5f * delta;
        bool to_exact = false;

        // ---------------- tile sweep
        const uint32_t j0 = row_lo >> kTileShift, j1 = (row_hi - 1) >> kTileShift;
        for (uint32_t j = j0; j <= j1 && !to_exact; ++j) {
            const uint32_t base = j << kTileShift;
            const uint32_t R0 = max(base, row_lo);
            const uint32_t R1 = min(base + kTile, row_hi);
            const uint32_t nrows = R1 - R0;
            if (tid < static_cast<int>(n_long)) {
                uint32_t i = S.long_list[tid];
                const uint32_t* tb = ix.tile_tab + static_cast<uint64_t>(S.t_slot[i]) * (ix.n_tiles + 1);
                S.seg_b[tid] = __ldg(tb + j);
                S.seg_e[tid] = __ldg(tb + j + 1);
            }
            if (tid < static_cast<int>(n_short)) {
                uint32_t i = S.short_list[tid];
                S.t_cur0[i] = S.t_cur[i];
            }
            for (int attempt = 0;; ++attempt) {
                __syncthreads();
                // long terms: all threads stream one term's segment, plain RMW
                for (uint32_t l = 0; l < n_long; ++l) {
                    const uint32_t i = S.long_list[l];
                    const float c = S.t_c32[i];
                    const uint64_t st = S.t_start[i];
                    const uint64_t b = st + S.seg_b[l], e = st + S.seg_e[l];
                    const uint64_t a4 = ((b + 3) & ~3ull) < e ? ((b + 3) & ~3ull) : e;
                    const uint64_t e4 = a4 + ((e - a4) & ~3ull);
                    auto one = [&](uint32_t p, uint64_t idx) {
                        uint32_t row = p >> cb;
                        if (row - R0 < nrows) {
                            float w = posting_w(ix, S, p, idx, row, k1, bb);
                            float* dst = &S.acc[row - base];
                            *dst = __fmaf_rn(c, w, *dst);
                        }
                    };
                    if (b + tid < a4) one(ldg_stream(ix.post + b + tid), b + tid);
                    if (e4 + tid < e) one(ldg_stream(ix.post + e4 + tid), e4 + tid);
                    const uint4* P4 = reinterpret_cast<const uint4*>(ix.post + a4);
                    const uint32_t nv = static_cast<uint32_t>((e4 - a4) >> 2);
                    constexpr int U = 4;
                    for (uint32_t v0 = tid; v0 < nv; v0 += kThreads * U) {
                        uint4 buf[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            uint32_t v = v0 + u * kThreads;
                            buf[u] = v < nv ? ldg_stream(P4 + v) : make_uint4(~0u, ~0u, ~0u, ~0u);
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            uint32_t v = v0 + u * kThreads;
                            if (v < nv) {
                                uint64_t idx = a4 + 4ull * v;
                                one(buf[u].x, idx);
                                one(buf[u].y, idx + 1);
                                one(buf[u].z, idx + 2);
                                one(buf[u].w, idx + 3);
                            }
                        }
                    }
                    __syncthreads();
                }
                // short terms: a warp per term walks its cursor, shared atomics
                for (uint32_t s = warp; s < n_short; s += kWarps) {
                    const uint32_t i = S.short_list[s];
                    const float c = S.t_c32[i];
                    const uint64_t end = S.t_end[i];
                    uint64_t cur = S.t_cur[i];
                    for (;;) {
                        uint64_t idx = cur + lane;
                        uint32_t p = idx < end ? __ldg(ix.post + idx) : 0xFFFFFFFFu;
                        uint32_t row = p >> cb;
                        bool in = idx < end && row < R1;
                        uint32_t bal = __ballot_sync(0xffffffffu, in);
                        if (in) atomicAdd(&S.acc[row - base], c * posting_w(ix, S, p, idx, row, k1, bb));
                        uint32_t cnt = __popc(bal);
                        cur += cnt;
                        if (cnt < 32) break;
                    }
                    if (lane == 0) S.t_cur[i] = cur;
                }
                __syncthreads();
                // scan: emit docs that can still make the top-k, zero the tile
                {
                    const float t_emit = S.L * f_slack;
                    const uint32_t lo = R0 - base, hi = R1 - base;
                    const uint32_t v0 = lo >> 2, v1 = (hi + 3) >> 2;
                    float4* acc4 = reinterpret_cast<float4*>(S.acc);
                    for (uint32_t vb = v0; vb < v1; vb += kThreads) {
                        const uint32_t v = vb + tid;
                        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
                        if (v < v1) {
                            x = acc4[v];
                            acc4[v] = make_float4(0.f, 0.f, 0.f, 0.f);
                        }
                        bool q0 = x.x > 0.f && x.x >= t_emit, q1 = x.y > 0.f && x.y >= t_emit;
                        bool q2 = x.z > 0.f && x.z >= t_emit, q3 = x.w > 0.f && x.w >= t_emit;
                        uint32_t cnt = q0 + q1 + q2 + q3;
                        if (__ballot_sync(0xffffffffu, cnt != 0)) {
                            uint32_t incl = warp_incl_scan(cnt);
                            uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
                            uint32_t bse = 0;
                            if (lane == 31) bse = atomicAdd(&S.n_c, tot);
                            bse = __shfl_sync(0xffffffffu, bse, 31);
                            if (lane == 31 && bse + tot > kCap) S.ovf = 1;
                            uint32_t slot = bse + incl - cnt;
                            const uint32_t r = base + 4 * v;
                            auto put = [&](bool ok, uint32_t row, float val) {
                                if (ok) {
                                    if (slot < kCap) {
                                        S.cand_row[slot] = row;
                                        S.cand_a[slot] = val;
                                    }
                                    ++slot;
                                }
                            };
                            put(q0, r, x.x);
                            put(q1, r + 1, x.y);
                            put(q2, r + 2, x.z);
                            put(q3, r + 3, x.w);
                        }
                    }
                }
                __syncthreads();
                if (!S.ovf) break;
                // ---- overflow: raise L from the (partial) list, drop this tile's
                // entries, re-accumulate the tile (postings are L2-hot)
                const uint32_t nc = min(S.n_c, static_cast<uint32_t>(kCap));
                float nl = block_kth_largest(S.cand_a, nc, k, S.hist, S.sel);
                if (attempt >= 3 || !(nl > S.L)) {
                    to_exact = true;
                    break;
                }
                if (warp == 0) {
                    const float thr = nl * f_slack;
                    uint32_t w = 0;
                    for (uint32_t b0 = 0; b0 < nc; b0 += 32) {
                        uint32_t i = b0 + lane;
                        uint32_t row = 0;
                        float v = 0.f;
                        bool keep = false;
                        if (i < nc) {
                            row = S.cand_row[i];
                            v = S.cand_a[i];
                            keep = (row < R0 || row >= R1) && v >= thr;
                        }
                        uint32_t bal = __ballot_sync(0xffffffffu, keep);
                        uint32_t pos = w + __popc(bal & ((1u << lane) - 1));
                        __syncwarp();
                        if (keep) {
                            S.cand_row[pos] = row;
                            S.cand_a[pos] = v;
                        }
                        w += __popc(bal);
                        __syncwarp();
                    }
                    if (lane == 0) {
                        S.n_c = w;
                        S.L = nl;
                        S.ovf = 0;
                    }
                }
                if (tid < static_cast<int>(n_short)) {
                    uint32_t i = S.short_list[tid];
                    S.t_cur[i] = S.t_cur0[i];
                }
            }
            if (to_exact) break;
            // ---- keep the list short: raise L and prune
            if (S.n_c > kCap / 2) {
                const uint32_t nc = S.n_c;
                float nl = block_kth_largest(S.cand_a, nc, k, S.hist, S.sel);
                if (warp == 0) {
                    const float L = fmaxf(S.L, nl);
                    const float thr = L * f_slack;
                    uint32_t w = 0;
                    for (uint32_t b0 = 0; b0 < nc; b0 += 32) {
                        uint32_t i = b0 + lane;
                        uint32_t row = 0;
                        float v = 0.f;
                        bool keep = false;
                        if (i < nc) {
                            row = S.cand_row[i];
                            v = S.cand_a[i];
                            keep = v >= thr;
                        }
                        uint32_t bal = __ballot_sync(0xffffffffu, keep);
                        uint32_t pos = w + __popc(bal & ((1u << lane) - 1));
                        __syncwarp();
                        if (keep) {
                            S.cand_row[pos] = row;
                            S.cand_a[pos] = v;
                        }
                        w += __popc(bal);
                        __syncwarp();
                    }
                    if (lane == 0) {
                        S.n_c = w;
                        S.L = L;
                    }
                }
                __syncthreads();
            }
        }
        __syncthreads();
        if (to_exact) {
            if (tid == 0) {
                a.exact_list[atomicAdd(&a.counters[1], 1u)] = q;
                if (a.out_post) a.out_post[q] = S.post;
            }
            continue;
        }

        // ---------------- epilogue: survivors, exact rescoring, ranking
        const uint32_t nc = S.n_c;
        float theta = 0.f;
        if (nc >= k) theta = block_kth_largest(S.cand_a, nc, k, S.hist, S.sel) * f_slack;
        SurvView sv = surv_view(S);
        if (warp == 0) {
            uint32_t w = 0;
            for (uint32_t b0 = 0; b0 < nc; b0 += 32) {
                uint32_t i = b0 + lane;
                bool keep = i < nc && S.cand_a[i] >= theta;
                uint32_t bal = __ballot_sync(0xffffffffu, keep);
                uint32_t pos = w + __popc(bal & ((1u << lane) - 1));
                if (keep && pos < kSurvCap) sv.row[pos] = S.cand_row[i];
                w += __popc(bal);
            }
            if (lane == 0) S.n_surv = w;
        }
        __syncthreads();
        const uint32_t ns = S.n_surv;
        if (ns > kSurvCap) {  // near-tie flood: exact kernel
            for (int i = tid; i < kSurvBytes / 4; i += kThreads) S.acc[i] = 0.f;
            if (tid == 0) {
                a.exact_list[atomicAdd(&a.counters[1], 1u)] = q;
                if (a.out_post) a.out_post[q] = S.post;
            }
            continue;
        }
        // warp per survivor, lanes over plan terms; fp64 sum in plan order
        for (uint32_t s = warp; s < ns; s += kWarps) {
            const uint32_t row = sv.row[s];
            double E = 0.0;
            for (uint32_t t0 = 0; t0 < m; t0 += 32) {
                const uint32_t t = t0 + lane;
                double val = 0.0;
                bool present = false;
                if (t < m) {
                    uint64_t lo, hi;
                    if (S.t_slot[t] >= 0) {
                        const uint32_t* tb = ix.tile_tab + static_cast<uint64_t>(S.t_slot[t]) * (ix.n_tiles + 1);
                        uint32_t jj = row >> kTileShift;
                        lo = S.t_start[t] + __ldg(tb + jj);
                        hi = S.t_start[t] + __ldg(tb + jj + 1);
                    } else {
                        lo = S.t_wlo[t];
                        hi = S.t_end[t];
                    }
                    uint64_t pos = lower_bound_packed(ix.post, lo, hi, row << cb);
                    if (pos < hi) {
                        uint32_t p = __ldg(ix.post + pos);
                        if ((p >> cb) == row) {
                            uint32_t code = p & ix.esc;
                            double tf, dl;
                            if (code < ix.n_codes) {
                                tf = S.code_tf[code];
                                dl = S.code_len[code];
                            } else {
                                tf = __ldg(ix.tf + pos);
                                dl = __ldg(ix.doc_lens + row);
                            }
                            val = bm25_exact(tf, S.t_idf[t], dl, ix.avgdl, k1, bb);
                            present = true;
                        }
                    }
                }
                const uint32_t cnt = min(32u, m - t0);
                for (uint32_t u = 0; u < cnt; ++u) {
                    double x = __shfl_sync(0xffffffffu, val, u);
                    bool pr = __shfl_sync(0xffffffffu, present, u);
                    if (pr) {
                        const uint32_t mu = S.t_mult[t0 + u];
                        for (uint32_t r = 0; r < mu; ++r) E = __dadd_rn(E, x);  // :94
                    }
                }
            }
            if (lane == 0) {
                sv.E[s] = E;
                sv.id[s] = __ldg(ix.doc_ids + row);
            }
        }
        __syncthreads();
        const uint32_t n2 = pow2_ceil(ns);
        for (uint32_t i = ns + tid; i < n2; i += kThreads) {
            sv.E[i] = -INFINITY;
            sv.id[i] = ~0ull;
            sv.row[i] = 0;
        }
        __syncthreads();
        block_bitonic(sv.E, sv.id, sv.row, n2);
        if (tid == 0) {
            uint32_t nout = 0;
            for (uint32_t i = 0; i < ns && nout < k; ++i) {
                if (!(sv.E[i] > 0.0)) break;  // zero scores never emitted (:56)
                a.out_ids[static_cast<uint64_t>(q) * k + nout] = sv.id[i];
                a.out_scores[static_cast<uint64_t>(q) * k + nout] = sv.E[i];
                ++nout;
            }
            a.out_n[q] = nout;
            if (a.out_post) a.out_post[q] = S.post;
            write_decision(a, q, sv.E, nout);
        }
        __syncthreads();
        for (int i = tid; i < kSurvBytes / 4; i += kThreads) S.acc[i] = 0.f;
    }
}

// ============================================================ exact kernel
struct __align__(16) ExactSmem {
    double acc[kExactTile];
    double cand_E[kExactCap];
    uint64_t cand_id[kExactCap];
    uint32_t cand_row[kExactCap];
    uint64_t t_start[kMaxTerms], t_wlo[kMaxTerms], t_end[kMaxTerms], t_cur[kMaxTerms],
        t_cur0[kMaxTerms], t_seg[kMaxTerms];
    double t_idf[kMaxTerms];
    uint32_t t_mult[kMaxTerms];
    uint32_t code_tf[kMaxCodes], code_len[kMaxCodes];
    uint64_t post;
    double LE;
    uint64_t Lid;
    uint32_t q, n_c, ovf, haveL;
};

// sort the exact list, keep the best `keep` entries, set L to the last kept
__device__ void exact_sort_keep(ExactSmem& S, uint32_t keep) {
    const uint32_t nc = min(S.n_c, static_cast<uint32_t>(kExactCap));
    const uint32_t n2 = pow2_ceil(nc);
    for (uint32_t i = nc + threadIdx.x; i < n2; i += kThreads) {
        S.cand_E[i] = -INFINITY;
        S.cand_id[i] = ~0ull;
        S.cand_row[i] = 0;
    }
    __syncthreads();
    block_bitonic(S.cand_E, S.cand_id, S.cand_row, n2);
    if (threadIdx.x == 0) {
        uint32_t nk = min(nc, keep);
        S.n_c = nk;
        if (nk == keep && keep > 0) {
            S.haveL = 1;
            S.LE = S.cand_E[nk - 1];
            S.Lid = S.cand_id[nk - 1];
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kThreads, 2) exact_kernel(DevIndex ix, BatchArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    ExactSmem& S = *reinterpret_cast<ExactSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31;
    const uint32_t cb = ix.code_bits;
    const uint32_t row_lo = a.row_lo, row_hi = a.row_hi;
    const double k1 = a.k1, bb = a.b;
    for (int i = tid; i < kExactTile; i += kThreads) S.acc[i] = 0.0;
    for (int i = tid; i < kMaxCodes; i += kThreads) {
        S.code_tf[i] = ix.code_tf[i];
        S.code_len[i] = ix.code_len[i];
    }
    for (;;) {
        __syncthreads();
        if (tid == 0) {
            uint32_t w = atomicAdd(&a.counters[2], 1u);
            S.q = w < a.counters[1] ? a.exact_list[w] : kNoTerm;
        }
        __syncthreads();
        const uint32_t q = S.q;
        if (q == kNoTerm) break;
        const uint32_t poff = a.q_off[q];
        const uint32_t m = a.plan_len[q];
        const uint32_t k = a.k;
        if (tid < static_cast<int>(m)) {
            uint32_t t = a.plan_tid[poff + tid];
            uint64_t s0 = ix.term_off[t], s1 = ix.term_off[t + 1];
            uint64_t w0 = s0, w1 = s1;
            if (row_lo > 0) w0 = lower_bound_row(ix.post, s0, s1, row_lo, cb);
            if (row_hi < ix.n_docs) w1 = lower_bound_row(ix.post, w0, s1, row_hi, cb);
            S.t_start[tid] = s0;
            S.t_wlo[tid] = w0;
            S.t_end[tid] = w1;
            S.t_cur[tid] = w0;
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
            const uint32_t j0 = row_lo >> kExactTileShift, j1 = (row_hi - 1) >> kExactTileShift;
            for (uint32_t j = j0; j <= j1; ++j) {
                const uint32_t base = j << kExactTileShift;
                const uint32_t R0 = max(base, row_lo);
                const uint32_t R1 = min(base + kExactTile, row_hi);
                if (tid < static_cast<int>(m)) {
                    uint64_t c = S.t_cur[tid];
                    S.t_cur0[tid] = c;
                    uint64_t lim = min(S.t_end[tid], c + (R1 - R0));
                    S.t_seg[tid] = lower_bound_row(ix.post, c, lim, R1, cb);
                }
                for (int attempt = 0;; ++attempt) {
                    __syncthreads();
                    // terms strictly in plan order: per-doc fp64 adds follow :87-101
                    for (uint32_t i = 0; i < m; ++i) {
                        const uint64_t b = S.t_cur0[i], e = S.t_seg[i];
                        const double idf = S.t_idf[i];
                        const uint32_t mu = S.t_mult[i];
                        for (uint64_t x = b + tid; x < e; x += kThreads) {
                            uint32_t p = __ldg(ix.post + x);
                            uint32_t row = p >> cb;
                            uint32_t code = p & ix.esc;
                            double tf, dl;
                            if (code < ix.n_codes) {
                                tf = S.code_tf[code];
                                dl = S.code_len[code];
                            } else {
                                tf = __ldg(ix.tf + x);
                                dl = __ldg(ix.doc_lens + row);
                            }
                            double s = bm25_exact(tf, idf, dl, ix.avgdl, k1, bb);
                            double v = S.acc[row - base];
                            for (uint32_t r = 0; r < mu; ++r) v = __dadd_rn(v, s);
                            S.acc[row - base] = v;
                        }
                        __syncthreads();
                    }
                    // scan: docs not worse than L (composite key) join the list
                    const bool haveL = S.haveL;
                    const double LE = S.LE;
                    const uint64_t Lid = S.Lid;
                    for (uint32_t rb = R0 - base; rb < R1 - base; rb += kThreads) {
                        const uint32_t r = rb + tid;
                        double E = 0.0;
                        if (r < R1 - base) {
                            E = S.acc[r];
                            S.acc[r] = 0.0;
                        }
                        bool qual = false;
                        uint64_t id = 0;
                        if (E > 0.0) {
                            id = __ldg(ix.doc_ids + base + r);
                            qual = !haveL || !better(LE, Lid, E, id);
                        }
                        uint32_t bal = __ballot_sync(0xffffffffu, qual);
                        if (bal) {
                            uint32_t bse = 0;
                            if (lane == 0) bse = atomicAdd(&S.n_c, __popc(bal));
                            bse = __shfl_sync(0xffffffffu, bse, 0);
                            if (lane == 0 && bse + __popc(bal) > kExactCap) S.ovf = 1;
                            uint32_t slot = bse + __popc(bal & ((1u << lane) - 1));
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
                            uint32_t row = S.cand_row[i];
                            if (row >= R0 && row < R1) continue;
                            S.cand_E[w] = S.cand_E[i];
                            S.cand_id[w] = S.cand_id[i];
                            S.cand_row[w] = row;
                            ++w;
                        }
                        S.n_c = w;
                        S.ovf = 0;
                        if (attempt > 64) atomicOr(&a.counters[3], 2u);
                    }
                    if (attempt > 64) break;
                }
                if (tid < static_cast<int>(m)) S.t_cur[tid] = S.t_seg[tid];
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

__device__ void merge_bitonic(double* sc, uint64_t* id, uint32_t n) {
    for (uint32_t k = 2; k <= n; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < n; i += kMergeThreads) {
                uint32_t p = i ^ j;
                if (p > i) {
                    bool up = (i & k) == 0;
                    bool sw = up ? better(sc[p], id[p], sc[i], id[i]) : better(sc[i], id[i], sc[p], id[p]);
                    if (sw) {
                        double ts = sc[i];
                        sc[i] = sc[p];
                        sc[p] = ts;
                        uint64_t ti = id[i];
                        id[i] = id[p];
                        id[p] = ti;
                    }
                }
            }
            __syncthreads();
        }
}

__global__ void __launch_bounds__(kMergeThreads) merge_kernel(
    uint32_t G, uint32_t nq, uint32_t k, const uint64_t* ids, const double* scores,
    const uint32_t* n, const double* tau, double tau_default, double eps, uint64_t* out_ids,
    double* out_scores, uint32_t* out_n, double* out_conf, uint8_t* out_skip) {
    __shared__ double sc[kMergeMax];
    __shared__ uint64_t id[kMergeMax];
    const uint32_t q = blockIdx.x;
    const uint32_t tot = G * k;
    const uint32_t n2 = pow2_ceil(tot);
    for (uint32_t i = threadIdx.x; i < n2; i += kMergeThreads) {
        double s = -INFINITY;
        uint64_t d = ~0ull;
        if (i < tot) {
            uint32_t g = i / k, r = i % k;
            if (r < n[static_cast<uint64_t>(g) * nq + q]) {
                uint64_t o = (static_cast<uint64_t>(g) * nq + q) * k + r;
                s = scores[o];
                d = ids[o];
            }
        }
        sc[i] = s;
        id[i] = d;
    }
    __syncthreads();
    merge_bitonic(sc, id, n2);
    if (threadIdx.x == 0) {
        uint32_t nout = 0;
        for (uint32_t i = 0; i < tot && nout < k; ++i) {
            if (!(sc[i] > 0.0)) break;
            out_ids[static_cast<uint64_t>(q) * k + nout] = id[i];
            out_scores[static_cast<uint64_t>(q) * k + nout] = sc[i];
            ++nout;
        }
        out_n[q] = nout;
        double conf = 0.0;
        if (nout >= 2 && sc[0] > 0.0) conf = __ddiv_rn(__dsub_rn(sc[0], sc[1]), fmax(sc[0], eps));
        double t = tau ? tau[q] : tau_default;
        if (out_conf) out_conf[q] = conf;
        if (out_skip) out_skip[q] = conf >= t ? 1 : 0;
    }
}

// ============================================================ launchers
cudaError_t launch_plan(const DevIndex& ix, const BatchArgs& a, uint32_t* order_in,
                        cudaStream_t st) {
    if (a.nq == 0) return cudaSuccess;
    plan_kernel<<<(a.nq + 127) / 128, 128, 0, st>>>(ix, a, order_in);
    return cudaGetLastError();
}

cudaError_t lpt_sort_bytes(uint32_t nq, size_t* bytes) {
    *bytes = 0;
    return cub::DeviceRadixSort::SortPairsDescending(nullptr, *bytes, (const uint64_t*)nullptr,
                                                     (uint64_t*)nullptr, (const uint32_t*)nullptr,
                                                     (uint32_t*)nullptr, static_cast<int>(nq));
}

cudaError_t launch_lpt_sort(void* temp, size_t bytes, const BatchArgs& a, uint64_t* cost_sorted,
                            const uint32_t* order_in, cudaStream_t st) {
    if (a.nq == 0) return cudaSuccess;
    return cub::DeviceRadixSort::SortPairsDescending(temp, bytes, a.cost, cost_sorted, order_in,
                                                     a.order, static_cast<int>(a.nq), 0, 64, st);
}

static bool g_attr_done = false;
static cudaError_t set_attrs() {
    if (g_attr_done) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(search_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sizeof(SearchSmem)));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(sizeof(ExactSmem)));
    if (e != cudaSuccess) return e;
    g_attr_done = true;
    return cudaSuccess;
}

cudaError_t launch_search(const DevIndex& ix, const BatchArgs& a, int grid, cudaStream_t st) {
    cudaError_t e = set_attrs();
    if (e != cudaSuccess) return e;
    search_kernel<<<grid, kThreads, sizeof(SearchSmem), st>>>(ix, a);
    return cudaGetLastError();
}

cudaError_t launch_exact(const DevIndex& ix, const BatchArgs& a, int grid, cudaStream_t st) {
    cudaError_t e = set_attrs();
    if (e != cudaSuccess) return e;
    exact_kernel<<<grid, kThreads, sizeof(ExactSmem), st>>>(ix, a);
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
    cudaError_t e = set_attrs();
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(sb, search_kernel, kThreads, sizeof(SearchSmem));
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(eb, exact_kernel, kThreads, sizeof(ExactSmem));
}

}  // namespace hm
