// search_fast_kernel: the fused BM25 hot path on sm_100a (v12).
//
// Two 8-warp CTAs per SM, persistent; each CTA owns one query at a time (LPT
// order) and sweeps its row window in kTile = 16384-row tiles.  Warp w OWNS
// the 2048-row unit [2048 w, 2048 w + 2048) of every tile:
//   * long terms stream the BAKED postings bk[] (bake.cu): one u32 carries the
//     byte offset of the row's fp32 accumulator (XOR-swizzled, conflict-free
//     for dense runs) and the idf-free impact truncated to 3 exponent + 16
//     mantissa bits -- no code-table lookup, no escapes.  The sub-tile table
//     gives the warp's contiguous sub-range of each term; it is read with
//     16-byte loads (ld.global.nc.v4, up to 8 per lane in flight) plus at most
//     6 unaligned boundary words;
//   * the first long term of a unit stores (acc = c*w) instead of
//     read-modify-write: the unit's accumulators are zero at that point;
//   * short terms: the tile segment (a few postings) is read by every warp and
//     filtered by row; their impacts come from a 256-entry code table;
//   * no other warp touches a unit's rows, so there are no atomics and no CTA
//     barrier anywhere in the tile loop;
//   * after a tile the warp scans its 2048 accumulators: docs that can still
//     reach the top-k join the warp's candidate list, accumulators are zeroed
//     (pitfall-3 sentinel reset, src/twophase.cpp:24-27).  A warp prunes its
//     list locally and publishes its k-th score to a CTA-wide lower bound Lg
//     that every warp uses as admission threshold.
// At the end of the query (one CTA barrier) the lists are merged, the
// survivors are rescored exactly in fp64 in the reference's operation and
// accumulation order (src/csr_index.cpp:10-15, 87-101), ranked by
// (score desc, DocId asc) (include/hybrid/types.hpp:21-25), and the Margin
// confidence + skip decision are written (src/cascade.cpp:15-21, 79-84).
//
// Exactness (bm25_search.cu has the argument): each fp32 contribution is
// c32 * w with c32 = fl(mult * idf) and w the baked impact, relative error
// < 2^-16 (truncation) + 2^-24; accumulation adds m roundings.  With
// delta = (m + 10) 2^-24 + 2^-16 every A(d) is within delta of E(d), and the
// admission slack 1 - 2.5 delta keeps the exact top-k among the survivors.
#include <cstdlib>

#include "hm_device.cuh"
#include "hm_launch.h"
#include "hm_ptx.cuh"

#include "probe.cuh"
#include "search_common.cuh"

namespace hm {

// ---------------------------------------------------------------- kernel

#ifdef HM_STATS  // development counters (scratch builds only): hm_dev_stats()
__device__ unsigned long long g_stats[8];
#define HM_STAT(i, v) atomicAdd(&g_stats[i], static_cast<unsigned long long>(v))
#else
#define HM_STAT(i, v) ((void)0)
#endif
// ---------------------------------------------------------------- essential-term mode
// Completion of a warp's pending rows (gp[0 .. np): (essential score bits <<
// 32) | row): every row is completed by probes of the terms its tile left out
// -- msorder[0 .. p) with p = the tile's prefix (p_lvl) -- in bound-descending
// order, dropped once (partial + unprobed bound)(1 + 3 delta) < te, and the
// complete fp32 scores A >= te are admitted into the warp's list exactly as
// the scan admits (prune beyond CAPW - 128 entries; a near-tie flood sets
// `flood`).  Out of line: the tile loop keeps its registers.
template <int CAPW, class Smem>
__device__ __noinline__ uint32_t ne_complete(const ProbeCtx<Smem>& pc, const uint64_t* gp, uint32_t np,
                                             uint32_t nw, float& Lw, float f_ub, float f_slack, uint32_t k,
                                             uint32_t j0, uint32_t n_ne, bool& flood) {
    Smem& S = pc.S;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float te = fmaxf(fmaxf(Lw, __uint_as_float(S.Lg)) * f_slack, kFltMin);
    if (lane == 0) HM_STAT(0, np);
    for (uint32_t b0 = 0; b0 < np && !flood; b0 += 128) {
        RowsN<4> rw;
        float A[4];
        uint32_t pr[4];
        uint32_t live = 0, pmax = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t i = b0 + lane + 32 * u;
            const uint64_t e = i < np ? gp[i] : 0ull;
            rw.r[u] = static_cast<uint32_t>(e);
            A[u] = __uint_as_float(static_cast<uint32_t>(e >> 32));
            uint32_t pj = 0;  // levels reached by the row's tile (p_lvl is ascending)
            const uint32_t jt = (rw.r[u] >> kTileShift) - j0;
            for (uint32_t l = 1; l <= n_ne && S.p_lvl[warp][l] <= jt; ++l) pj = l;
            pr[u] = pj;
            if (i < np) {
                live |= 1u << u;
                pmax = max(pmax, pj);
            }
        }
        pmax = __reduce_max_sync(0xffffffffu, pmax);
        for (int j = static_cast<int>(pmax) - 1; j >= 0; --j) {
            const float rem = S.rem_ub[j + 1];  // msorder[0 .. j] unprobed
            uint32_t need = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (!((live >> u) & 1u) || pr[u] <= static_cast<uint32_t>(j)) continue;
                if ((A[u] + rem) * f_ub < te) live &= ~(1u << u);
                else need |= 1u << u;
            }
            if (need) {
                HM_STAT(2, __popc(need));
                const ValsN<4> x = seed_probeN<Smem, 4>(pc, S.msorder[j], rw, need);
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if ((need >> u) & 1u) A[u] += x.v[u];
            }
        }
        uint32_t ok = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (((live >> u) & 1u) && A[u] >= te) ok |= 1u << u;
        const uint32_t cnt = __popc(ok);
        const uint32_t incl = warp_incl_scan(cnt);
        if (lane == 31) HM_STAT(3, incl);
        uint32_t slot = nw + incl - cnt;
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if ((ok >> u) & 1u) {
                S.cl_row[warp][slot] = rw.r[u];
                S.cl_val[warp][slot] = A[u];
                ++slot;
            }
        nw += __shfl_sync(0xffffffffu, incl, 31);
        __syncwarp();
        if (nw > static_cast<uint32_t>(CAPW - 128)) {
            nw = warp_prune(S, warp, nw, k, Lw, f_slack);
            te = fmaxf(fmaxf(Lw, __uint_as_float(S.Lg)) * f_slack, kFltMin);
            if (nw > static_cast<uint32_t>(CAPW - 128)) flood = true;  // near-tie flood
        }
    }
    return nw;
}

#ifndef HM_NE_ALL
#define HM_NE_ALL 0
#endif
// the essential-term variant serves the queries handed over with a bound
// (HM_NE_ALL: every query of the sweep)
__host__ __device__ __forceinline__ bool sweep_ne_on(const BatchArgs& a) {
    return !(a.flags & kFlagNoNeSkip);
}
// fb_list values: 0 served by the seeded pass, 1 no bound, else the bound's
// bits; kFbPlain marks a query the essential-term variant gave back (overflow)
constexpr uint32_t kFbPlain = 0x80000000u;
__device__ __forceinline__ bool ne_takes(const BatchArgs& a, uint32_t fb, uint32_t q) {
    if (fb & kFbPlain) return false;
    if (HM_NE_ALL || (a.flags & kFlagNeAll)) return true;
    const uint32_t m = a.plan_len[a.split > 1 ? q % a.nq_real : q];
    return m >= kNeMinTerms && m <= kFastTerms;  // as counted by plan_kernel (counters[8])
}

// NE = true: the essential-term variant, launched first over the queries the
// seeded pass handed over WITH a lower bound; NE = false serves the others
// (every query without the seeded pass).  Two instantiations keep the plain
// sweep's register allocation free of the probe code.
template <int CAPW, bool NE>
__global__ void __launch_bounds__(kCons, 2) search_fast_kernel(DevIndex ix, BatchArgs a) {
    using Smem = FastSmem<CAPW>;
    constexpr int kGatherBytes = 8 * kConsWarps * CAPW;
    static_assert(kSurvBytes <= static_cast<int>(sizeof(float)) * kTile &&
                      kGatherBytes <= static_cast<int>(sizeof(float)) * kTile,
                  "epilogue buffers fit in the accumulator array");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    auto csync = [] { __syncthreads(); };
    const uint32_t cb = ix.code_bits;
    const double k1 = a.k1, bb = a.b;
    const uint32_t stride = a.stab_stride;
    uint32_t* stab = a.stab + static_cast<uint64_t>(blockIdx.x) * kMaxTerms * stride;
    const uint32_t kmax = FastCfg<CAPW>::kMaxKServed;
    constexpr int kC = FastCfg<CAPW>::kC;
    const uint32_t wbase = static_cast<uint32_t>(warp) * (kUnitRows * 4);  // my unit, bytes into acc
    char* const accw = reinterpret_cast<char*>(S.acc) + wbase;

    if (NE && !HM_NE_ALL && !(a.flags & kFlagNeAll) && a.counters[8] == 0) return;  // no plan for this variant
    for (int i = tid; i < kTile; i += kCons) S.acc[i] = 0.f;
    for (int i = tid; i < kShortCodes; i += kCons) S.w32s[i] = a.w32[i];
    if (tid < kConsWarps) S.n_w[tid] = 0;
    if (tid == 0) S.Lg = 0u;
    float Lw = 0.f;  // this warp's own k-th lower bound

    for (;;) {
        __syncthreads();
        if (tid == 0) {
            // after the seeded kernel: only the queries it handed over, still in
            // LPT order (the ones it served are skipped)
            // (NE: those with a bound, cursor counters[7]; the plain variant
            // leaves them out unless the essential-term mode is off)
            const bool ne_on = sweep_ne_on(a);
            uint32_t q = kNoTerm;
            for (;;) {
                const uint32_t w = atomicAdd(&a.counters[NE ? 7 : a.fb_list ? 5 : 0], 1u);
                if (w >= a.nq) {
                    q = kNoTerm;
                    break;
                }
                q = a.order[w];
                const uint32_t fb = a.fb_list ? a.fb_list[q] : 1u;  // 0: served by the seeded pass
                if (fb && (NE ? ne_takes(a, fb, q) : !ne_on || !ne_takes(a, fb, q))) break;
            }
            S.q = q;
        }
        __syncthreads();
        const uint32_t q = S.q;
        if (q == kNoTerm) break;
        uint32_t qr, row_lo, row_hi;  // the real query and this (slab) query's rows
        query_window(a, q, qr, row_lo, row_hi);
        const uint32_t poff = a.q_off[qr];
        const uint32_t m = a.plan_len[qr];
        const uint32_t k = a.k;
        if (m > kMaxTerms) {  // the wide path (wide.cu) serves it after the batch
            if (tid == 0 && a.wide_list) {
                a.wide_list[atomicAdd(&a.counters[6], 1u)] = q;
            } else if (tid == 0) {
                atomicOr(&a.counters[3], kErrTooManyTerms);
                a.out_n[q] = 0;
                if (a.out_post) a.out_post[q] = 0;
                write_decision(a, q, nullptr, 0);
            }
            continue;
        }
        if (m > kFastTerms || k > kmax || (a.flags & 1u)) {  // the exact kernel serves it
            if (tid == 0) a.exact_list[atomicAdd(&a.counters[1], 1u)] = q;
            continue;
        }
        // ---------------- prologue: plan, window bounds
        if (tid < static_cast<int>(m)) {
            const uint32_t t = a.plan_tid[poff + tid];
            const uint32_t mult = a.plan_mult[poff + tid];
            const double idf = ix.idf[t];
            const int32_t slot = ix.long_slot[t];
            const uint64_t s0 = ix.term_off[t], s1 = ix.term_off[t + 1];
            const uint64_t w0 = row_lo > 0 ? first_at_or_after(ix, slot, s0, s1, row_lo) : s0;
            const uint64_t w1 = row_hi < ix.n_docs ? first_at_or_after(ix, slot, s0, s1, row_hi) : s1;
            S.t_start[tid] = s0;
            S.t_wlo[tid] = w0;
            S.t_end[tid] = w1;
            S.t_idf[tid] = idf;
            S.t_mult[tid] = mult;
            // selection scores are score * 2^-61; long terms pair c with the
            // baked impact * 2^-ks, short terms with the plain impact table
            const int sh = slot >= 0 ? static_cast<int>(ix.bk_ks) - kScoreShift : -kScoreShift;
            S.t_c32[tid] = static_cast<float>(ldexp(static_cast<double>(mult) * idf, sh));
            S.t_slot[tid] = slot;
            S.t_trow[tid] = slot < 0 ? ix.short_tab_row[t] : kNoTabRow;
            S.t_bkb[tid] = slot >= 0 ? ix.bk_base[slot] : 0;
            S.t_dense[tid] = slot >= 0 ? ix.dense_of_slot[slot] : -1;  // (the exact rescoring's lookups)
        }
        if (NE && tid < static_cast<int>(m)) {  // bounds and probe weights of the essential-term mode (below)
            const uint32_t t = a.plan_tid[poff + tid];
            const uint32_t mult = a.plan_mult[poff + tid];
            const double idf = ix.idf[t];
            const int32_t slot = ix.long_slot[t];
            const float cu = static_cast<float>(ldexp(static_cast<double>(mult) * idf, -kScoreShift));
            S.t_cu[tid] = cu;
            S.t_ms[tid] = cu * ix.tmax[t] * 1.0000010f;  // rounded up: an upper bound
        }
        __syncthreads();
        if (tid == 0) {
            uint64_t post = 0;
            uint32_t nl = 0, ns = 0, bad = 0;
            // Essential-term mode (MaxScore inside the sweep, csr_index.cpp:
            // 106-207): the long terms by bound ascending (msorder[0..n_ne))
            // with the bound of every prefix (rem_ub[p], rounded up).  Each warp
            // leaves the first p of them out of its stream for a tile, p the
            // longest prefix whose bound stays below kNeAlpha * (its admission
            // threshold at that point); a row is then completed by probes only
            // if its essential score plus that bound can reach the threshold.
            uint32_t n_ne = 0;
            if (NE) {
                float U = 0.f;
                for (uint32_t i = 0; i < m; ++i) {
                    U += S.t_ms[i];
                    S.t_spos[i] = 0xFFu;  // rank among the long terms by bound (reused field)
                    if (S.t_slot[i] < 0) continue;
                    uint32_t p = n_ne++;
                    while (p > 0 && S.t_ms[S.msorder[p - 1]] > S.t_ms[i]) {
                        S.msorder[p] = S.msorder[p - 1];
                        --p;
                    }
                    S.msorder[p] = static_cast<uint8_t>(i);
                }
                float r = 0.f;
                S.rem_ub[0] = 0.f;
                for (uint32_t p = 0; p < n_ne; ++p) {
                    r += S.t_ms[S.msorder[p]];
                    S.rem_ub[p + 1] = r * 1.00001f;
                    S.t_spos[S.msorder[p]] = static_cast<uint8_t>(p);
                }
                if (a.flags & kFlagNoNeSkip) n_ne = 0;
                // admission histogram: 32 buckets per binade over the 8 binades
                // below the query's largest possible score (search_fast: hist_bound)
                const uint32_t ub = __float_as_uint(U * 1.001f) & 0x7F800000u;
                S.hbase = ub > (8u << 23) ? ub - (8u << 23) : 0u;
            }
            S.n_ne = n_ne;
            for (uint32_t i = 0; i < m; ++i) {
                post += S.t_end[i] - S.t_wlo[i];
                const double idf = S.t_idf[i];
                if (!(idf > 0.0) || !isfinite(idf)) bad = 1;
                if (S.t_slot[i] >= 0) {  // long terms by df descending: the first one stores
                    const uint64_t df = S.t_end[i] - S.t_wlo[i];
                    uint32_t p = nl++;
                    while (p > 0 && S.t_end[S.order_list[p - 1]] - S.t_wlo[S.order_list[p - 1]] < df) {
                        S.order_list[p] = S.order_list[p - 1];
                        --p;
                    }
                    S.order_list[p] = static_cast<uint16_t>(i);
                }
            }
            S.pref[0] = 0;
            for (uint32_t i = 0; i < m; ++i)
                if (S.t_slot[i] < 0) {
                    S.order_list[nl + ns] = static_cast<uint16_t>(i);
                    S.t_spos[i] = static_cast<uint8_t>(ns);  // stab row (the NE ranks are long terms only)
                    S.pref[ns + 1] =  // (a term with an index tile table is not scanned)
                        S.pref[ns] + (S.t_trow[i] != kNoTabRow ? 0u : static_cast<uint32_t>(S.t_end[i] - S.t_wlo[i]));
                    ++ns;
                }
            S.post = post;
            S.n_long = nl;
            S.n_short = ns;
            S.bad = bad;
            S.flood = 0;
            if (!(a.flags & 2u)) S.Lg = 0u;  // HM_FLAG_DEBUG_NO_RESET skips the sentinel reset
            // a query handed over by the seeded pass may carry a lower bound on
            // the k-th selection score (search_seed.cu: hand_over)
            const uint32_t fbq = a.fb_list ? a.fb_list[q] & ~kFbPlain : 0u;
            if (fbq > 1u) S.Lg = max(S.Lg, fbq);
            if (a.ext_bound) {  // doc shards: the union's bound (seed domain, slack for this one)
                const float e = a.ext_bound[qr] * kExtSlack;
                if (e > 0.f) S.Lg = max(S.Lg, __float_as_uint(e));
            }
        }
        if (!(a.flags & 2u)) {
            if (tid < kConsWarps) S.n_w[tid] = 0;
            Lw = 0.f;
        }
        if (NE)
            for (int i = tid; i < 256; i += kCons) S.hist[i] = 0u;
        __syncthreads();
        if (S.bad) {
            if (tid == 0) a.exact_list[atomicAdd(&a.counters[1], 1u)] = q;
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
        const uint32_t j0 = row_lo >> kTileShift, j1 = (row_hi - 1) >> kTileShift;
        const uint32_t nt = j1 - j0 + 1;
        // ---------------- short-term tile tables (per-CTA scratch)
        short_tables(ix, S, S.order_list + n_long, n_short, stab, stride, j0, nt, cb);

        // =============================================== tile sweep (per warp)
        const float delta = static_cast<float>(m + 10) * 5.9604645e-08f + 1.5258789e-05f;  // (m+10) 2^-24 + 2^-16
        const float f_slack = 1.0f - 2.5f * delta;
        const uint32_t wr0 = static_cast<uint32_t>(warp) << kUnitShift;  // my rows in a tile
        uint32_t nw = S.n_w[warp];
        bool flood = false;
        // my baked range of every long term for a tile: lane x prefetches term
        // x's two unit offsets for the NEXT tile into registers (plain loads,
        // latency covered by a tile's work) and installs them in smem when the
        // pipeline enters that tile
        uint32_t pre0 = 0, pre1 = 0;
        auto prefetch = [&](uint32_t j) {
            if (static_cast<uint32_t>(lane) < n_long) {
                const uint32_t* uo = ix.bk_uoff +
                                     static_cast<uint64_t>(S.t_slot[S.order_list[lane]]) * (ix.n_units + 1) +
                                     j * kUnitsPerTile + warp;
                pre0 = __ldg(uo);
                pre1 = __ldg(uo + 1);
            }
        };
        // lane x: term x's baked base address and fp32 weight
        const uint32_t* my_bk = nullptr;
        float my_c = 0.f;
        if (static_cast<uint32_t>(lane) < n_long) {
            const uint32_t i = S.order_list[lane];
            my_bk = ix.bk + S.t_bkb[i];
            my_c = S.t_c32[i];
        }
        uint32_t nrd = 0;  // ranges in rdesc for the installed tile
        auto live = [&](uint32_t j, uint32_t& u0, uint32_t& u1) {
            const uint32_t base = j << kTileShift;
            u0 = max(base + wr0, row_lo) - base;
            u1 = min(base + wr0 + kUnitRows, row_hi) - base;
            return u0 < u1;
        };
        // tile j's nonempty ranges of my unit as a compact descriptor list (the
        // previous tile's list is no longer read once the pipeline enters j)
        // essential-term mode: the prefix length p of the bound-ascending long
        // terms this warp leaves out of tile j, decided when the pipeline enters
        // j (which may run several empty tiles ahead of the scans) and never
        // decreasing: p_lvl records the first tile of every level, the scan of
        // tile j recovers its p from it
        const uint32_t n_ne = NE ? S.n_ne : 0u;
        const float f_ub = 1.0f + 3.0f * delta;
        uint64_t* const gp = NE ? a.ne_pend + (static_cast<uint64_t>(blockIdx.x) * kConsWarps + warp) * kNePendCap
                                : nullptr;
        uint32_t np = 0;  // pending rows of this warp (completed after the sweep)
        bool overflow = false;  // more than kNePendCap pending rows: handed to the plain sweep
        uint32_t p_inst = 0;
        if (NE) {
            S.p_lvl[warp][lane + 1] = 0xFFFFu;
            __syncwarp();
        }
        auto p_of_tile = [&](uint32_t j) -> uint32_t {
            const bool ok = static_cast<uint32_t>(lane) < n_ne && S.p_lvl[warp][lane + 1] <= j - j0;
            return __popc(__ballot_sync(0xffffffffu, ok));
        };
        const uint32_t my_rank = NE && static_cast<uint32_t>(lane) < n_long ? S.t_spos[S.order_list[lane]] : 0xFFu;
        auto pick_p = [&]() -> uint32_t {
            if (!n_ne || np > kNePendCap / 2) return 0u;  // no further growth under buffer pressure
            const float cap = kNeAlpha * fmaxf(fmaxf(Lw, __uint_as_float(S.Lg)) * f_slack, kFltMin);
            const bool ok = static_cast<uint32_t>(lane) < n_ne && S.rem_ub[lane + 1] * f_ub < cap;
            return __popc(__ballot_sync(0xffffffffu, ok));  // rem_ub increases: a prefix
        };
        auto install = [&](uint32_t j) {
            __syncwarp();  // every lane is done reading the previous tile's descriptors
            uint32_t u0, u1;
            uint32_t pj = 0;
            if constexpr (NE) {
                pj = max(p_inst, pick_p());
                if (static_cast<uint32_t>(lane) >= p_inst && static_cast<uint32_t>(lane) < pj)
                    S.p_lvl[warp][lane + 1] = static_cast<uint16_t>(j - j0);
                p_inst = pj;
            }
            const bool ok = static_cast<uint32_t>(lane) < n_long && pre1 > pre0 && live(j, u0, u1) && my_rank >= pj;
            const uint32_t bal = __ballot_sync(0xffffffffu, ok);
            if (ok) {
                const uint64_t addr = reinterpret_cast<uint64_t>(my_bk + pre0);
                S.rdesc[warp][__popc(bal & ((1u << lane) - 1u))] =
                    make_uint4(static_cast<uint32_t>(addr), static_cast<uint32_t>(addr >> 32), (pre1 - pre0) >> 2,
                               __float_as_uint(my_c));
            }
            nrd = __popc(bal);
            __syncwarp();
            if (j < j1) prefetch(j + 1);
        };
        // Long terms run as a software pipeline of steps over (tile, range,
        // chunk), FastCfg::kStages deep (2 measured best on C2; 3 supported):
        // the loads of the next step(s) -- possibly ranges of later tiles --
        // are in flight while the current step is applied, and across the
        // short-term pass and the scan.
        // ---- essential-term mode: scan of a unit whose first p bound-ascending
        // long terms were not streamed (U = rem_ub[p]).  Rows with
        // (A_E + U)(1 + 3 delta) >= te are collected at the tail of the warp's
        // list (<= 128 pending) and completed by probes of the left-out terms
        // in bound-descending order, each dropped once (partial + unprobed
        // bound)(1 + 3 delta) < te; the complete fp32 scores are admitted with
        // the usual rule (A >= te).  A row below the first test cannot reach te:
        // its score is at most (A_E + U)(1 + 3 delta) -- the seeded pass's
        // argument.  Admitted scores also go into a CTA-wide histogram whose
        // k-th bucket floor is a lower bound on the k-th largest score (hist_bound).
        const ProbeCtx<Smem> pc{ix, a, S, stab, stride, j0, cb, k1, bb};
        const uint32_t hbase = NE ? S.hbase : 0u;
        auto hist_add = [&](float A) {
            const uint32_t u = __float_as_uint(A);
            atomicAdd(&S.hist[u <= hbase ? 0u : min((u - hbase) >> 18, 255u)], 1u);
        };
        // every counted document is distinct (a row is admitted once per query)
        // and has A >= the floor of its bucket: the floor of the bucket holding
        // the k-th largest count is a valid Lg (counts only grow: stale reads
        // give a smaller, still valid bound)
        auto hist_bound = [&]() {
            uint32_t loc[8], sum = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                loc[j] = S.hist[lane * 8 + j];
                sum += loc[j];
            }
            uint32_t incl = sum;  // over lanes >= lane
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t nb = __shfl_down_sync(0xffffffffu, incl, o);
                if (lane + o < 32) incl += nb;
            }
            const uint32_t above = incl - sum;
            uint32_t bkt = 0;
            if (above < k && k <= incl) {
                uint32_t cum = above;
                for (int j = 7; j >= 0; --j) {
                    cum += loc[j];
                    if (cum >= k) {
                        bkt = static_cast<uint32_t>(lane * 8 + j);
                        break;
                    }
                }
            }
            bkt = __reduce_max_sync(0xffffffffu, bkt);
            if (lane == 0 && bkt > 0) atomicMax(&S.Lg, hbase + (bkt << 18));
        };
        auto scan_ne = [&](float4* acc4, uint32_t base, float te, uint32_t pj) {
            constexpr uint32_t kV = kUnitRows / 4;
            const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
            const float ubne = S.rem_ub[pj];
            auto pend = [&](float4 x4, uint32_t v) {
                const bool q0 = (x4.x + ubne) * f_ub >= te, q1 = (x4.y + ubne) * f_ub >= te;
                const bool q2 = (x4.z + ubne) * f_ub >= te, q3 = (x4.w + ubne) * f_ub >= te;
                const uint32_t cnt = q0 + q1 + q2 + q3;
                if (!__any_sync(0xffffffffu, cnt != 0)) return;
                const uint32_t incl = warp_incl_scan(cnt);
                const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
                if (np + tot > kNePendCap) {  // full: the plain sweep serves the query (below)
                    overflow = true;
                    return;
                }
                uint64_t* dst = gp + np + incl - cnt;
                const uint32_t P = wr0 + 4 * v;
                auto put = [&](bool okp, uint32_t pos, float val) {
                    if (okp) {
                        *dst++ = (static_cast<uint64_t>(__float_as_uint(val)) << 32) | (base + swz10(pos));
                        hist_add(val);  // a partial score: a lower bound of the row's score
                    }
                };
                put(q0, P, x4.x);
                put(q1, P + 1, x4.y);
                put(q2, P + 2, x4.z);
                put(q3, P + 3, x4.w);
                np += tot;
            };
#pragma unroll 1
            for (uint32_t vb = 0; vb < kV && !overflow; vb += 128) {
                float4 x[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    x[q] = acc4[vb + 32 * q + lane];
                    acc4[vb + 32 * q + lane] = z4;
                }
                const float m0 = max3f(x[0].x, x[0].y, x[0].z), m1 = max3f(x[0].w, x[1].x, x[1].y);
                const float m2 = max3f(x[1].z, x[1].w, x[2].x), m3 = max3f(x[2].y, x[2].z, x[2].w);
                const float m4 = max3f(x[3].x, x[3].y, x[3].z);
                const float mx = fmaxf(max3f(m0, m1, m2), max3f(m3, m4, x[3].w));
                if (__any_sync(0xffffffffu, (mx + ubne) * f_ub >= te)) {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (!overflow) pend(x[q], vb + 32 * q + lane);
                }
            }
            if (overflow)  // the plain sweep takes the query: finish zeroing my rows
                for (uint32_t z = lane; z < kV; z += 32) acc4[z] = z4;
            __syncwarp();
        };
        // short terms: lane s holds term s's segment of the next tile to process
        uint64_t ss_b = 0, ss_e = 0;
        float my_sc = 0.f;
        const uint32_t* my_stab = nullptr;
        uint64_t my_s0 = 0;
        if (static_cast<uint32_t>(lane) < n_short) {
            const uint32_t i = S.order_list[n_long + lane];
            my_sc = S.t_c32[i];
            my_stab = stab + static_cast<uint64_t>(lane) * stride;
            my_s0 = S.t_start[i];
        }
        auto short_prefetch = [&](uint32_t j) {
            if (static_cast<uint32_t>(lane) < n_short) {
                ss_b = my_s0 + my_stab[j - j0];
                ss_e = my_s0 + my_stab[j - j0 + 1];
            }
        };
        if (NE && n_short) short_prefetch(j0);
        uint32_t ready = j0;  // the tile whose ranges are in rdesc
        prefetch(j0);
        install(j0);
        // first nonempty range at or after (j, x)
        auto seek = [&](uint32_t j, uint32_t x, bool fst) -> Step {
            for (;;) {
                if (j > j1) return Step{nullptr, 0, 0, j, 0, 0.f, false};
                if (j > ready) {
                    ready = j;
                    install(j);
                }
                if (x < nrd) {
                    const uint4 d = S.rdesc[warp][x];
                    return Step{reinterpret_cast<const uint4*>((static_cast<uint64_t>(d.y) << 32) | d.x), 0, d.z, j, x,
                                __uint_as_float(d.w), x == 0};
                }
                ++j;
                x = 0;
            }
        };
        auto advance = [&](const Step& s) -> Step {
            if (s.o + 32 * kC < s.nch) {
                Step t = s;
                t.o += 32 * kC;
                return t;
            }
            return seek(s.j, s.x + 1, false);
        };
        Step cur = seek(j0, 0, true);
        constexpr int kSt = FastCfg<CAPW>::kStages;
        uint32_t stage = 0;  // cur's stage; nx1 (3 stages) is in stage + 1
        if (cur.j <= j1) step_issue<kC>(cur, S.stg[warp][0]);
        asm volatile("cp.async.commit_group;" ::: "memory");
        Step nx1 = cur;
        if (kSt == 3) {
            nx1 = cur.j <= j1 ? advance(cur) : cur;
            if (nx1.j <= j1) step_issue<kC>(nx1, S.stg[warp][1]);
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        for (uint32_t j = j0; j <= j1; ++j) {
            const uint32_t base = j << kTileShift;
            uint32_t u0, u1;
            const bool unit_live = live(j, u0, u1);
            const bool clip = (u1 - u0) != static_cast<uint32_t>(kUnitRows);
            const Clip ck{wr0, u0, u1};
            // ---- long terms of this tile (df descending; the first one stores)
            while (cur.j == j) {
                Step nxt;  // the step after cur
                if (kSt == 3) {
                    const Step nx2 = nx1.j <= j1 ? advance(nx1) : nx1;
                    if (nx2.j <= j1) step_issue<kC>(nx2, S.stg[warp][stage >= 1 ? stage - 1 : 2]);
                    asm volatile("cp.async.commit_group;" ::: "memory");
                    asm volatile("cp.async.wait_group 2;" ::: "memory");  // cur's chunks have landed
                    nxt = nx1;
                    nx1 = nx2;
                } else {
                    nxt = advance(cur);
                    if (nxt.j <= j1) step_issue<kC>(nxt, S.stg[warp][stage ^ 1]);
                    asm volatile("cp.async.commit_group;" ::: "memory");
                    asm volatile("cp.async.wait_group 1;" ::: "memory");  // cur's chunks have landed
                }
                const uint4* stg = S.stg[warp][stage];
                if (!clip) {
                    if (cur.first) step_apply<kC, true, false>(S.acc, wbase, cur, stg, ck);
                    else step_apply<kC, false, false>(S.acc, wbase, cur, stg, ck);
                } else {
                    if (cur.first) step_apply<kC, true, true>(S.acc, wbase, cur, stg, ck);
                    else step_apply<kC, false, true>(S.acc, wbase, cur, stg, ck);
                }
                // the next range (another term) may touch the same rows from other
                // lanes (a lane only ever reads the stage slots it filled itself)
                if (nxt.j != cur.j || nxt.x != cur.x) __syncwarp();
                cur = nxt;
                stage = stage + 1 == static_cast<uint32_t>(kSt) ? 0 : stage + 1;
            }
            // ---- short terms: the tile segments of all of them (a few postings
            // each) flattened across the lanes -- lane s holds short term s's
            // segment (offsets prefetched one tile ahead), a warp scan of the
            // lengths, then every lane takes postings f = lane, lane + 32, ...
            // of the concatenation (loads in flight together); every warp
            // keeps the rows of its own unit.  Two lanes of one step may hold
            // the same row (a document with two short terms): rows are merged
            // with a match before the read-modify-write.
            if (!NE) {  // short terms one after the other: the tile segment is small; every warp filters its rows
                for (uint32_t st = 0; st < n_short; ++st) {
                    const uint32_t i = S.order_list[n_long + st];
                    const float c = S.t_c32[i];
                    const uint32_t* tab = stab + static_cast<uint64_t>(st) * stride;
                    const uint64_t b = S.t_start[i] + tab[j - j0], e = S.t_start[i] + tab[j - j0 + 1];
                    for (uint64_t b0 = b; b0 < e; b0 += 32) {
                        const uint64_t g = b0 + lane;
                        if (g < e) {
                            const uint32_t p = __ldg(ix.post + g);
                            const uint32_t local = (p >> cb) - base;
                            if (local - wr0 < static_cast<uint32_t>(kUnitRows)) {
                                const uint32_t code = p & ix.esc_short;
                                const float w = code < ix.n_codes_short ? S.w32s[code] : esc_w(ix, g, base + local, k1, bb);
                                float* acc = reinterpret_cast<float*>(accw) + (swz10(local) & (kUnitRows - 1));
                                *acc = __fmaf_rn(c, w, *acc);
                            }
                        }
                    }
                    __syncwarp();
                }
            } else if (n_short) {
                const uint32_t slen = ss_e > ss_b ? static_cast<uint32_t>(ss_e - ss_b) : 0u;
                const uint64_t sbg = ss_b;
                const uint32_t incl = warp_incl_scan(slen), spre = incl - slen;
                const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
                if (j < j1) short_prefetch(j + 1);
                constexpr int kSU = 4;
                for (uint32_t f0 = 0; f0 < total; f0 += 32 * kSU) {
                    uint64_t g[kSU];
                    float c[kSU];
                    uint32_t p[kSU];
#pragma unroll
                    for (int u = 0; u < kSU; ++u) {
                        const uint32_t f = f0 + 32 * u + lane;
                        uint32_t lo = 0, hi = n_short;  // largest term s with spre_s <= f
#pragma unroll
                        for (int it = 0; it < 5; ++it) {
                            const uint32_t mid = (lo + hi) >> 1;
                            const uint32_t pm = __shfl_sync(0xffffffffu, spre, mid & 31);
                            if (hi - lo > 1) {
                                if (pm <= f) lo = mid;
                                else hi = mid;
                            }
                        }
                        g[u] = __shfl_sync(0xffffffffu, sbg, lo) + (f - __shfl_sync(0xffffffffu, spre, lo));
                        c[u] = __shfl_sync(0xffffffffu, my_sc, lo);
                    }
#pragma unroll
                    for (int u = 0; u < kSU; ++u) p[u] = f0 + 32 * u + lane < total ? __ldg(ix.post + g[u]) : 0u;
#pragma unroll
                    for (int u = 0; u < kSU; ++u) {
                        const uint32_t local = (p[u] >> cb) - base;
                        const bool mine = f0 + 32 * u + lane < total && local - wr0 < static_cast<uint32_t>(kUnitRows);
                        float v = 0.f;
                        if (mine) {
                            const uint32_t code = p[u] & ix.esc_short;
                            v = c[u] * (code < ix.n_codes_short ? S.w32s[code] : esc_w(ix, g[u], base + local, k1, bb));
                        }
                        // lanes holding the same row: the lowest one adds the group's sum
                        const uint32_t key = mine ? local : 0xFFFFFFFFu;
                        const uint32_t grp = __match_any_sync(0xffffffffu, key);
                        if (mine) {
                            if (__popc(grp) > 1) {
                                float sum = 0.f;
                                for (uint32_t mm = grp; mm; mm &= mm - 1) sum += __shfl_sync(grp, v, __ffs(mm) - 1);
                                v = sum;
                            }
                            if ((__ffs(grp) - 1) == lane) {
                                float* acc = reinterpret_cast<float*>(accw) + (swz10(local) & (kUnitRows - 1));
                                *acc += v;
                            }
                        }
                        __syncwarp();  // the next step's lanes may hold the same rows
                    }
                }
                __syncwarp();
            }
            // ---- scan my unit: admit candidates, zero accumulators.  Rows
            // outside the window were never accumulated (zero), so the whole
            // unit is scanned.
            float4* acc4 = reinterpret_cast<float4*>(accw);
            constexpr uint32_t kV = kUnitRows / 4;
            const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
            if (flood || overflow) {  // this query goes elsewhere: only keep acc clean
                for (uint32_t z = lane; z < kV; z += 32) acc4[z] = z4;
                __syncwarp();
                continue;
            }
            // admission: A > 0 and A >= L * slack  <=>  A >= max(L * slack, FLT_MIN) (scaled
            // scores of real documents are >= ~1e-29, far above FLT_MIN)
            float te = fmaxf(fmaxf(Lw, __uint_as_float(S.Lg)) * f_slack, kFltMin);
            // append the qualifying entries of one float4 per lane (slow path)
            auto admit = [&](float4 x4, uint32_t v) {
                if (nw > static_cast<uint32_t>(CAPW - 128)) {
                    nw = warp_prune(S, warp, nw, k, Lw, f_slack);
                    te = fmaxf(fmaxf(Lw, __uint_as_float(S.Lg)) * f_slack, kFltMin);
                    if (nw > static_cast<uint32_t>(CAPW - 128)) {  // near-tie flood
                        flood = true;
                        return;
                    }
                }
                const bool q0 = x4.x >= te, q1 = x4.y >= te, q2 = x4.z >= te, q3 = x4.w >= te;
                const uint32_t cnt = q0 + q1 + q2 + q3;
                if (!__any_sync(0xffffffffu, cnt != 0)) return;
                const uint32_t incl = warp_incl_scan(cnt);
                uint32_t slot = nw + incl - cnt;
                const uint32_t P = wr0 + 4 * v;  // tile-local position of x4.x
                auto put = [&](bool ok, uint32_t pos, float val) {
                    if (ok) {
                        S.cl_row[warp][slot] = base + swz10(pos);  // position -> row (involution)
                        S.cl_val[warp][slot] = val;
                        ++slot;
                        if constexpr (NE) hist_add(val);
                    }
                };
                put(q0, P, x4.x);
                put(q1, P + 1, x4.y);
                put(q2, P + 2, x4.z);
                put(q3, P + 3, x4.w);
                nw += __shfl_sync(0xffffffffu, incl, 31);
                __syncwarp();
            };
            if constexpr (NE) {
                const uint32_t pj = p_of_tile(j);
                if (lane == 0) HM_STAT(pj ? 4 : 5, 1);
                if (pj) {
                    scan_ne(acc4, base, te, pj);
                    hist_bound();
                    continue;
                }
            }
#pragma unroll 1
            for (uint32_t vb = 0; vb < kV && !flood; vb += 128) {  // 4 float4 (16 rows) per lane
                float4 x[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    x[q] = acc4[vb + 32 * q + lane];
                    acc4[vb + 32 * q + lane] = z4;
                }
                const float m0 = max3f(x[0].x, x[0].y, x[0].z), m1 = max3f(x[0].w, x[1].x, x[1].y);
                const float m2 = max3f(x[1].z, x[1].w, x[2].x), m3 = max3f(x[2].y, x[2].z, x[2].w);
                const float m4 = max3f(x[3].x, x[3].y, x[3].z);
                const float mx = fmaxf(max3f(m0, m1, m2), max3f(m3, m4, x[3].w));
                if (__any_sync(0xffffffffu, mx >= te)) {
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (!flood) admit(x[q], vb + 32 * q + lane);
                }
            }
            if (flood)  // the query goes to the exact kernel: finish zeroing my rows
                for (uint32_t z = lane; z < kV; z += 32) acc4[z] = z4;
            __syncwarp();
            if constexpr (NE) {
                if (n_ne) hist_bound();
            }
        }
        if constexpr (NE) {
            if (overflow && lane == 0) atomicMax(&S.flood, 2u);
            if (np && !flood && !overflow) {
                __syncwarp();  // gp entries of every lane written
                nw = ne_complete<CAPW>(pc, gp, np, nw, Lw, f_ub, f_slack, k, j0, n_ne, flood);
            }
        }
        if (lane == 0) {
            S.n_w[warp] = nw;
            if (flood) atomicMax(&S.flood, 1u);
        }
        csync();
        if (NE && S.flood == 2u && a.fb_list) {  // a warp's pending rows overflowed: the plain sweep
            // (launched next) takes the query, with the seeded pass's bound
            if (tid == 0) a.fb_list[q] = kFbPlain | (a.fb_list[q] > 1u ? a.fb_list[q] : 1u);
            csync();
            if (tid < kConsWarps) S.n_w[tid] = 0;
            continue;
        }
        if (S.flood) {
            if (tid == 0) a.exact_list[atomicAdd(&a.counters[1], 1u)] = q;
            csync();
            if (tid < kConsWarps) S.n_w[tid] = 0;
            continue;
        }

        finish_query<CAPW>(ix, a, S, q, m, k, nw, f_slack, k1, bb, stab, stride, j0, cb);
    }
}

template <int CAPW>
static cudaError_t fast_attr() {
    static bool done = false;
    if (done) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(search_fast_kernel<CAPW, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(sizeof(FastSmem<CAPW>)));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(search_fast_kernel<CAPW, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(sizeof(FastSmem<CAPW>)));
    if (e == cudaSuccess) done = true;
    return e;
}

template <int CAPW>
static cudaError_t launch_fast_w(const DevIndex& ix, const BatchArgs& a, int sms, cudaStream_t st) {
    const cudaError_t e = fast_attr<CAPW>();
    if (e != cudaSuccess) return e;
    if (sweep_ne_launched(a)) search_fast_kernel<CAPW, true><<<2 * sms, kCons, sizeof(FastSmem<CAPW>), st>>>(ix, a);
    search_fast_kernel<CAPW, false><<<2 * sms, kCons, sizeof(FastSmem<CAPW>), st>>>(ix, a);
    return cudaGetLastError();
}

bool sweep_ne_launched(const BatchArgs& a) { return sweep_ne_on(a); }

// CAPW 192 (k <= 32) or 320 (k <= 128); two 8-warp CTAs per SM either way.
cudaError_t launch_search(const DevIndex& ix, const BatchArgs& a, int sms, cudaStream_t st) {
    return a.k <= FastCfg<192>::kMaxKServed ? launch_fast_w<192>(ix, a, sms, st) : launch_fast_w<320>(ix, a, sms, st);
}

cudaError_t search_occupancy_fast(int* blocks) {
    int b[2] = {0, 0};
    cudaError_t e = fast_attr<192>();
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b[0], search_fast_kernel<192, false>, kCons,
                                                          sizeof(FastSmem<192>));
    if (e == cudaSuccess) e = fast_attr<320>();
    if (e == cudaSuccess)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b[1], search_fast_kernel<320, false>, kCons,
                                                          sizeof(FastSmem<320>));
    if (e != cudaSuccess) return e;
    if (b[0] < 2 || b[1] < 2) return cudaErrorInvalidConfiguration;
    *blocks = 1;  // grid is sized in launch_search from the SM count
    return e;
}

size_t search_smem_bytes() { return sizeof(FastSmem<192>); }

}  // namespace hm

#ifdef HM_STATS
extern "C" int hm_dev_stats(unsigned long long* out, int reset) {
    if (cudaMemcpyFromSymbol(out, hm::g_stats, sizeof(hm::g_stats)) != cudaSuccess) return -1;
    if (reset) {
        static const unsigned long long z[8] = {};
        cudaMemcpyToSymbol(hm::g_stats, z, sizeof(z));
    }
    return 0;
}
#endif
