// search_seed_kernel: seeded MaxScore -- the sparse, document-at-a-time
// counterpart of the reference's lossless pruning (CsrIndex::
// bm25_topk_maxscore, src/csr_index.cpp:106-207; output identical to the
// exhaustive bm25_topk, acceptance.cpp:144-171), run BEFORE the exhaustive
// tile sweep.  For every query that has a short plan term (df <= 32 * n_tiles):
//
//   1. seeds: every posting of t*, the short term with the largest bound
//      ms_t = mult * idf * (max impact of the term), is scored completely by
//      probing each plan term (dense per-row code arrays for the most frequent
//      terms: one load; binary search in the term's 1,024-row sub-tile range or
//      short-term tile segment otherwise).  The k-th best seed score theta0 is
//      the k-th best score of real documents: a valid lower bound L.
//   2. split: the non-essential terms NE are the longest prefix of the
//      bound-ascending order with sum(ms) * (1 + 3 delta) < te = L (1 - 2.5
//      delta).  A document without t* and without any essential term scores
//      at most that sum: it cannot be admitted.
//   3. candidates: the postings of the essential terms (t* and the rest, E')
//      are accumulated per row in a shared-memory hash table (chunks of whole
//      tiles, fixed-point integer atomics; rows holding t* flagged -- the seeds
//      scored them), unless E' has more than kEMax postings -- then the query
//      falls back to the exhaustive kernel with L as its starting bound.  Rows
//      whose essential score plus the non-essential bound can still reach the
//      threshold are completed by probing the non-essential terms (bound
//      descending, early exit);
//   4. admission into the per-warp candidate lists with the exhaustive
//      kernel's rule (A >= L (1 - 2.5 delta)), then the common exact epilogue
//      (finish_query: survivors rescored in fp64 in the reference's order).
//
// Every document the exhaustive kernel would admit is scored here, and all
// fp32 scores carry the same delta bound, so the survivors -- and the
// bit-identical fp64 results -- are the same.  Queries without a short term,
// with too many essential postings, or with more candidates than the lists can
// hold are appended to the fallback list that the exhaustive kernel serves.
#include <cstddef>

#include "hm_device.cuh"
#include "hm_launch.h"
#include "hm_ptx.cuh"
#include "probe.cuh"
#include "search_common.cuh"

namespace hm {

#ifndef HM_SEED_PCOST
#define HM_SEED_PCOST 32
#endif
constexpr uint64_t kProbeCost = HM_SEED_PCOST;  // seeds: a probe (short dependent-load chain) ~ 32 streamed postings
#ifndef HM_SEED_EMAX
#define HM_SEED_EMAX 131072
#endif
constexpr uint64_t kEMax = HM_SEED_EMAX;    // essential (non-seed) postings served here (best measured on C2)
constexpr uint32_t kSeedMaxTerms = 16;  // longer plans go straight to the exhaustive kernel
constexpr uint64_t kSeedMaxDf = kSeedScratch / 2;  // seed term: the strongest bound among terms with fewer postings
// queries with fewer postings than n_docs / 540 (16K at C2) stay on the sweep;
// relative to the index so doc shards keep the same split (measured:
// 65,536 fixed: C2 26.7 ms, 1/8 shard 7.96 ms; n_docs / 540: 26.4 / 7.79 ms)
constexpr uint32_t kSeedMinPostDiv = 540;

// leave query q to the exhaustive kernel (which walks the LPT order itself).
// lb > 0: a lower bound, in the exhaustive kernel's selection domain, on the
// k-th largest selection score -- its starting Lg (fb_list holds its bits;
// positive floats order like their bit patterns; 1 = no bound)
__device__ __forceinline__ void hand_over(const BatchArgs& a, uint32_t q, float lb = 0.f) {
    a.fb_list[q] = lb > 0.f ? max(__float_as_uint(lb), 1u) : 1u;
    atomicAdd(&a.counters[4], 1u);
}

#ifdef HM_SEED_STATS  // development counters (scratch builds only): hm_seed_stats()
// (g_seed_stats[40]: search_common.cuh, one copy per translation unit)
#define SST(i, v) atomicAdd(&g_seed_stats[i], static_cast<unsigned long long>(v))
#define SCNT(var, v) (var += (v))
#else
#define SST(i, v) ((void)0)
#define SCNT(var, v) ((void)0)
#endif


template <int CAPW>
#ifndef HM_SEED_MINB
#define HM_SEED_MINB 2
#endif
__global__ void __launch_bounds__(kCons, HM_SEED_MINB) search_seed_kernel(DevIndex ix, BatchArgs a) {
    using Smem = SeedSmem<CAPW>;
    static_assert(16 * CAPW * 4 >= kSurvBytes, "epilogue scratch fits");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t cb = ix.code_bits;
    const double k1 = a.k1, bb = a.b;
    const uint32_t stride = a.stab_stride;
    uint32_t* stab = a.stab + static_cast<uint64_t>(blockIdx.x) * kMaxTerms * stride;
    // seed scores, then seed rows (n_seed <= min(kSeedMaxDf, n_docs) = seed_half):
    // in shared memory (the hash table's area, idle until then) up to
    // kSeedSmemMax seeds, else in the CTA's global scratch
    float* const gA = reinterpret_cast<float*>(a.seed_scratch + static_cast<uint64_t>(blockIdx.x) * 2u * a.seed_half);
    const uint32_t kmax = FastCfg<CAPW>::kMaxKServed;

    for (int i = tid; i < 16 * CAPW; i += kCons) S.acc[i] = 0.f;
    for (int i = tid; i < kShortCodes; i += kCons) S.w32s[i] = a.w32[i];
    if (tid < kConsWarps) S.n_w[tid] = 0;
    if (tid == 0) S.Lg = 0u;

    for (;;) {
        __syncthreads();
        if (tid == 0) {
            const uint32_t w = atomicAdd(&a.counters[0], 1u);
            S.q = w < a.nq ? (a.order_seed ? a.order_seed[w] : a.order[w]) : kNoTerm;
        }
        __syncthreads();
        const uint32_t q = S.q;
        if (q == kNoTerm) break;
#ifdef HM_SEED_STATS
        long long c_t0 = clock64(), c_t1 = 0, c_t2 = 0, c_t3 = 0;
        uint32_t c_sp = 0, c_ep = 0, c_np = 0, c_en = 0, c_ns = 0;  // c_ep / c_ns: probe slots (kP per call)
#endif
        uint32_t qr, row_lo, row_hi;  // the real query and this (slab) query's rows
        query_window(a, q, qr, row_lo, row_hi);
        const uint32_t poff = a.q_off[qr];
        const uint32_t m = a.plan_len[qr];
        const uint32_t k = a.k;
        // doc shards: ext = a bound of the union of the shards (same seed-domain
        // scores, global statistics); HM_FLAG_BOUND_ONLY: report this shard's L only
        const float ext = a.ext_bound ? a.ext_bound[qr] : 0.f;
        const bool bonly = (a.flags & kFlagBoundOnly) != 0;
        // with the union's bound the seeds need not be scored first: L = ext and
        // the seed term is hashed like every other essential term (its complete
        // seed scores were the bound pass's work)
        const bool seedless = ext > 0.f && !bonly;
        auto give_up = [&] {  // tid 0: no bound of our own -- the sweep takes the query
            if (bonly)
                for (uint32_t i = 0; i < k; ++i) a.out_bound[static_cast<uint64_t>(qr) * k + i] = 0.f;
            else hand_over(a, q, ext * kExtSlack);
        };
        // anything unusual goes to the exhaustive kernel, which routes it on
        // (plans longer than kSeedMaxTerms go to the sweep before the prologue's
        // serial bound sort: C4's 24-32-term plans)
        if (m == 0 || m > kFastTerms || k == 0 || k > kmax || (a.flags & 1u) || row_hi <= row_lo ||
            (m > kSeedMaxTerms && !(a.flags & 32u))) {
            if (tid == 0) give_up();
            continue;
        }
        // ---------------- prologue: plan, window bounds, bounds
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
            S.t_slot[tid] = slot;
            S.t_trow[tid] = slot < 0 ? ix.short_tab_row[t] : kNoTabRow;
            const float cu = static_cast<float>(ldexp(static_cast<double>(mult) * idf, -kScoreShift));
            S.t_cu[tid] = cu;
            S.t_ms[tid] = cu * ix.tmax[t] * 1.0000010f;  // rounded up: an upper bound
            S.t_dense[tid] = slot >= 0 ? ix.dense_of_slot[slot] : -1;
        }
        __syncthreads();
        if (tid == 0) {
            uint64_t post = 0;
            uint32_t ns = 0, bad = 0, seed = kNoTerm;
            S.pref[0] = 0;
            for (uint32_t i = 0; i < m; ++i) {
                post += S.t_end[i] - S.t_wlo[i];
                const double idf = S.t_idf[i];
                if (!(idf > 0.0) || !isfinite(idf)) bad = 1;
                if (S.t_slot[i] < 0) {
                    S.order_list[ns] = static_cast<uint16_t>(i);
                    S.t_spos[i] = static_cast<uint8_t>(ns);
                    S.pref[ns + 1] =  // (a term with an index tile table is not scanned)
                        S.pref[ns] + (S.t_trow[i] != kNoTabRow ? 0u : static_cast<uint32_t>(S.t_end[i] - S.t_wlo[i]));
                    ++ns;
                }
                if (S.t_end[i] - S.t_wlo[i] <= kSeedMaxDf && (seed == kNoTerm || S.t_ms[i] > S.t_ms[seed]))
                    seed = i;
            }
            // plan indices by bound ascending (ties by index)
            for (uint32_t i = 0; i < m; ++i) {
                uint32_t p = i;
                while (p > 0 && S.t_ms[S.msorder[p - 1]] > S.t_ms[i]) {
                    S.msorder[p] = S.msorder[p - 1];
                    --p;
                }
                S.msorder[p] = static_cast<uint8_t>(i);
            }
            S.post = post;
            S.n_short = ns;
            S.n_long = seed;  // reused: the seed term
            // serve the query here only when probing the seeds is cheaper than
            // streaming its postings (a dependent-load probe ~ 32 streamed
            // postings) and the plan is short enough for the bounds to bite
            bool worth = (seed != kNoTerm || seedless) && (m <= kSeedMaxTerms || (a.flags & 32u));
            if (worth && seedless) {
                worth = post >= ix.n_docs / kSeedMinPostDiv || (a.flags & 32u);
            } else if (worth && !(a.flags & 32u)) {  // HM_FLAG_SEED_ALL (tests) skips the cost rule
                const uint64_t n_seed = S.t_end[seed] - S.t_wlo[seed];
                worth = post >= ix.n_docs / kSeedMinPostDiv && n_seed * m * kProbeCost < post;
            }
            S.bad = bad || !worth;
            S.flood = 0;
            S.Lg = 0u;
        }
        if (tid < kConsWarps) S.n_w[tid] = 0;
        __syncthreads();
        if (S.bad) {  // no short term (or a non-positive idf): the exhaustive kernel
            if (tid == 0) give_up();
            continue;
        }
        const uint32_t n_short = S.n_short, ts = seedless ? kNoTerm : S.n_long;
        const uint32_t j0 = row_lo >> kTileShift, j1 = (row_hi - 1) >> kTileShift;
        const uint32_t nt = j1 - j0 + 1;
        // ---------------- short-term tile tables (probes of short terms)
#ifdef HM_SEED_STATS
        const long long c_tab = clock64();
#endif
        short_tables(ix, S, S.order_list, n_short, stab, stride, j0, nt, cb);
#ifdef HM_SEED_STATS
        if (tid == 0) {
            SST(24, clock64() - c_tab);
            SST(25, S.pref[n_short]);
        }
#endif
#ifdef HM_SEED_STATS
        c_t1 = clock64();
#endif
        const float delta = static_cast<float>(m + 10) * 5.9604645e-08f + 1.5258789e-05f;  // (m+10) 2^-24 + 2^-16
        const float f_slack = 1.0f - 2.5f * delta;
        const float f_ub = 1.0f + 3.0f * delta;
        const ProbeCtx<Smem> sc{ix, a, S, stab, stride, j0, cb, k1, bb};
        auto full_score = [&](uint32_t row) {
            float A = 0.f;
            for (uint32_t i = 0; i < m; ++i) A += seed_probe(sc, i, row);
            return A;
        };

        // ---------------- 1. seeds: every posting of t* in the window.  sR[e] = the
        // row of its e-th posting; sA[e] = the row's complete score, or 0 for a
        // row proven unable to reach the admission threshold (0 never exceeds a
        // real score, so the k-th largest sA stays a valid lower bound)
        const uint64_t sw0 = seedless ? 0ull : S.t_wlo[ts];
        const uint32_t n_seed = seedless ? 0u : static_cast<uint32_t>(S.t_end[ts] - sw0);
        const bool seed_sm = n_seed <= kSeedSmemMax;
        float* const sA = seed_sm ? S.acc : gA;
        uint32_t* const sR = seed_sm ? reinterpret_cast<uint32_t*>(S.acc + kSeedSmemMax)
                                     : reinterpret_cast<uint32_t*>(gA) + a.seed_half;  // seed rows
#ifndef HM_SEED_KP
#define HM_SEED_KP 4
#endif
        constexpr int kP = HM_SEED_KP;  // rows per lane, probed together
        // segments of postings (a term's range in one tile, or a short term's
        // range in a chunk) flattened by an exclusive scan of their lengths:
        // every posting of a segment list is then one independent load
        uint64_t* const seg_b = reinterpret_cast<uint64_t*>(S.acc + 2 * kHashSlots);
        uint32_t* const seg_pref = reinterpret_cast<uint32_t*>(seg_b + kMaxSeg);
        uint32_t* const seg_meta = seg_pref + kMaxSeg + 1;
        auto seg_scan = [&](uint32_t nseg) {  // seg_pref: lengths -> exclusive prefix; + total
            __syncthreads();
            if (warp == 0) {
                constexpr uint32_t kPer = kMaxSeg / 32;
                uint32_t loc = 0;
                for (uint32_t u = 0; u < kPer; ++u) {
                    const uint32_t x = lane * kPer + u;
                    loc += x < nseg ? seg_pref[x] : 0u;
                }
                const uint32_t incl = warp_incl_scan(loc);
                uint32_t run = incl - loc;
                for (uint32_t u = 0; u < kPer; ++u) {
                    const uint32_t x = lane * kPer + u;
                    if (x < nseg) {
                        const uint32_t l = seg_pref[x];
                        seg_pref[x] = run;
                        run += l;
                    }
                }
                if (lane == 31) seg_pref[nseg] = incl;
            }
            __syncthreads();
        };
        auto seg_find = [&](uint32_t f, uint32_t nseg) {  // largest s with seg_pref[s] <= f
            uint32_t lo = 0, hi = nseg;
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (seg_pref[mid] <= f) lo = mid;
                else hi = mid;
            }
            return lo;
        };
        if (seedless) {
        } else if (S.t_slot[ts] < 0) {
#pragma unroll 4
            for (uint32_t e = tid; e < n_seed; e += kCons) sR[e] = __ldg(ix.post + sw0 + e) >> cb;
        } else {  // a long seed term: rows from the tile offsets, tiles as segments
            const uint32_t* tb = tile_row(ix, S.t_slot[ts]);
            const uint64_t s0 = S.t_start[ts], sw1 = S.t_end[ts];
            for (uint32_t jb = j0; jb <= j1; jb += kMaxSeg) {
                const uint32_t ns = min(j1 - jb + 1, kMaxSeg);
                for (uint32_t x = tid; x < ns; x += kCons) {
                    const uint64_t b = max(s0 + __ldg(tb + static_cast<uint64_t>(jb + x) * kSubPerTile), sw0);
                    const uint64_t e = min(s0 + __ldg(tb + static_cast<uint64_t>(jb + x + 1) * kSubPerTile), sw1);
                    seg_b[x] = b;
                    seg_pref[x] = e > b ? static_cast<uint32_t>(e - b) : 0u;
                }
                seg_scan(ns);
                const uint32_t total = seg_pref[ns];
                for (uint32_t f0 = tid; f0 < total; f0 += 4 * kCons) {
                    uint64_t g[4];
                    uint32_t jt[4], p[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint32_t f = f0 + u * kCons;
                        const uint32_t sg = seg_find(f, ns);
                        g[u] = seg_b[sg] + (f - seg_pref[sg]);
                        jt[u] = jb + sg;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) p[u] = f0 + u * kCons < total ? __ldg(ix.post + g[u]) : 0u;
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (f0 + u * kCons < total) sR[g[u] - sw0] = (jt[u] << kTileShift) + (p[u] >> kCodeBitsLong);
                }
                __syncthreads();
            }
        }
#ifdef HM_SEED_STATS
        __syncthreads();
        if (tid == 0) SST(26, clock64() - c_t1);  // seeds collected
#endif
        // t*'s own contribution to seed e (its posting's code, no probe)
        auto seed_imp = [&](uint32_t e) -> float {
            const uint32_t p = __ldg(ix.post + sw0 + e);
            const uint32_t row = sR[e];
            float w;
            if (S.t_slot[ts] >= 0) {
                const uint32_t code = p & kEscLong;
                w = code < ix.n_codes ? code_w(sc, code)
                                      : impact32(static_cast<double>(__ldg(ix.tf + sw0 + e)),
                                                 static_cast<double>(__ldg(ix.doc_lens + row)), ix.avgdl, k1, bb);
            } else {
                const uint32_t code = p & ix.esc_short;
                w = code < ix.n_codes_short ? S.w32s[code]
                                            : impact32(static_cast<double>(__ldg(ix.tf + sw0 + e)),
                                                       static_cast<double>(__ldg(ix.doc_lens + row)), ix.avgdl, k1,
                                                       bb);
            }
            return S.t_cu[ts] * w;
        };
        // bound of the terms other than t* still unprobed: probes run in
        // bound-descending order, so after the j largest bounds the rest is the
        // ascending prefix msorder[0 .. m-1-j) without t* (rounded up)
        if (warp == 0) {
            const uint32_t i = static_cast<uint32_t>(lane) < m ? S.msorder[lane] : 0u;
            float v = static_cast<uint32_t>(lane) < m && i != ts ? S.t_ms[i] : 0.f;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const float nb = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += nb;
            }
            if (static_cast<uint32_t>(lane) < m) S.rem_ub[lane + 1] = v * 1.00001f;
            if (lane == 0) S.rem_ub[0] = 0.f;
        }
        __syncthreads();
        // score rows e_u (u < kP, bit u of vm): every term (full) or, with
        // early exit, t*'s impact first and the others by descending bound,
        // dropping a row once (partial + unprobed bound) (1 + 3 delta) < thr
        auto score_seeds = [&](const uint32_t (&eu)[kP], uint32_t vm, bool early, float thr) {
            if (!vm) return;
            RowsN<kP> rw;
#pragma unroll
            for (int u = 0; u < kP; ++u) rw.r[u] = (vm >> u) & 1u ? sR[eu[u]] : 0u;
            float A[kP] = {};
            uint32_t live = vm;
            if (!early) {  // t*'s contribution from the seed's own posting, the others probed
#pragma unroll
                for (int u = 0; u < kP; ++u)
                    if ((vm >> u) & 1u) A[u] = seed_imp(eu[u]);
                for (uint32_t i = 0; i < m; ++i) {
                    if (i == ts) continue;
                    SCNT(c_sp, __popc(vm));
                    SCNT(c_ep, kP);
                    const ValsN<kP> x = seed_probeN<Smem, kP>(sc, i, rw, vm);
#pragma unroll
                    for (int u = 0; u < kP; ++u) A[u] += x.v[u];
                }
            } else {
#pragma unroll
                for (int u = 0; u < kP; ++u)
                    if ((vm >> u) & 1u) A[u] = seed_imp(eu[u]);
                for (int j = static_cast<int>(m) - 1; j >= 0 && live; --j) {
                    const uint32_t i = S.msorder[j];
                    if (i == ts) continue;
                    const float rem = S.rem_ub[j + 1];  // bounds of msorder[0..j] but t*
#pragma unroll
                    for (int u = 0; u < kP; ++u)
                        if (((live >> u) & 1u) && (A[u] + rem) * f_ub < thr) live &= ~(1u << u);
                    if (!live) break;
                    SCNT(c_sp, __popc(live));
                    SCNT(c_ep, kP);
                    const ValsN<kP> x = seed_probeN<Smem, kP>(sc, i, rw, live);
#pragma unroll
                    for (int u = 0; u < kP; ++u)
                        if ((live >> u) & 1u) A[u] += x.v[u];
                }
            }
#pragma unroll
            for (int u = 0; u < kP; ++u)
                if ((vm >> u) & 1u) sA[eu[u]] = (live >> u) & 1u ? A[u] : 0.f;
        };
        // pass over the seeds: select(e) picks the rows of this pass
        auto seed_pass = [&](auto select, bool early, float thr) {
            for (uint32_t e = tid; e < n_seed; e += kP * kCons) {
                uint32_t eu[kP], vm = 0;
#pragma unroll
                for (int u = 0; u < kP; ++u) {
                    eu[u] = e + u * kCons;
                    if (eu[u] < n_seed && select(eu[u])) vm |= 1u << u;
                }
                score_seeds(eu, vm, early, thr);
            }
        };
#ifndef HM_SEED_FULL
#define HM_SEED_FULL 2048
#endif
#ifndef HM_BOUND_FULL
#define HM_BOUND_FULL 512  // (2,048 / 1,024 / 256 / 128 with or without (b): profiles/r02_shard_scaling.md)
#endif
#ifndef HM_BOUND_SKIP_B
#define HM_BOUND_SKIP_B 1
#endif
        // (the bound pass of doc shards may score fewer seeds completely: its
        // k best only need to be good, the other shards add theirs)
        const uint32_t n_full = max(static_cast<uint32_t>(bonly ? HM_BOUND_FULL : HM_SEED_FULL), 8u * k);
        float L = 0.f;
#ifdef HM_SEED_STATS
        const long long c_s0 = clock64();
#endif
        if (n_seed <= n_full) {  // few seeds: every one complete
            seed_pass([](uint32_t) { return true; }, false, 0.f);
            __syncthreads();
        } else {
            // (a) the n_full seeds with the largest t* impact, complete: L0
#pragma unroll 4
            for (uint32_t e = tid; e < n_seed; e += kCons) sA[e] = seed_imp(e);
            __syncthreads();
            const float v0 = block_kth_largest<kCons>(sA, n_seed, n_full, S.hist, S.sel, [] { __syncthreads(); }, 16);
            if (tid == 0) S.total = 0;
            __syncthreads();
            // rows left for (b) hold the smallest denormal: below every complete
            // score (>= n_full >= k complete rows are normal and positive), so
            // the k-th largest is the complete rows' lower bound L0
            constexpr uint32_t kTodo = 1u;
            // the selected seeds are compacted into a list first (the candidate
            // lists' area, free until admission), so the probes run densely --
            // scattered picks would keep most lanes of every probe round idle
            uint32_t* const pick = &S.cl_row[0][0];
            constexpr uint32_t kPickCap = 2u * kConsWarps * CAPW;  // cl_row + cl_val
            static_assert(offsetof(Smem, cl_val) == offsetof(Smem, cl_row) + sizeof(uint32_t) * kConsWarps * CAPW,
                          "the candidate lists are contiguous");
            const uint32_t cap = min(2u * n_full, kPickCap);
            for (uint32_t e = tid; e < n_seed; e += kCons) {
                const uint32_t pos = sA[e] >= v0 ? atomicAdd(&S.total, 1u) : cap;
                if (pos < cap) pick[pos] = e;
                else sA[e] = __uint_as_float(kTodo);
            }
            __syncthreads();
            const uint32_t npick = min(S.total, cap);
            for (uint32_t x = tid; x < npick; x += kP * kCons) {
                uint32_t eu[kP], vm = 0;
#pragma unroll
                for (int u = 0; u < kP; ++u) {
                    const uint32_t xi = x + u * kCons;
                    eu[u] = xi < npick ? pick[xi] : 0u;
                    vm |= (xi < npick ? 1u : 0u) << u;
                }
                score_seeds(eu, vm, false, 0.f);
            }
            __syncthreads();
#ifdef HM_SEED_STATS
            if (tid == 0) SST(27, clock64() - c_s0);  // (a) incl. its selection
#endif
            const float L0 = block_kth_largest<kCons>(sA, n_seed, k, S.hist, S.sel, [] { __syncthreads(); }, 8);
            const float te0 = fmaxf(L0 * f_slack, kFltMin);
            // (b) the other seeds with early exit against te0 (the bound pass of
            // doc shards may stop at (a): its k best need only be good)
            if (!(bonly && HM_BOUND_SKIP_B)) {
                seed_pass([&](uint32_t e) { return __float_as_uint(sA[e]) == kTodo; }, true, te0);
                __syncthreads();
            }
        }
        if (bonly) {  // the bound pass of doc-sharded search: the k best complete seed scores
            // (the multiset {scores > L} + (k - that count) x L, L the exact k-th
            // largest; zeros when there are fewer than k seeds): the k-th largest
            // over every shard's k values is a k-th score of real documents
            if (n_seed >= k) L = block_kth_largest<kCons>(sA, n_seed, k, S.hist, S.sel, [] { __syncthreads(); });
            if (tid == 0) S.total = 0;
            __syncthreads();
            float* ob = a.out_bound + static_cast<uint64_t>(qr) * k;
            for (uint32_t e = tid; e < n_seed; e += kCons)
                if (sA[e] > L) {
                    const uint32_t i = atomicAdd(&S.total, 1u);
                    if (i < k) ob[i] = sA[e];
                }
            __syncthreads();
            for (uint32_t i = S.total + tid; i < k; i += kCons) ob[i] = L;
            continue;
        }
#ifdef HM_SEED_STATS
        const long long c_s1 = clock64();
        if (tid == 0) {
            SST(28, c_s1 - c_s0);  // all seed scoring
            SST(29, n_seed > n_full ? 1 : 0);
        }
#endif
        if (n_seed >= k) L = block_kth_largest<kCons>(sA, n_seed, k, S.hist, S.sel, [] { __syncthreads(); }, 8);
#ifdef HM_SEED_STATS
        if (tid == 0) SST(30, clock64() - c_s1);  // final selection
#endif
        // the union's bound: every document of the union's top-k scores above it
        // (a k-th score of real documents of some shard, in the same domain)
        L = fmaxf(L, ext);
        const float te = fmaxf(L * f_slack, kFltMin);  // admission threshold (as the exhaustive kernel's)
        if (tid == 0) S.Lg = __float_as_uint(L);
#ifdef HM_SEED_STATS
        c_t2 = clock64();
        if (tid == 0) {
            SST(0, 1);
            SST(1, n_seed);
        }
#endif
        // ---------------- 2. non-essential terms: longest bound-ascending prefix
        // whose bound sum cannot reach te; the rest (but t*) must be enumerated
        if (warp == 0) {
            float v = static_cast<uint32_t>(lane) < m ? S.t_ms[S.msorder[lane]] : 0.f;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const float nb = __shfl_up_sync(0xffffffffu, v, o);
                if (lane >= o) v += nb;
            }
            const bool isne = static_cast<uint32_t>(lane) < m && v * f_ub < te;
            // t* is never non-essential: its postings are the seeds, and the
            // candidate pass recognises seed rows only by probing t* (a term
            // tied with t*'s bound can sort after it and stay essential).
            // The bound sum still includes t*: an over-estimate, safe.
            const uint32_t ne =
                __reduce_or_sync(0xffffffffu, isne ? 1u << S.msorder[lane] : 0u) & (ts < 32u ? ~(1u << ts) : ~0u);
            const uint32_t bal = __ballot_sync(0xffffffffu, isne);
            const float ub = bal ? __shfl_sync(0xffffffffu, v, 31 - __clz(bal)) : 0.f;
            if (lane == 0) S.ubne_q = ub;
            uint64_t ne_post = 0;
            if (lane == 0) {
                for (uint32_t i = 0; i < m; ++i)
                    if (i != ts && !((ne >> i) & 1u)) ne_post += S.t_end[i] - S.t_wlo[i];
                S.sel[0] = ne;  // reused: essential mask complement
                S.flood = ne_post > kEMax && !(a.flags & 32u) ? 2u : 0u;
            }
        }
        __syncthreads();
        if (S.flood == 2u) {  // too many essential postings: the exhaustive kernel
            // k seeds have complete scores S >= L here; in the sweep's domain
            // (baked impacts) each has A >= (1-delta) E >= S (1-delta)/(1+delta)
            // >= L (1 - 2 delta): a valid starting bound for its admission
            if (tid == 0) {
                SST(10, 1);
                hand_over(a, q, L * (1.0f - 2.0f * delta - 1e-6f));
            }
            continue;
        }
        const uint32_t ne = S.sel[0];
        // ---------------- 3./4. admission of seeds, then of essential candidates
        uint32_t nw = 0;
        float Lw = 0.f;
        bool flood = false;
        auto admit = [&](bool ok_in, uint32_t row, float A) {  // warp-synchronous
            if (nw > static_cast<uint32_t>(CAPW - 32)) {
                nw = warp_prune(S, warp, nw, k, Lw, f_slack);
                if (nw > static_cast<uint32_t>(CAPW - 32)) flood = true;
            }
            const float t = fmaxf(fmaxf(fmaxf(Lw, __uint_as_float(S.Lg)) * f_slack, te), kFltMin);
            const bool ok = ok_in && !flood && A >= t;
            const uint32_t bal = __ballot_sync(0xffffffffu, ok);
            if (ok) {
                const uint32_t pos = nw + __popc(bal & ((1u << lane) - 1u));
                S.cl_row[warp][pos] = row;
                S.cl_val[warp][pos] = A;
            }
            nw += __popc(bal);
            __syncwarp();
        };
        for (uint32_t e0 = warp * 32; e0 < n_seed && !flood; e0 += kConsWarps * 32) {
            const uint32_t e = e0 + lane;
            const bool v = e < n_seed;
            admit(v, v ? sR[e] : 0u, v ? sA[e] : 0.f);
        }
        const float ubne = S.ubne_q;
        // ---------------- essential candidates without probes: the postings of
        // the essential terms (t* and E') are accumulated per row in a
        // shared-memory hash table (row -> essential score A_E), chunk by chunk
        // of whole tiles sized to fill it about half; rows holding t* get -inf
        // (the seeds scored them completely).  A row then needs the
        // non-essential probes only if (A_E + U_NE)(1 + 3 delta) reaches the
        // threshold -- those run in bound-descending order with early exit --
        // and is admitted with the usual rule.  A table overflow hands the
        // query to the sweep with the seeds' bound.
        {
            // key = row, value = the row's essential score in fixed point
            // (2^-sx units, integer adds are native shared-memory atomics);
            // bit 31 flags a row holding t*
            uint32_t* hkey = reinterpret_cast<uint32_t*>(S.acc);
            uint32_t* hval = reinterpret_cast<uint32_t*>(S.acc) + kHashSlots;
            // per-chunk segments of the essential terms' postings: one per short
            // term (rows in the postings), one per (long term, tile) (rows need
            // the tile); flattened by an exclusive scan of their lengths
            uint64_t TE = 0;
            uint32_t n_el = 0, n_es = 0;
            for (uint32_t i = 0; i < m; ++i)
                if (!((ne >> i) & 1u)) {
                    TE += S.t_end[i] - S.t_wlo[i];
                    if (S.t_slot[i] < 0) ++n_es;
                    else ++n_el;
                }
#ifndef HM_HASH_FILL
#define HM_HASH_FILL 2  // postings per chunk = slots * HM_HASH_FILL / 4
#endif
            uint64_t tpc64 = TE ? (static_cast<uint64_t>(kHashSlots * HM_HASH_FILL / 4) * nt) / TE : nt;
            if (n_el && tpc64 > (kMaxSeg - n_es) / n_el) tpc64 = (kMaxSeg - n_es) / n_el;
            const uint32_t tpc = tpc64 < 1 ? 1u : tpc64 > nt ? nt : static_cast<uint32_t>(tpc64);
            __syncthreads();  // the seeds (possibly in this area) are admitted
            for (uint32_t x = tid; x < kHashSlots; x += kCons) {
                hkey[x] = kHashEmpty;
                hval[x] = 0u;
            }
            __syncthreads();
            // fixed-point scale: the E' bounds sum to at most 2^30 units, so a
            // row's sum stays below bit 31; rounding adds at most m/2 units --
            // read back rounded up by m units (an over-estimate, safe for both
            // the filter and admission), which must stay far inside the
            // selection slack: m 2^-sx <= 2^-20 L, else the sweep takes the query
            float UE = 0.f;
            uint32_t n_ep = 0;  // E' terms: none -> every candidate holds t* (no work)
            for (uint32_t i = 0; i < m; ++i)
                if (!((ne >> i) & 1u) && i != ts) {
                    UE += S.t_ms[i];
                    ++n_ep;
                }
            int ex = 0;
            frexpf(fmaxf(UE * 1.0001f, kFltMin), &ex);
            const int sx = 30 - ex;
            const float up = ldexpf(1.f, sx), down = ldexpf(1.f, -sx);
            const bool fix_ok = static_cast<float>(m) * down <= ldexpf(L, -20) && sx < 126 && sx > -126;
            if (n_ep && !fix_ok && tid == 0) S.flood = 2u;
            auto insert = [&](uint32_t row, uint32_t v) {
                uint32_t h = (row * 0x9E3779B1u) >> (32 - kHashBits);
                for (uint32_t pr = 0; pr < kHashSlots; ++pr) {
                    const uint32_t old = atomicCAS(hkey + h, kHashEmpty, row);
                    if (old == kHashEmpty || old == row) {
                        atomicAdd(hval + h, v);
                        return;
                    }
                    h = (h + 1) & (kHashSlots - 1);
                }
                S.flood = 2u;  // full: the sweep serves the query
            };
            constexpr uint32_t kPerWarp = kHashSlots / kConsWarps;
            const uint32_t region = warp * kPerWarp;
            __syncthreads();
#ifdef HM_SEED_STATS
            if (tid == 0 && n_ep) {
                SST(16, TE);
                SST(17, 1);
                SST(18, n_seed);
            }
#endif
            for (uint32_t c0 = j0; n_ep && c0 <= j1 && S.flood != 2u; c0 += tpc) {
                const uint32_t c1 = min(c0 + tpc - 1, j1);
                const uint32_t ntc = c1 - c0 + 1;
#ifdef HM_SEED_STATS
                long long h_t0 = clock64();
                if (tid == 0) SST(12, 1);
#endif
                // (a) segments [b, e) of every essential term in the chunk
                const uint32_t nseg = n_es + n_el * ntc;
                for (uint32_t x = tid; x < nseg; x += kCons) {
                    uint32_t i = 0, o = 0, tile = c0;
                    for (; i < m; ++i) {
                        if ((ne >> i) & 1u) continue;
                        const uint32_t c = S.t_slot[i] < 0 ? 1u : ntc;
                        if (x < o + c) {
                            tile = c0 + (x - o);
                            break;
                        }
                        o += c;
                    }
                    const uint64_t w0 = S.t_wlo[i], w1 = S.t_end[i], s0 = S.t_start[i];
                    uint64_t b, e;
                    if (S.t_slot[i] < 0) {
                        const uint32_t* tab = stab + static_cast<uint64_t>(S.t_spos[i]) * stride;
                        b = max(s0 + tab[c0 - j0], w0);
                        e = min(s0 + tab[c1 + 1 - j0], w1);
                    } else {
                        const uint32_t* tb = tile_row(ix, S.t_slot[i]);
                        b = max(s0 + __ldg(tb + static_cast<uint64_t>(tile) * kSubPerTile), w0);
                        e = min(s0 + __ldg(tb + static_cast<uint64_t>(tile + 1) * kSubPerTile), w1);
                    }
                    seg_b[x] = b;
                    seg_pref[x] = e > b ? static_cast<uint32_t>(e - b) : 0u;
                    seg_meta[x] = (i << 27) | tile;
                }
                seg_scan(nseg);
#ifdef HM_SEED_STATS
                if (tid == 0) SST(15, clock64() - h_t0);
#endif
                // (b) every posting of the chunk into the table: kU postings per
                // thread located and loaded together, then inserted
                const uint32_t total = seg_pref[nseg];
#ifndef HM_SEED_KU
#define HM_SEED_KU 4
#endif
                constexpr int kU = HM_SEED_KU;
                for (uint32_t f0 = tid; f0 < total; f0 += kU * kCons) {
                    uint32_t p[kU], meta[kU];
                    uint64_t g[kU];
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        const uint32_t f = f0 + u * kCons;
                        const uint32_t lo = seg_find(f, nseg);
                        g[u] = seg_b[lo] + (f - seg_pref[lo]);
                        meta[u] = seg_meta[lo];
                    }
#pragma unroll
                    for (int u = 0; u < kU; ++u) p[u] = f0 + u * kCons < total ? __ldg(ix.post + g[u]) : 0u;
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        if (f0 + u * kCons >= total) break;
                        const uint32_t i = meta[u] >> 27;
                        uint32_t row;
                        float v = 0.f;
                        if (S.t_slot[i] < 0) {
                            row = p[u] >> cb;
                            if (i != ts) {
                                const uint32_t code = p[u] & ix.esc_short;
                                v = S.t_cu[i] * (code < ix.n_codes_short
                                                     ? S.w32s[code]
                                                     : impact32(static_cast<double>(__ldg(ix.tf + g[u])),
                                                                static_cast<double>(__ldg(ix.doc_lens + row)),
                                                                ix.avgdl, k1, bb));
                            }
                        } else {
                            row = ((meta[u] & 0x7FFFFFFu) << kTileShift) + (p[u] >> kCodeBitsLong);
                            if (i != ts) {
                                const uint32_t code = p[u] & kEscLong;
                                v = S.t_cu[i] * (code < ix.n_codes
                                                     ? code_w(sc, code)
                                                     : impact32(static_cast<double>(__ldg(ix.tf + g[u])),
                                                                static_cast<double>(__ldg(ix.doc_lens + row)),
                                                                ix.avgdl, k1, bb));
                            }
                        }
                        insert(row, i == ts ? 0x80000000u : __float2uint_rn(v * up));
                    }
                }
                __syncthreads();
#ifdef HM_SEED_STATS
                long long h_t1 = clock64();
                if (tid == 0) SST(13, h_t1 - h_t0);
#endif
                if (S.flood == 2u) break;
                // (c) scan of warp w's slots: candidates (rows without t* whose
                // essential score + U_NE can reach the threshold) compacted to the
                // front of the region, every slot cleared
                uint32_t ncand = 0;
                {
                    const float tn = fmaxf(fmaxf(Lw, __uint_as_float(S.Lg)) * f_slack, te);
                    for (uint32_t g0 = 0; g0 < kPerWarp; g0 += 128) {
                        uint32_t r4[4], v4[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            r4[u] = hkey[region + g0 + 32 * u + lane];
                            v4[u] = hval[region + g0 + 32 * u + lane];
                        }
                        __syncwarp();
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            hkey[region + g0 + 32 * u + lane] = kHashEmpty;
                            hval[region + g0 + 32 * u + lane] = 0u;
                        }
                        __syncwarp();
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            // rows with t* (bit 31) were scored as seeds
                            const float ae = __fmul_ru(__uint2float_ru(v4[u] + m), down);
                            const bool ok = r4[u] != kHashEmpty && !(v4[u] >> 31) && (ae + ubne) * f_ub >= tn;
                            const uint32_t bal = __ballot_sync(0xffffffffu, ok);
                            if (ok) {
                                const uint32_t pos = region + ncand + __popc(bal & ((1u << lane) - 1u));
                                hkey[pos] = r4[u];
                                hval[pos] = __float_as_uint(ae);
                            }
                            ncand += __popc(bal);
                        }
                        __syncwarp();
                    }
                }
                SCNT(c_en, lane == 0 ? ncand : 0u);
                // (d) the candidates: non-essential terms by bound descending with
                // early exit, then admission
                for (uint32_t c = 0; c < ncand; c += 32 * kP) {
                    RowsN<kP> rw;
                    float A[kP];
                    uint32_t vm = 0;
#pragma unroll
                    for (int u = 0; u < kP; ++u) {
                        const uint32_t x = c + 32 * u + lane;
                        rw.r[u] = x < ncand ? hkey[region + x] : 0u;
                        A[u] = x < ncand ? __uint_as_float(hval[region + x]) : 0.f;
                        vm |= (x < ncand ? 1u : 0u) << u;
                    }
                    const float tn = fmaxf(fmaxf(Lw, __uint_as_float(S.Lg)) * f_slack, te);
                    uint32_t live = vm;
                    for (int jn = static_cast<int>(m) - 1; jn >= 0 && live && ne; --jn) {
                        const uint32_t i2 = S.msorder[jn];
                        if (!((ne >> i2) & 1u)) continue;
                        const float rem = S.rem_ub[jn + 1];  // bounds of msorder[0..jn] but t*
#pragma unroll
                        for (int u = 0; u < kP; ++u)
                            if (((live >> u) & 1u) && (A[u] + rem) * f_ub < tn) live &= ~(1u << u);
                        if (!live) break;
                        SCNT(c_np, __popc(live));
                        SCNT(c_ns, kP);
                        const ValsN<kP> xv = seed_probeN<Smem, kP>(sc, i2, rw, live);
#pragma unroll
                        for (int u = 0; u < kP; ++u)
                            if ((live >> u) & 1u) A[u] += xv.v[u];
                    }
#pragma unroll
                    for (int u = 0; u < kP; ++u) admit((live >> u) & 1u, rw.r[u], A[u]);
                    if (flood) break;
                }
                __syncwarp();
                for (uint32_t x = lane; x < ncand; x += 32) {
                    hkey[region + x] = kHashEmpty;
                    hval[region + x] = 0u;
                }
                if (flood && lane == 0) atomicMax(&S.flood, 1u);
                __syncthreads();
#ifdef HM_SEED_STATS
                if (tid == 0) SST(14, clock64() - h_t1);
#endif
                if (S.flood) break;
            }
        }
        if (lane == 0) {
            S.n_w[warp] = nw;
            if (flood) atomicMax(&S.flood, 1u);
        }
#ifdef HM_SEED_STATS
        {
            const uint32_t vs[5] = {c_sp, c_en, c_ep, c_np, c_ns};
            for (int z = 0; z < 5; ++z) {
                uint32_t v = vs[z];
                for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0) SST(z < 4 ? 2 + z : 31, v);
            }
        }
#endif
        __syncthreads();
#ifdef HM_SEED_STATS
        c_t3 = clock64();
#endif
        if (S.flood) {  // the lists cannot hold the near-ties (1) or the hash table
                        // overflowed (2, with the seeds' bound): the exhaustive kernel
            if (tid == 0) {
                if (S.flood == 2u) hand_over(a, q, L * (1.0f - 2.0f * delta - 1e-6f));
                else hand_over(a, q);
            }
            __syncthreads();
            if (tid < kConsWarps) S.n_w[tid] = 0;
            continue;
        }
        finish_query<CAPW>(ix, a, S, q, m, k, nw, f_slack, k1, bb, stab, stride, j0, cb);
#ifdef HM_SEED_STATS
        if (tid == 0) {
            SST(6, c_t1 - c_t0);
            SST(7, c_t2 - c_t1);
            SST(8, c_t3 - c_t2);
            SST(9, clock64() - c_t3);
            SST(11, 1);
        }
#endif
    }
#ifdef HM_SEED_STATS  // tail: CTA exit times (globaltimer, ns; tools/seed_tail.py)
    if (tid == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        atomicMax(&g_seed_stats[20], t);
        atomicMin(&g_seed_stats[21], t);
        SST(22, t >> 10);
        SST(23, 1);
    }
#endif
}

template <int CAPW>
static cudaError_t seed_attr() {
    static bool done = false;
    if (done) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(search_seed_kernel<CAPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(sizeof(SeedSmem<CAPW>)));
    if (e == cudaSuccess) done = true;
    return e;
}

// `cap`: CTAs the per-CTA scratch (a.seed_scratch, a.stab) was sized for.
// The pass is latency-bound (dependent probe chains): as many resident CTAs
// as registers allow, one wave.
template <int CAPW>
static cudaError_t launch_seed_w(const DevIndex& ix, const BatchArgs& a, int cap, cudaStream_t st) {
    cudaError_t e = seed_attr<CAPW>();
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, search_seed_kernel<CAPW>, kCons,
                                                             sizeof(SeedSmem<CAPW>))) != cudaSuccess)
        return e;
    const int grid = per_sm * sms < cap ? per_sm * sms : cap;
    search_seed_kernel<CAPW><<<grid, kCons, sizeof(SeedSmem<CAPW>), st>>>(ix, a);
    return cudaGetLastError();
}

cudaError_t launch_search_seed(const DevIndex& ix, const BatchArgs& a, int cap, cudaStream_t st) {
    return a.k <= FastCfg<192>::kMaxKServed ? launch_seed_w<192>(ix, a, cap, st) : launch_seed_w<320>(ix, a, cap, st);
}

}  // namespace hm

#ifdef HM_SEED_STATS
extern "C" int hm_seed_stats(unsigned long long* out, int reset) {
    if (cudaMemcpyFromSymbol(out, hm::g_seed_stats, sizeof(hm::g_seed_stats)) != cudaSuccess) return -1;
    if (reset) {
        unsigned long long z[40] = {};
        z[21] = ~0ull;  // running minimum of the CTA exit times
        cudaMemcpyToSymbol(hm::g_seed_stats, z, sizeof(z));
    }
    return 0;
}
#endif
