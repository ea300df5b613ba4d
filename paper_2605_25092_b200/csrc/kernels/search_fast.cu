// search_fast_kernel: the fused BM25 hot path on sm_100a.
//
// One CTA (16 warps) owns one query at a time (persistent, LPT order) and
// sweeps its row window in kTile = 16384-row tiles.  Warp w OWNS rows
// [1024 w, 1024 w + 1024) of every tile:
//   * long terms: the sub-tile table gives, for every 1024-row sub-tile, the
//     offset of its first posting, so a warp streams exactly its own
//     contiguous sub-range of each term's postings straight from HBM/L2 with
//     8 independent coalesced loads per lane in flight
//     (ld.global.nc.L1::no_allocate);
//   * short terms: the tile segment (a few postings) is read by every warp and
//     filtered by row;
//   * fp32 scores accumulate in shared memory with plain read-modify-writes --
//     no other warp touches these rows, so there are no atomics and no CTA
//     barrier anywhere in the tile loop;
//   * after a tile the warp scans its 1024 accumulators: docs that can still
//     reach the top-k join the warp's candidate list, the accumulators are
//     zeroed (pitfall-3 sentinel reset, src/twophase.cpp:24-27).  A warp prunes
//     its list locally and publishes its k-th score to a CTA-wide lower bound
//     Lg that every warp uses as admission threshold.
// At the end of the query (one CTA barrier) the lists are merged, the
// survivors are rescored exactly in fp64 in the reference's operation and
// accumulation order (src/csr_index.cpp:10-15, 87-101), ranked by
// (score desc, DocId asc) (include/hybrid/types.hpp:21-25), and the Margin
// confidence + skip decision are written (src/cascade.cpp:15-21, 79-84).
// See bm25_search.cu for the exactness argument of the fp32 selection.
#include <cstdlib>

#include "hm_device.cuh"
#include "hm_launch.h"
#include "hm_ptx.cuh"

namespace hm {

constexpr int kCons = kThreads;           // 512 threads
constexpr int kConsWarps = kCons / 32;    // 16: warp w owns sub-tile w of a tile
constexpr int kFastTerms = 32;            // plan size served by this kernel
constexpr int kR = 8;                     // postings per lane in flight
static_assert(kConsWarps == kSubPerTile, "one warp per 1024-row sub-tile");

// per-warp candidate list capacity -> largest k served (room for one scan
// round of 128 appends plus near-ties)
template <int CAPW>
struct FastCfg {
    static constexpr int kMaxKServed = CAPW == 192 ? 32 : 128;
};

template <int CAPW>
struct __align__(16) FastSmem {
    float acc[kTile];
    float w32[kMaxCodes];                  // [kCodeMask] = 0
    uint32_t cl_row[kConsWarps][CAPW];     // per-warp candidate lists
    float cl_val[kConsWarps][CAPW];
    uint64_t t_start[kFastTerms], t_wlo[kFastTerms], t_end[kFastTerms];
    double t_idf[kFastTerms];
    uint32_t t_mult[kFastTerms];
    float t_c32[kFastTerms];
    int32_t t_slot[kFastTerms];
    uint8_t t_esc[kFastTerms];             // long term has escaped postings
    uint32_t wsub[2][kConsWarps][kFastTerms][2];  // warp's sub-range of each long term (tile parity)
    uint16_t order_list[kFastTerms];       // long terms, then short terms
    uint32_t pref[kFastTerms + 1];         // short-window prefix sums / gather offsets
    uint32_t hist[256];
    uint32_t sel[2];
    uint32_t n_w[kConsWarps];
    uint64_t post;
    uint32_t q, n_long, n_short, bad, n_surv, flood, Lg, total;
};

struct SurvView {
    double* E;
    uint64_t* id;
    uint32_t* row;
};
constexpr int kSurvBytes = 20 * kSurvCap;

__device__ __forceinline__ float esc_w(const DevIndex& ix, uint64_t gidx, uint32_t row, double k1,
                                       double b) {
    return impact32(static_cast<double>(__ldg(ix.tf + gidx)),
                    static_cast<double>(__ldg(ix.doc_lens + row)), ix.avgdl, k1, b);
}

// ---------------------------------------------------------------- per-warp list
// Raise the warp's k-th bound from its own list (exact k-th largest by a
// binary search over the float bit pattern, values are >= 0), keep the
// admissible entries (>= max(Lw, Lg) * slack, stable compaction), publish the
// bound to the CTA-wide Lg.  Warp-synchronous; returns the new list length.
template <int CAPW>
__device__ uint32_t warp_prune(FastSmem<CAPW>& S, int w, uint32_t n, uint32_t k, float& Lw, float slack) {
    const int lane = threadIdx.x & 31;
    uint32_t* rows = S.cl_row[w];
    float* vals = S.cl_val[w];
    constexpr int R = CAPW / 32;
    float v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t i = lane + 32 * r;
        v[r] = i < n ? vals[i] : -1.f;
    }
    if (n >= k) {
        uint32_t lo = 0, hi = 0x7F800001u;  // count(>= lo) >= k > count(>= hi)
        while (hi - lo > 1) {
            const uint32_t mid = lo + ((hi - lo) >> 1);
            const float t = __uint_as_float(mid);
            uint32_t c = 0;
#pragma unroll
            for (int r = 0; r < R; ++r) c += v[r] >= t;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
            if (c >= k) lo = mid;
            else hi = mid;
        }
        Lw = fmaxf(Lw, __uint_as_float(lo));
        if (lane == 0) atomicMax(&S.Lg, __float_as_uint(Lw));
    }
    const float thr = fmaxf(Lw, __uint_as_float(S.Lg)) * slack;
    uint32_t keep = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t i = lane + 32 * r;
        const bool ok = i < n && v[r] >= thr;
        const uint32_t bal = __ballot_sync(0xffffffffu, ok);
        const uint32_t row = i < n ? rows[i] : 0u;
        __syncwarp();
        if (ok) {
            const uint32_t pos = keep + __popc(bal & ((1u << lane) - 1));
            rows[pos] = row;
            vals[pos] = v[r];
        }
        keep += __popc(bal);
        __syncwarp();
    }
    return keep;
}

// Accumulate one contiguous posting range of a long term (the warp's own rows)
// into the tile accumulators: 8 independent coalesced loads per lane in
// flight, then plain RMWs (rows of one term are distinct and no other warp
// owns them).  CLIP: the tile is cut by the row window; ESC: the term has
// postings whose (tf, len) pair is outside the code table (code kEscLong,
// which masks to kCodeMask whose impact is 0; their exact impact is added
// separately).
template <bool CLIP, bool ESC>
__device__ __forceinline__ void range_rmw(float* __restrict__ acc, const float* __restrict__ w32,
                                          const uint32_t* __restrict__ pb, uint32_t n, float c,
                                          uint32_t rlo, uint32_t rn, const DevIndex& ix,
                                          uint64_t gbase, uint32_t base, double k1, double b) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t o = 0;
    for (; o + 32 * kR <= n; o += 32 * kR) {
        uint32_t p[kR];
#pragma unroll
        for (int u = 0; u < kR; ++u) p[u] = ldg_stream(pb + o + u * 32 + lane);
        float av[kR], w[kR];
#pragma unroll
        for (int u = 0; u < kR; ++u) {
            w[u] = w32[p[u] & kCodeMask];
            if (CLIP && (p[u] >> kCodeBitsLong) - rlo >= rn) w[u] = 0.f;
            av[u] = acc[p[u] >> kCodeBitsLong];
        }
#pragma unroll
        for (int u = 0; u < kR; ++u) acc[p[u] >> kCodeBitsLong] = __fmaf_rn(c, w[u], av[u]);
        if (ESC) {
            bool e = false;
#pragma unroll
            for (int u = 0; u < kR; ++u) e |= (p[u] & kEscLong) == kEscLong;
            if (__any_sync(0xffffffffu, e)) {
#pragma unroll
                for (int u = 0; u < kR; ++u) {
                    const uint32_t loc = p[u] >> kCodeBitsLong;
                    if ((p[u] & kEscLong) == kEscLong && (!CLIP || loc - rlo < rn))
                        acc[loc] += c * impact32(static_cast<double>(__ldg(ix.tf + gbase + o + u * 32 + lane)),
                                                 static_cast<double>(__ldg(ix.doc_lens + base + loc)),
                                                 ix.avgdl, k1, b);
                }
            }
        }
    }
    if (o < n) {  // remainder (< 256 postings): all of its loads in flight at once
        uint32_t p[kR];
#pragma unroll
        for (int u = 0; u < kR; ++u) {
            const uint32_t e = o + u * 32 + lane;
            p[u] = e < n ? ldg_stream(pb + e) : kCodeMask;
        }
#pragma unroll
        for (int u = 0; u < kR; ++u) {
            if (o + u * 32 >= n) break;  // warp-uniform
            const uint32_t e = o + u * 32 + lane;
            const uint32_t loc = p[u] >> kCodeBitsLong;
            float w = w32[p[u] & kCodeMask];
            if (CLIP && loc - rlo >= rn) w = 0.f;
            if (ESC && e < n && (p[u] & kEscLong) == kEscLong && (!CLIP || loc - rlo < rn))
                w = impact32(static_cast<double>(__ldg(ix.tf + gbase + e)),
                             static_cast<double>(__ldg(ix.doc_lens + base + loc)), ix.avgdl, k1, b);
            if (e < n) acc[loc] = __fmaf_rn(c, w, acc[loc]);
        }
    }
}


// Software-pipelined streaming: a "step" is up to 32*kR postings of one long
// term's range; the loads of step s+1 are issued before step s is applied, so
// two steps (and two terms at term boundaries) are in flight per lane.
__device__ __forceinline__ void step_load(uint32_t* p, const uint32_t* __restrict__ pb, uint32_t o,
                                          uint32_t n) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int u = 0; u < kR; ++u) {
        const uint32_t e = o + u * 32 + lane;
        p[u] = e < n ? ldg_stream(pb + e) : kCodeMask;  // padding: impact 0
    }
}

template <bool CLIP, bool ESC>
__device__ __forceinline__ void step_apply(float* __restrict__ acc, const float* __restrict__ w32,
                                           const uint32_t* p, uint32_t o, uint32_t n, float c,
                                           uint32_t rlo, uint32_t rn, const DevIndex& ix,
                                           uint64_t gbase, uint32_t base, double k1, double b) {
    const uint32_t lane = threadIdx.x & 31;
    if (o + 32 * kR <= n) {  // full step: every element valid
        float av[kR], w[kR];
#pragma unroll
        for (int u = 0; u < kR; ++u) {
            w[u] = w32[p[u] & kCodeMask];
            if (CLIP && (p[u] >> kCodeBitsLong) - rlo >= rn) w[u] = 0.f;
            av[u] = acc[p[u] >> kCodeBitsLong];
        }
#pragma unroll
        for (int u = 0; u < kR; ++u) acc[p[u] >> kCodeBitsLong] = __fmaf_rn(c, w[u], av[u]);
    } else {  // partial step: rows of one term are distinct, so element order is free
#pragma unroll
        for (int u = 0; u < kR; ++u) {
            if (o + u * 32 >= n) break;  // warp-uniform
            const uint32_t loc = p[u] >> kCodeBitsLong;
            float w = w32[p[u] & kCodeMask];
            if (CLIP && loc - rlo >= rn) w = 0.f;
            if (o + u * 32 + lane < n) acc[loc] = __fmaf_rn(c, w, acc[loc]);
        }
    }
    if (ESC) {  // escaped postings: exact (tf, len) from HBM, added once
        bool e = false;
#pragma unroll
        for (int u = 0; u < kR; ++u) e |= o + u * 32 + lane < n && (p[u] & kEscLong) == kEscLong;
        if (__any_sync(0xffffffffu, e)) {
#pragma unroll
            for (int u = 0; u < kR; ++u) {
                const uint32_t el = o + u * 32 + lane;
                const uint32_t loc = p[u] >> kCodeBitsLong;
                if (el < n && (p[u] & kEscLong) == kEscLong && (!CLIP || loc - rlo < rn))
                    acc[loc] += c * impact32(static_cast<double>(__ldg(ix.tf + gbase + el)),
                                             static_cast<double>(__ldg(ix.doc_lens + base + loc)),
                                             ix.avgdl, k1, b);
            }
        }
    }
}

// ---------------------------------------------------------------- kernel
template <int CAPW>
__global__ void __launch_bounds__(kCons, CAPW == 192 ? 2 : 1) search_fast_kernel(DevIndex ix, BatchArgs a) {
    using Smem = FastSmem<CAPW>;
    constexpr int kGatherBytes = 8 * kConsWarps * CAPW;
    static_assert(kSurvBytes <= kGatherBytes && kGatherBytes <= static_cast<int>(sizeof(float)) * kTile,
                  "epilogue buffers fit in the accumulator array");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Smem& S = *reinterpret_cast<Smem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    auto csync = [] { __syncthreads(); };
    const uint32_t cb = ix.code_bits;
    const uint32_t row_lo = a.row_lo, row_hi = a.row_hi;
    const double k1 = a.k1, bb = a.b;
    const uint32_t stride = a.stab_stride;
    uint32_t* stab = a.stab + static_cast<uint64_t>(blockIdx.x) * kMaxTerms * stride;
    const uint32_t kmax = FastCfg<CAPW>::kMaxKServed;

    for (int i = tid; i < kTile; i += kCons) S.acc[i] = 0.f;
    for (int i = tid; i < kMaxCodes; i += kCons) S.w32[i] = a.w32[i];
    if (tid < kConsWarps) S.n_w[tid] = 0;
    if (tid == 0) S.Lg = 0u;
    float Lw = 0.f;  // this warp's own k-th lower bound

    for (;;) {
        __syncthreads();
        if (tid == 0) {
            const uint32_t w = atomicAdd(&a.counters[0], 1u);
            S.q = w < a.nq ? a.order[w] : kNoTerm;
        }
        __syncthreads();
        const uint32_t q = S.q;
        if (q == kNoTerm) break;
        const uint32_t poff = a.q_off[q];
        const uint32_t m = a.plan_len[q];
        const uint32_t k = a.k;
        if (m > kMaxTerms) {
            if (tid == 0) {
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
            S.t_c32[tid] = static_cast<float>(static_cast<double>(mult) * idf);
            S.t_slot[tid] = slot;
            S.t_esc[tid] = slot >= 0 ? ix.long_esc[slot] : 0;
        }
        __syncthreads();
        if (tid == 0) {
            uint64_t post = 0;
            uint32_t nl = 0, ns = 0, bad = 0;
            for (uint32_t i = 0; i < m; ++i) {
                post += S.t_end[i] - S.t_wlo[i];
                const double idf = S.t_idf[i];
                if (!(idf > 0.0) || !isfinite(idf)) bad = 1;
                if (S.t_slot[i] >= 0) S.order_list[nl++] = static_cast<uint16_t>(i);
            }
            S.pref[0] = 0;
            for (uint32_t i = 0; i < m; ++i)
                if (S.t_slot[i] < 0) {
                    S.order_list[nl + ns] = static_cast<uint16_t>(i);
                    S.pref[ns + 1] = S.pref[ns] + static_cast<uint32_t>(S.t_end[i] - S.t_wlo[i]);
                    ++ns;
                }
            S.post = post;
            S.n_long = nl;
            S.n_short = ns;
            S.bad = bad;
            S.flood = 0;
            if (!(a.flags & 2u)) S.Lg = 0u;  // HM_FLAG_DEBUG_NO_RESET skips the sentinel reset
        }
        if (!(a.flags & 2u)) {
            if (tid < kConsWarps) S.n_w[tid] = 0;
            Lw = 0.f;
        }
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
        if (n_short) {
            const uint32_t total = S.pref[n_short];
            for (uint32_t f = tid; f < total; f += kCons) {
                uint32_t lo = 0, hi = n_short;  // s: pref[s] <= f < pref[s+1]
                while (hi - lo > 1) {
                    const uint32_t mid = (lo + hi) >> 1;
                    if (S.pref[mid] <= f) lo = mid;
                    else hi = mid;
                }
                const uint32_t s = lo, i = S.order_list[n_long + s];
                const uint64_t w0 = S.t_wlo[i], w1 = S.t_end[i], s0 = S.t_start[i];
                const uint64_t g = w0 + (f - S.pref[s]);
                const int jt = static_cast<int>((__ldg(ix.post + g) >> cb) >> kTileShift) - static_cast<int>(j0);
                const int jp = g == w0 ? -1
                                       : static_cast<int>((__ldg(ix.post + g - 1) >> cb) >> kTileShift) -
                                             static_cast<int>(j0);
                uint32_t* tab = stab + static_cast<uint64_t>(s) * stride;
                for (int jj = jp + 1; jj <= jt; ++jj) tab[jj] = static_cast<uint32_t>(g - s0);
                if (g + 1 == w1)
                    for (int jj = jt + 1; jj <= static_cast<int>(nt); ++jj) tab[jj] = static_cast<uint32_t>(w1 - s0);
            }
            for (uint32_t x = tid; x < n_short * (nt + 1); x += kCons) {
                const uint32_t s = x / (nt + 1), jj = x % (nt + 1), i = S.order_list[n_long + s];
                if (S.t_wlo[i] == S.t_end[i])
                    stab[static_cast<uint64_t>(s) * stride + jj] = static_cast<uint32_t>(S.t_wlo[i] - S.t_start[i]);
            }
        }
        __syncthreads();

        // =============================================== tile sweep (per warp)
        const float delta = static_cast<float>(m + 10) * 5.9604645e-08f;  // (m+10) * 2^-24
        const float f_slack = 1.0f - 2.5f * delta;
        const uint32_t wr0 = static_cast<uint32_t>(warp) << kSubShift;  // my rows in a tile
        uint32_t nw = S.n_w[warp];
        bool flood = false;
        // my sub-range of every long term: lane x holds term x's for the next
        // tile (prefetched during the current one), the current tile's are in smem
        // my sub-range of every long term for a tile: copied global -> smem with
        // cp.async (no registers held), one tile ahead, double-buffered by parity
        auto load_sub = [&](uint32_t j) {
            if (static_cast<uint32_t>(lane) < n_long) {
                const uint32_t* tb = tile_row(ix, S.t_slot[S.order_list[lane]]);
                const uint64_t sub = static_cast<uint64_t>(j) * kSubPerTile + warp;
                uint32_t* dst = S.wsub[j & 1][warp][lane];
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(tb + sub) : "memory");
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst + 1)), "l"(tb + sub + 1) : "memory");
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        auto wait_sub = [&] {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            __syncwarp();
        };
        load_sub(j0);
        for (uint32_t j = j0; j <= j1; ++j) {
            const uint32_t base = j << kTileShift;
            const uint32_t R0 = max(base, row_lo);
            const uint32_t R1 = min(base + kTile, row_hi);
            const uint32_t rlo = R0 - base, rn = R1 - R0;
            const bool clip = rn != kTile;
            wait_sub();
            if (j < j1) load_sub(j + 1);
            const uint32_t (*wsub)[2] = S.wsub[j & 1][warp];
            // ---- long terms: my contiguous sub-range of each, straight from HBM/L2
            if (CAPW == 320) {
                // one CTA per SM (registers to spare): two steps in flight
                uint32_t x = 0, o = 0;
                auto range_n = [&](uint32_t xx) { return wsub[xx][1] - wsub[xx][0]; };
                auto range_p = [&](uint32_t xx) {
                    return ix.post + S.t_start[S.order_list[xx]] + wsub[xx][0];
                };
                while (x < n_long && range_n(x) == 0) ++x;
                uint32_t pc[kR];
                if (x < n_long) step_load(pc, range_p(x), 0, range_n(x));
                while (x < n_long) {
                    const uint32_t n = range_n(x);
                    uint32_t nx = x, no = o + 32 * kR;
                    if (no >= n) {
                        no = 0;
                        ++nx;
                        while (nx < n_long && range_n(nx) == 0) ++nx;
                    }
                    uint32_t pn[kR];
                    if (nx < n_long) step_load(pn, range_p(nx), no, range_n(nx));
                    const uint32_t i = S.order_list[x];
                    const float c = S.t_c32[i];
                    const uint64_t gb = S.t_start[i] + wsub[x][0];
                    const bool esc = S.t_esc[i] != 0;
                    if (!clip && !esc) step_apply<false, false>(S.acc, S.w32, pc, o, n, c, rlo, rn, ix, gb, base, k1, bb);
                    else if (!esc) step_apply<true, false>(S.acc, S.w32, pc, o, n, c, rlo, rn, ix, gb, base, k1, bb);
                    else if (!clip) step_apply<false, true>(S.acc, S.w32, pc, o, n, c, rlo, rn, ix, gb, base, k1, bb);
                    else step_apply<true, true>(S.acc, S.w32, pc, o, n, c, rlo, rn, ix, gb, base, k1, bb);
                    if (nx != x) __syncwarp();  // the next term may touch the same rows
#pragma unroll
                    for (int u = 0; u < kR; ++u) pc[u] = pn[u];
                    x = nx;
                    o = no;
                }
            } else {
                for (uint32_t x = 0; x < n_long; ++x) {
                    const uint32_t i = S.order_list[x];
                    const float c = S.t_c32[i];
                    const uint32_t rb = wsub[x][0], re = wsub[x][1];
                    const uint64_t B = S.t_start[i] + rb;
                    const uint32_t n = re - rb;
                    const bool esc = S.t_esc[i] != 0;
                    if (n) {
                        if (!clip && !esc) range_rmw<false, false>(S.acc, S.w32, ix.post + B, n, c, rlo, rn, ix, B, base, k1, bb);
                        else if (!esc) range_rmw<true, false>(S.acc, S.w32, ix.post + B, n, c, rlo, rn, ix, B, base, k1, bb);
                        else if (!clip) range_rmw<false, true>(S.acc, S.w32, ix.post + B, n, c, rlo, rn, ix, B, base, k1, bb);
                        else range_rmw<true, true>(S.acc, S.w32, ix.post + B, n, c, rlo, rn, ix, B, base, k1, bb);
                    }
                    __syncwarp();  // the next term may touch the same rows from other lanes
                }
            }
            // ---- short terms: the tile segment is small; every warp filters its rows
            for (uint32_t s = 0; s < n_short; ++s) {
                const uint32_t i = S.order_list[n_long + s];
                const float c = S.t_c32[i];
                const uint32_t* tab = stab + static_cast<uint64_t>(s) * stride;
                const uint64_t b = S.t_start[i] + tab[j - j0], e = S.t_start[i] + tab[j - j0 + 1];
                for (uint64_t b0 = b; b0 < e; b0 += 32) {
                    const uint64_t g = b0 + lane;
                    if (g < e) {
                        const uint32_t p = __ldg(ix.post + g);
                        const uint32_t local = (p >> cb) - base;
                        if (local - wr0 < (1u << kSubShift)) {
                            const uint32_t code = p & ix.esc_short;
                            const float w = code < ix.n_codes_short ? S.w32[code] : esc_w(ix, g, base + local, k1, bb);
                            S.acc[local] = __fmaf_rn(c, w, S.acc[local]);
                        }
                    }
                }
                __syncwarp();
            }
            // ---- scan my rows of the tile: admit candidates, zero accumulators
            const uint32_t r_lo = max(wr0, rlo), r_hi = min(wr0 + (1u << kSubShift), rlo + rn);
            float4* acc4 = reinterpret_cast<float4*>(S.acc);
            if (flood) {  // this query goes to the exact kernel: only keep acc clean
                if (r_lo < r_hi)
                    for (uint32_t z = (r_lo >> 2) + lane; z < ((r_hi + 3) >> 2); z += 32)
                        acc4[z] = make_float4(0.f, 0.f, 0.f, 0.f);
                __syncwarp();
                continue;
            }
            if (r_lo < r_hi) {
                const uint32_t v0 = r_lo >> 2, v1 = (r_hi + 3) >> 2;
                // admission: A > 0 and A >= L * slack  <=>  A >= max(L * slack, min denormal)
                float te = fmaxf(fmaxf(Lw, __uint_as_float(S.Lg)) * f_slack, 1.4e-45f);
                // append the qualifying entries of one float4 per lane (slow path)
                auto admit = [&](float4 x4, uint32_t v) {
                    if (nw > static_cast<uint32_t>(CAPW - 128)) {
                        nw = warp_prune(S, warp, nw, k, Lw, f_slack);
                        te = fmaxf(fmaxf(Lw, __uint_as_float(S.Lg)) * f_slack, 1.4e-45f);
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
                    const uint32_t r = base + 4 * v;
                    auto put = [&](bool ok, uint32_t row, float val) {
                        if (ok) {
                            S.cl_row[warp][slot] = row;
                            S.cl_val[warp][slot] = val;
                            ++slot;
                        }
                    };
                    put(q0, r, x4.x);
                    put(q1, r + 1, x4.y);
                    put(q2, r + 2, x4.z);
                    put(q3, r + 3, x4.w);
                    nw += __shfl_sync(0xffffffffu, incl, 31);
                    __syncwarp();
                };
                const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
                for (uint32_t vb = v0; vb < v1 && !flood; vb += 64) {
                    const uint32_t va = vb + lane, vc = vb + 32 + lane;
                    float4 xa = z4, xc = z4;
                    if (va < v1) {
                        xa = acc4[va];
                        acc4[va] = z4;
                    }
                    if (vc < v1) {
                        xc = acc4[vc];
                        acc4[vc] = z4;
                    }
                    const float mx = fmaxf(fmaxf(fmaxf(xa.x, xa.y), fmaxf(xa.z, xa.w)),
                                           fmaxf(fmaxf(xc.x, xc.y), fmaxf(xc.z, xc.w)));
                    if (__any_sync(0xffffffffu, mx >= te)) {
                        admit(xa, va);
                        if (!flood) admit(xc, vc);
                    }
                }
                if (flood)  // the query goes to the exact kernel: finish zeroing my rows
                    for (uint32_t z = v0 + lane; z < v1; z += 32) acc4[z] = z4;
                __syncwarp();
            }
        }
        if (lane == 0) {
            S.n_w[warp] = nw;
            if (flood) S.flood = 1;
        }
        csync();
        if (S.flood) {
            if (tid == 0) a.exact_list[atomicAdd(&a.counters[1], 1u)] = q;
            csync();
            if (tid < kConsWarps) S.n_w[tid] = 0;
            continue;
        }

        // ---------------- epilogue: merge lists, survivors, exact rescoring, ranking
        char* sp = reinterpret_cast<char*>(S.acc);
        float* gv = reinterpret_cast<float*>(sp);
        uint32_t* gr = reinterpret_cast<uint32_t*>(sp + 4 * kConsWarps * CAPW);
        if (tid == 0) {
            uint32_t t = 0;
            for (int w = 0; w < kConsWarps; ++w) {
                S.pref[w] = t;  // reused: gather offsets
                t += S.n_w[w];
            }
            S.total = t;
        }
        csync();
        {
            const uint32_t off = S.pref[warp];
            for (uint32_t i = lane; i < nw; i += 32) {
                gv[off + i] = S.cl_val[warp][i];
                gr[off + i] = S.cl_row[warp][i];
            }
        }
        csync();
        const uint32_t nc = S.total;
        float theta = 0.f;
        if (nc >= k) theta = block_kth_largest<kCons>(gv, nc, k, S.hist, S.sel, csync) * f_slack;
        if (warp == 0) {
            uint32_t w = 0;
            for (uint32_t b0 = 0; b0 < nc; b0 += 32) {
                const uint32_t i = b0 + lane;
                const bool keep = i < nc && gv[i] >= theta;
                const uint32_t bal = __ballot_sync(0xffffffffu, keep);
                const uint32_t pos = w + __popc(bal & ((1u << lane) - 1));
                if (keep && pos < kSurvCap) S.cl_row[0][pos] = gr[i];  // list area is free now
                w += __popc(bal);
                __syncwarp();
            }
            if (lane == 0) S.n_surv = w;
        }
        csync();
        const uint32_t ns = S.n_surv;
        for (int i = tid; i < kGatherBytes / 4; i += kCons) S.acc[i] = 0.f;  // zero for the next query
        if (tid < kConsWarps) S.n_w[tid] = 0;
        csync();
        if (ns > kSurvCap) {  // near-tie flood: the exact kernel takes the query
            if (tid == 0) a.exact_list[atomicAdd(&a.counters[1], 1u)] = q;
            continue;
        }
        SurvView sv{reinterpret_cast<double*>(sp), reinterpret_cast<uint64_t*>(sp + 8 * kSurvCap),
                    reinterpret_cast<uint32_t*>(sp + 16 * kSurvCap)};
        for (uint32_t i = tid; i < ns; i += kCons) sv.row[i] = S.cl_row[0][i];
        csync();
        // warp per survivor, lanes over plan terms; fp64 sum in plan order
        for (uint32_t s = warp; s < ns; s += kConsWarps) {
            const uint32_t row = sv.row[s];
            double E = 0.0;
            for (uint32_t t0 = 0; t0 < m; t0 += 32) {
                const uint32_t t = t0 + lane;
                double val = 0.0;
                bool present = false;
                if (t < m) {
                    double tf, dl;
                    if (find_posting(ix, S.t_slot[t], S.t_start[t], S.t_end[t], row, ix.code_tf,
                                     ix.code_len, &tf, &dl)) {
                        val = bm25_exact(tf, S.t_idf[t], dl, ix.avgdl, k1, bb);
                        present = true;
                    }
                }
                const uint32_t cnt = min(32u, m - t0);
                for (uint32_t u = 0; u < cnt; ++u) {
                    const double x = __shfl_sync(0xffffffffu, val, u);
                    const bool pr = __shfl_sync(0xffffffffu, present, u);
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
        csync();
        const uint32_t n2 = pow2_ceil(ns);
        for (uint32_t i = ns + tid; i < n2; i += kCons) {
            sv.E[i] = -INFINITY;
            sv.id[i] = ~0ull;
            sv.row[i] = 0;
        }
        csync();
        block_bitonic<kCons>(sv.E, sv.id, sv.row, n2, csync);
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
        csync();
        for (int i = tid; i < kSurvBytes / 4; i += kCons) S.acc[i] = 0.f;
    }
}

template <int CAPW>
static cudaError_t fast_attr() {
    static bool done = false;
    if (done) return cudaSuccess;
    const cudaError_t e = cudaFuncSetAttribute(search_fast_kernel<CAPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(sizeof(FastSmem<CAPW>)));
    if (e == cudaSuccess) done = true;
    return e;
}

// CAPW 192 (k <= 32): two 16-warp CTAs per SM; CAPW 320 (k <= 128): one.
// HM_FAST_CTAS=1 forces the one-CTA variant (experiments).
cudaError_t launch_search(const DevIndex& ix, const BatchArgs& a, int sms, cudaStream_t st) {
    static const bool force1 = [] {
        const char* e = getenv("HM_FAST_CTAS");
        return e && e[0] == '1';
    }();
    if (a.k <= FastCfg<192>::kMaxKServed && !force1) {
        const cudaError_t e = fast_attr<192>();
        if (e != cudaSuccess) return e;
        search_fast_kernel<192><<<2 * sms, kCons, sizeof(FastSmem<192>), st>>>(ix, a);
    } else {
        const cudaError_t e = fast_attr<320>();
        if (e != cudaSuccess) return e;
        search_fast_kernel<320><<<sms, kCons, sizeof(FastSmem<320>), st>>>(ix, a);
    }
    return cudaGetLastError();
}

cudaError_t search_occupancy_fast(int* blocks) {
    cudaError_t e = fast_attr<192>();
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, search_fast_kernel<192>, kCons,
                                                      sizeof(FastSmem<192>));
    if (e != cudaSuccess) return e;
    int b320 = 0;
    e = fast_attr<320>();
    if (e != cudaSuccess) return e;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b320, search_fast_kernel<320>, kCons,
                                                      sizeof(FastSmem<320>));
    if (*blocks < 2 || b320 < 1) return cudaErrorInvalidConfiguration;
    *blocks = 1;  // grid is sized in launch_search from the SM count
    return e;
}

size_t search_smem_bytes() { return sizeof(FastSmem<192>); }

}  // namespace hm
