// Device pieces of the fused search kernel (search_fast.cu): CTA geometry,
// shared-memory layout, per-warp candidate lists, the baked-posting
// decode/apply, the cp.async step pipeline and the exact epilogue.
#pragma once
#include "hm_device.cuh"
#include "hm_ptx.cuh"

namespace hm {
#ifdef HM_SEED_STATS  // development counters (scratch builds): [32..39] the epilogue's phases
static __device__ unsigned long long g_seed_stats[40];
#define FIN_T(i, t0)                                                                         \
    do {                                                                                     \
        if (threadIdx.x == 0) atomicAdd(&g_seed_stats[i], static_cast<unsigned long long>(clock64() - (t0))); \
        t0 = clock64();                                                                      \
    } while (0)
#define FIN_CNT() atomicAdd(&g_seed_stats[38], 1ull)
#else
#define FIN_T(i, t0) ((void)0)
#define FIN_CNT() ((void)0)
#endif
constexpr int kCons = 256;                // threads per CTA
constexpr int kConsWarps = kCons / 32;    // 8: warp w owns unit w of a tile
constexpr int kUnitRows = 1 << kUnitShift;  // 2048 rows per warp unit (hm_types.h)
constexpr int kFastTerms = 32;            // plan size served by this kernel
constexpr uint32_t kOffMask = (kUnitRows * 4 - 1) & ~3u;  // bk: impact (19 bits) | byte offset (13 bits)
constexpr int kImpShift = 2 + kUnitShift - (23 - kBakeMantBits);
constexpr float kFltMin = 1.17549435e-38f;
#ifndef HM_NE_ALPHA
#define HM_NE_ALPHA 0.3f
#endif
// essential-term variant of the sweep (search_fast.cu): the left-out terms'
// bound stays below kNeAlpha * the warp's admission threshold (0.3 measured
// best on C4 among 0.3-0.5); it serves plans of >= kNeMinTerms terms (C2's
// 3-6-term plans measured no faster there), every query with
// HM_FLAG_NE_ALL, none with HM_FLAG_NO_NESKIP
constexpr float kNeAlpha = HM_NE_ALPHA;
constexpr uint32_t kFlagNoNeSkip = 128u;
constexpr uint32_t kFlagNeAll = 256u;
static_assert(kConsWarps * kUnitRows == kTile, "one warp per 2048-row unit");
static_assert(2 + kUnitShift + 3 + kBakeMantBits == 32, "bk = 19-bit impact | 13-bit offset");

#ifndef HM_KC320
#define HM_KC320 2
#endif
#ifndef HM_ST320
#define HM_ST320 2
#endif
template <int CAPW>
struct FastCfg {
    static constexpr int kMaxKServed = CAPW == 192 ? 32 : 128;
    static constexpr int kC = CAPW == 192 ? 3 : HM_KC320;   // 16-byte chunks per lane per pipeline step
    static constexpr int kStages = CAPW == 192 ? 2 : HM_ST320;  // staged steps (1 applied + kStages - 1 in flight)
};

// Shared-memory layout.  ACC floats of accumulators (the tile sweep: kTile;
// the seeded pass only needs the epilogue's gather/survivor scratch) and,
// when STG, the sweep's cp.async staging.
template <int CAPW, int ACC, int STG>
struct __align__(16) SmemT {
    float acc[ACC];                        // first member: bk offsets are byte offsets into it
    float w32s[kShortCodes];               // impacts of the short-term codes
    uint32_t cl_row[kConsWarps][CAPW];     // per-warp candidate lists
    float cl_val[kConsWarps][CAPW];
    uint64_t t_start[kFastTerms], t_wlo[kFastTerms], t_end[kFastTerms];
    double t_idf[kFastTerms];
    uint32_t t_mult[kFastTerms];
    float t_c32[kFastTerms];
    int32_t t_slot[kFastTerms];
    uint32_t t_trow[kFastTerms];           // short terms: row of the index's tile table (kNoTabRow: none)
    uint4 stg[kConsWarps][STG ? FastCfg<CAPW>::kStages : 1][STG ? FastCfg<CAPW>::kC * 32 : 1];  // per-warp cp.async staging of baked postings
    uint64_t t_bkb[kFastTerms];            // long terms: start of the term's baked ranges in bk
    uint4 rdesc[kConsWarps][kFastTerms];  // per warp: the unit's nonempty long-term ranges in this tile
                                          // {bk address lo, hi, chunks, c bits}, df descending
    uint16_t order_list[kFastTerms];       // long terms (df descending), then short terms
    uint32_t pref[kFastTerms + 1];         // short-window prefix sums / gather offsets
    uint32_t hist[256];
    uint32_t sel[2];
    uint32_t n_w[kConsWarps];
    uint64_t post;
    uint32_t q, n_long, n_short, bad, n_surv, flood, Lg, total;
    // seeded MaxScore kernel (search_seed.cu) only
    float t_cu[kFastTerms];                // mult * idf * 2^-61 (selection-score domain)
    float t_ms[kFastTerms];                // t_cu * max impact of the term (rounded up)
    int32_t t_dense[kFastTerms];           // dense probe array of the term, -1 if none
    uint8_t msorder[kFastTerms];           // plan indices by t_ms ascending
    uint8_t t_spos[kFastTerms];            // short terms: index among the short terms (stab row)
    float ubne_q;                          // sum of the non-essential terms' bounds
    float rem_ub[kFastTerms + 1];          // seeds: bound of the ascending-bound prefix without t*;
                                           // sweep: bound of the first p terms of msorder (long terms)
    uint16_t p_lvl[kConsWarps][kFastTerms + 1];  // sweep, per warp: first tile (- j0) whose left-out
                                                 // prefix is >= l terms (0xFFFF: none yet)
    uint32_t n_ne, hbase;                  // sweep: long terms in msorder / histogram base bits
};

template <int CAPW>
using FastSmem = SmemT<CAPW, kTile, 1>;
// the seeded pass: epilogue scratch only (gather lists 8 B x 8 warps x CAPW >= survivors)
// seeded pass's essential-score hash table (search_seed.cu), in the
// accumulator area before the epilogue uses it: kHashSlots keys + values
#ifndef HM_HASH_BITS
#define HM_HASH_BITS 12
#endif
constexpr int kHashBits = HM_HASH_BITS;
constexpr uint32_t kHashSlots = 1u << kHashBits;
constexpr uint32_t kHashEmpty = 0xFFFFFFFFu;
// + the per-chunk segment table (kMaxSeg x (u64 start, u32 prefix, u32 meta) + 1)
#ifndef HM_MAX_SEG
#define HM_MAX_SEG 512
#endif
constexpr uint32_t kMaxSeg = HM_MAX_SEG;
constexpr uint32_t kSeedSmemMax = kHashSlots;  // seeds kept in the same area (scores, rows)
constexpr int kSeedAcc = 2 * static_cast<int>(kHashSlots) + 4 * static_cast<int>(kMaxSeg) + 4;
template <int CAPW>
using SeedSmem = SmemT<CAPW, (16 * CAPW > kSeedAcc ? 16 * CAPW : kSeedAcc), 0>;

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

// ---------------------------------------------------------------- short-term tile tables
// Row tab[jj] of short term s (list[s], its window [t_wlo, t_end) with prefix
// pref[s] in the concatenation of the scanned short terms' windows -- length 0
// for a term with an index tile table, filled from it): the offset (from
// t_start) of its first posting in tile j0 + jj, tab[nt] the window's end.
// Every posting f fills the entries of the tiles from its predecessor's tile
// (exclusive) to its own; HM_SHORT_U postings per thread are loaded before any
// entry is written (their loads in flight together).  Empty windows are filled
// by the second loop.  Ends with the CTA barrier.
#ifndef HM_SHORT_U
#define HM_SHORT_U 4
#endif
template <class Sm>
__device__ __forceinline__ void short_tables(const DevIndex& ix, Sm& S, const uint16_t* list, uint32_t n_short,
                                             uint32_t* stab, uint32_t stride, uint32_t j0, uint32_t nt,
                                             uint32_t cb) {
    constexpr int U = HM_SHORT_U;
    constexpr int NT = kCons;
    const uint32_t total = S.pref[n_short];
    for (uint32_t f0 = threadIdx.x; f0 < total; f0 += U * NT) {
        uint64_t g[U], w0[U];
        uint32_t sl[U], pc[U], pv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t f = f0 + u * NT;
            uint32_t lo = 0, hi = n_short;  // s: pref[s] <= f < pref[s+1]
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) >> 1;
                if (S.pref[mid] <= f) lo = mid;
                else hi = mid;
            }
            sl[u] = lo;
            w0[u] = S.t_wlo[list[lo]];
            g[u] = w0[u] + (f - S.pref[lo]);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool ok = f0 + u * NT < total;
            pc[u] = ok ? __ldg(ix.post + g[u]) : 0u;
            pv[u] = ok && g[u] != w0[u] ? __ldg(ix.post + g[u] - 1) : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (f0 + u * NT >= total) break;
            const uint32_t i = list[sl[u]];
            const uint64_t w1 = S.t_end[i], s0 = S.t_start[i];
            const int jt = static_cast<int>((pc[u] >> cb) >> kTileShift) - static_cast<int>(j0);
            const int jp = g[u] == w0[u] ? -1 : static_cast<int>((pv[u] >> cb) >> kTileShift) - static_cast<int>(j0);
            uint32_t* tab = stab + static_cast<uint64_t>(sl[u]) * stride;
            for (int jj = jp + 1; jj <= jt; ++jj) tab[jj] = static_cast<uint32_t>(g[u] - s0);
            if (g[u] + 1 == w1)
                for (int jj = jt + 1; jj <= static_cast<int>(nt); ++jj) tab[jj] = static_cast<uint32_t>(w1 - s0);
        }
    }
    // empty windows, and the terms with an index tile table (their postings
    // were not scanned): the table clamped to the window
    for (uint32_t x = threadIdx.x; x < n_short * (nt + 1); x += NT) {
        const uint32_t s = x / (nt + 1), jj = x % (nt + 1), i = list[s];
        const uint32_t lo = static_cast<uint32_t>(S.t_wlo[i] - S.t_start[i]);
        const uint32_t hi = static_cast<uint32_t>(S.t_end[i] - S.t_start[i]);
        const uint32_t r = S.t_trow[i];
        if (r != kNoTabRow) {
            const uint32_t v = jj == nt ? hi : __ldg(ix.short_tab + static_cast<uint64_t>(r) * (ix.n_tiles + 1) + j0 + jj);
            stab[static_cast<uint64_t>(s) * stride + jj] = min(max(v, lo), hi);
        } else if (lo == hi) {
            stab[static_cast<uint64_t>(s) * stride + jj] = lo;
        }
    }
    __syncthreads();
}

// ---------------------------------------------------------------- per-warp list
// Raise the warp's k-th bound from its own list (exact k-th largest by a
// binary search over the float bit pattern, values are >= 0), keep the
// admissible entries (>= max(Lw, Lg) * slack, stable compaction), publish the
// bound to the CTA-wide Lg.  Warp-synchronous; returns the new list length.
template <int CAPW, int ACC, int STG>
__device__ uint32_t warp_prune(SmemT<CAPW, ACC, STG>& S, int w, uint32_t n, uint32_t k, float& Lw, float slack) {
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

// ---------------------------------------------------------------- long terms
// Baked postings (hm_types.h): impact in the top 19 bits, accumulator byte
// offset in the low 13.  float(p >> 6) is the impact times 2^-ks (the
// offset's top 7 bits land below the 16 kept mantissa bits: relative error
// < 2^-16, covered by delta); a NULL posting decodes to a denormal and the
// flush-to-zero multiply makes its contribution exactly 0.  acc is the first
// smem member and warp units are 8 KB-aligned: the address is one OR.  CLIP (a
// window cuts the unit): postings whose tile-local row is outside [u0, u1)
// are skipped.
struct Clip {
    uint32_t wr0, u0, u1;
};
__device__ __forceinline__ uint32_t bk_off(uint32_t wbase, uint32_t p) { return wbase | (p & kOffMask); }
__device__ __forceinline__ float bk_w(uint32_t p) { return __uint_as_float(p >> kImpShift); }
__device__ __forceinline__ bool bk_in(const Clip& k, uint32_t p) {
    return (k.wr0 + swz10((p & kOffMask) >> 2)) - k.u0 < k.u1 - k.u0;
}
__device__ __forceinline__ float max3f(float a, float b, float c) {  // FMNMX3 (sm_100)
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ float mul_ftz(float a, float b) {
    float d;
    asm("mul.rn.ftz.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}
__device__ __forceinline__ float fma_ftz(float a, float b, float c) {
    float d;
    asm("fma.rn.ftz.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// apply N baked postings (the rows are distinct: all loads, then all stores)
template <bool FIRST, bool CLIP, int N>
__device__ __forceinline__ void apply_n(float* __restrict__ acc, uint32_t wbase, const uint32_t* p, float c,
                                        const Clip& k) {
    char* base = reinterpret_cast<char*>(acc);
    float a[N];
    if (!FIRST) {
#pragma unroll
        for (int e = 0; e < N; ++e)
            if (!CLIP || bk_in(k, p[e])) a[e] = *reinterpret_cast<float*>(base + bk_off(wbase, p[e]));
    }
#pragma unroll
    for (int e = 0; e < N; ++e) {
        if (CLIP && !bk_in(k, p[e])) continue;
        float* dst = reinterpret_cast<float*>(base + bk_off(wbase, p[e]));
        if (FIRST) *dst = mul_ftz(c, bk_w(p[e]));
        else *dst = fma_ftz(c, bk_w(p[e]), a[e]);
    }
}

// One pipeline step of a long term's baked range in the warp's unit: up to
// 32*kC 16-byte chunks, staged in shared memory by per-lane cp.async (each
// lane copies and later reads only its own chunks: no warp sync needed).
struct Step {
    const uint4* base;    // the range's first chunk in bk
    uint32_t o, nch;      // chunk offset of this step, chunks in the range
    uint32_t j, x;        // tile, range (long-term slot in order_list); j > j1: none
    float c;              // mult * idf * 2^(ks - 61) of the term
    bool first;           // first range of the unit in this tile: store instead of read-modify-write
};

template <int KC>
__device__ __forceinline__ void step_issue(const Step& s, uint4* stg) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int u = 0; u < KC; ++u) {
        const uint32_t c = s.o + 32 * u + lane;
        if (c < s.nch)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(stg + 32 * u + lane)),
                         "l"(s.base + c)
                         : "memory");
    }
}

template <int KC, bool FIRST, bool CLIP>
__device__ __forceinline__ void step_apply(float* __restrict__ acc, uint32_t wbase, const Step& s,
                                           const uint4* stg, const Clip& k) {
    const uint32_t lane = threadIdx.x & 31;
#pragma unroll
    for (int u = 0; u < KC; u += 2) {
        if (s.o + 32 * u >= s.nch) break;  // warp-uniform
        const bool ok0 = s.o + 32 * u + lane < s.nch;
        const bool ok1 = u + 1 < KC && s.o + 32 * (u + 1) + lane < s.nch;
        if (ok1) {
            const uint4 v0 = stg[32 * u + lane], v1 = stg[32 * (u + 1) + lane];
            const uint32_t p[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
            apply_n<FIRST, CLIP, 8>(acc, wbase, p, s.c, k);
        } else if (ok0) {
            const uint4 v0 = stg[32 * u + lane];
            const uint32_t p[4] = {v0.x, v0.y, v0.z, v0.w};
            apply_n<FIRST, CLIP, 4>(acc, wbase, p, s.c, k);
        }
    }
}

// Epilogue of a query (both kernels): merge the warps' candidate lists, keep
// the survivors of the k-th fp32 value (slack f_slack), rescore them exactly
// in fp64 in plan order with the reference's operation order
// (src/csr_index.cpp:10-15, 87-101), rank by (score desc, DocId asc)
// (include/hybrid/types.hpp:21-25), write the top-k, postings_touched and the
// Margin confidence + skip (src/cascade.cpp:15-21, 79-84).  A near-tie flood
// (> kSurvCap survivors) hands the query to the exact kernel.  Leaves the
// accumulator area zero.
// (tf, doc length) of plan term i in a row of the query's window, for the
// exact rescoring: a dense term's per-row code (one load), a short term's
// tile segment (stab row t_spos[i]), else find_posting's sub-tile search.
template <class Sm>
__device__ __forceinline__ bool exact_lookup(const DevIndex& ix, const Sm& S, const uint32_t* stab, uint32_t stride,
                                             uint32_t j0, uint32_t cb, uint32_t i, uint32_t row, double* tf,
                                             double* dl) {
    const int32_t slot = S.t_slot[i];
    if (slot >= 0) {
        const int32_t d = S.t_dense[i];
        if (d >= 0) {
            const uint16_t code = __ldg(ix.dense + static_cast<uint64_t>(d) * ix.n_docs + row);
            if (code == kDenseAbsent) return false;
            if (code != kDenseEscape) {
                *tf = ix.code_tf[code];
                *dl = ix.code_len[code];
                return true;
            }
        }
        return find_posting(ix, slot, S.t_start[i], S.t_end[i], row, ix.code_tf, ix.code_len, tf, dl);
    }
    const uint32_t* tab = stab + static_cast<uint64_t>(S.t_spos[i]) * stride;
    const uint32_t jj = (row >> kTileShift) - j0;
    const uint64_t s0 = S.t_start[i];
    const uint64_t lo = s0 + tab[jj], hi = s0 + tab[jj + 1];
    const uint64_t pos = lower_bound_row(ix.post, lo, hi, row, cb);
    if (pos >= hi) return false;
    const uint32_t p = __ldg(ix.post + pos);
    if ((p >> cb) != row) return false;
    const uint32_t code = p & ix.esc_short;
    if (code < ix.n_codes_short) {
        *tf = ix.code_tf[code];
        *dl = ix.code_len[code];
    } else {
        *tf = __ldg(ix.tf + pos);
        *dl = __ldg(ix.doc_lens + row);
    }
    return true;
}

template <int CAPW, int ACC, int STG>
__device__ __forceinline__ void finish_query(const DevIndex& ix, const BatchArgs& a, SmemT<CAPW, ACC, STG>& S, uint32_t q,
                                             uint32_t m, uint32_t k, uint32_t nw, float f_slack, double k1,
                                             double bb, const uint32_t* stab, uint32_t stride, uint32_t j0,
                                             uint32_t cb) {
    constexpr int kGatherBytes = 8 * kConsWarps * CAPW;
    static_assert(kSurvBytes + 8 * kCons <= 4 * ACC, "survivors + the rescoring batch fit in the accumulator area");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef HM_SEED_STATS
    long long ft = clock64();
#endif
    auto csync = [] { __syncthreads(); };
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
    FIN_T(32, ft);
    if (nc >= k) theta = block_kth_largest<kCons>(gv, nc, k, S.hist, S.sel, csync) * f_slack;
    FIN_T(33, ft);
    if (warp == 0) {
        uint32_t w = 0;
        for (uint32_t b0 = 0; b0 < nc; b0 += 32) {
            const uint32_t i = b0 + lane;
            const bool keep = i < nc && gv[i] >= theta;
            const uint32_t bal = __ballot_sync(0xffffffffu, keep);
            const uint32_t pos = w + __popc(bal & ((1u << lane) - 1));
            if (keep && pos < kSurvCap) (&S.cl_row[0][0])[pos] = gr[i];  // list area is free now
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
        return;
    }
    FIN_T(34, ft);
    SurvView sv{reinterpret_cast<double*>(sp), reinterpret_cast<uint64_t*>(sp + 8 * kSurvCap),
                reinterpret_cast<uint32_t*>(sp + 16 * kSurvCap)};
    for (uint32_t i = tid; i < ns; i += kCons) sv.row[i] = (&S.cl_row[0][0])[i];
    csync();
    // (survivor, term) pairs over all threads, a batch of kCons lookups in flight
    // together; then every survivor adds its terms' exact scores in plan order
    // (fp64, mult repeats, the reference's accumulation :87-101) -- a term
    // absent from the row (-1) adds nothing
    double* const pv = reinterpret_cast<double*>(sp + kSurvBytes);
    for (uint32_t i = tid; i < ns; i += kCons) {
        sv.E[i] = 0.0;
        sv.id[i] = __ldg(ix.doc_ids + sv.row[i]);  // (in flight with the first batch of lookups)
    }
    const uint32_t npair = ns * m;
    for (uint32_t p0 = 0; p0 < npair; p0 += kCons) {
        const uint32_t p = p0 + tid;
        double val = -1.0;
        if (p < npair) {
            const uint32_t s = p / m, t = p - s * m;
            double tf, dl;
            if (exact_lookup(ix, S, stab, stride, j0, cb, t, sv.row[s], &tf, &dl))
                val = bm25_exact(tf, S.t_idf[t], dl, ix.avgdl, k1, bb);
        }
        pv[tid] = val;
        csync();
        const uint32_t s = p0 / m + tid;
        if (s < ns && s * m < p0 + kCons) {
            const uint32_t x0 = max(s * m, p0), x1 = min(min(s * m + m, p0 + kCons), npair);
            double E = sv.E[s];
            for (uint32_t x = x0; x < x1; ++x) {
                const double v = pv[x - p0];
                if (v >= 0.0) {
                    const uint32_t mu = S.t_mult[x - s * m];
                    for (uint32_t r = 0; r < mu; ++r) E = __dadd_rn(E, v);  // :94
                }
            }
            sv.E[s] = E;
        }
        csync();
    }
    FIN_T(35, ft);
    // rank of every survivor in (score desc, DocId asc) order -- the pairs are
    // distinct (DocIds are) -- by counting the survivors ranked before it; the
    // top k land in rank order in the rescoring batch's area (k <= 128)
    double* const tE = reinterpret_cast<double*>(sp + kSurvBytes);
    uint64_t* const tI = reinterpret_cast<uint64_t*>(sp + kSurvBytes + 8 * 128);
    static_assert(16 * 128 <= 8 * kCons, "the top-k fits in the rescoring batch's area");
    // (an index may repeat a DocId: equal pairs are then ordered by row, so the
    // ranks stay distinct -- any order of equal pairs is the same output)
    for (uint32_t i = tid; i < ns; i += kCons) {
        const double e = sv.E[i];
        const uint64_t id = sv.id[i];
        uint32_t r = 0;
        for (uint32_t j = 0; j < ns; ++j)
            r += better(sv.E[j], sv.id[j], e, id) || (sv.E[j] == e && sv.id[j] == id && j < i) ? 1u : 0u;
        if (r < k) {
            tE[r] = e;
            tI[r] = id;
        }
    }
    csync();
    FIN_T(36, ft);
    if (tid == 0) {
        uint32_t nout = 0;
        for (uint32_t i = 0; i < ns && nout < k; ++i) {
            if (!(tE[i] > 0.0)) break;  // zero scores never emitted (:56)
            a.out_ids[static_cast<uint64_t>(q) * k + nout] = tI[i];
            a.out_scores[static_cast<uint64_t>(q) * k + nout] = tE[i];
            ++nout;
        }
        a.out_n[q] = nout;
        if (a.out_post) a.out_post[q] = S.post;
        write_decision(a, q, tE, nout);
    }
    csync();
    for (int i = tid; i < (kSurvBytes + 8 * kCons) / 4; i += kCons) S.acc[i] = 0.f;  // survivors + rescoring batch
    FIN_T(37, ft);
    if (threadIdx.x == 0) FIN_CNT();
}

}  // namespace hm
