// search_pipe_kernel: the fused BM25 hot path on sm_100a (one CTA per SM).
//
// Warp-specialised: 16 consumer warps + 1 producer warp.  The producer walks
// the current query's row window tile by tile (kTile = 16384 rows) and, for
// every plan term, streams that term's posting segment of the tile from HBM
// into a 6-slot x 16 KB shared-memory ring with 1-D TMA bulk copies
// (cp.async.bulk ... mbarrier::complete_tx), several tiles ahead of the
// consumers.  Consumers wait on the slot's transaction barrier, accumulate
// fp32 scores into a per-tile shared accumulator (long terms: plain
// read-modify-write, one term at a time; short terms: shared atomics), then
// scan the tile once: docs that can still reach the top-k join a candidate
// list and the accumulators are zeroed (pitfall-3 sentinel reset).  When the
// query's window is exhausted the survivors are rescored exactly in fp64 in
// the reference's operation/accumulation order (src/csr_index.cpp:10-15, 87-101),
// ranked by (score desc, DocId asc) (include/hybrid/types.hpp:21-25), and the
// Margin confidence + skip decision are written (src/cascade.cpp:15-21, 79-84).
// See bm25_search.cu for the exactness argument of the fp32 selection.
#include "hm_device.cuh"
#include "hm_launch.h"
#include "hm_ptx.cuh"

namespace hm {

constexpr int kCons = kThreads;           // 512 consumer threads
constexpr int kPipeThreads = kCons + 32;  // + 1 producer warp
constexpr int kSlots = 6;
constexpr int kSlotElems = 4096;          // 16 KB per slot
constexpr int kSegs = 32;                 // segments per slot
constexpr int kUnroll = 8;                // postings per consumer thread per step
constexpr int kEscCap = 512;              // deferred escaped postings per tile

struct SlotMeta {
    uint32_t n_seg, last;
    uint16_t term[kSegs], lo[kSegs], hi[kSegs];
    uint64_t goff[kSegs];  // global posting index of slot element 0 for this segment
};

struct __align__(128) PipeSmem {
    uint32_t ring[kSlots][kSlotElems];
    float acc[kTile];
    float w32[kMaxCodes + 4];  // [kMaxCodes] = 0: impact of escaped / padded postings
    uint32_t cand_row[kCap];
    float cand_a[kCap];
    SlotMeta meta[kSlots];
    uint64_t full[kSlots], empty[kSlots];
    uint64_t t_start[kMaxTerms], t_wlo[kMaxTerms], t_end[kMaxTerms];
    double t_idf[kMaxTerms];
    uint32_t t_mult[kMaxTerms];
    float t_c32[kMaxTerms];
    int32_t t_slot[kMaxTerms];
    uint16_t order_list[kMaxTerms];  // long terms, then short terms
    uint32_t pref[kMaxTerms + 1];    // prefix sums of short windows
    uint32_t pb[2][kMaxTerms], pe[2][kMaxTerms];
    uint32_t hist[256];
    uint32_t sel[2];
    uint64_t esc_gidx[kEscCap];
    uint32_t esc_row[kEscCap];
    uint16_t esc_term[kEscCap];
    uint64_t post;
    uint32_t q, n_long, n_short, n_c, ovf, bad, n_surv, n_esc;
    float L;
};

static_assert(sizeof(PipeSmem) <= 227 * 1024, "PipeSmem exceeds the 227 KB per-CTA shared memory");

struct SurvView {
    double* E;
    uint64_t* id;
    uint32_t* row;
};
constexpr int kSurvBytes = 20 * kSurvCap;
static_assert(kSurvBytes <= static_cast<int>(sizeof(float)) * kTile, "survivors fit in acc");

__device__ __forceinline__ float esc_w(const DevIndex& ix, uint64_t gidx, uint32_t row, double k1,
                                       double b) {
    return impact32(static_cast<double>(__ldg(ix.tf + gidx)),
                    static_cast<double>(__ldg(ix.doc_lens + row)), ix.avgdl, k1, b);
}

// Escaped posting (its (tf, len) pair has no code): queue it for a batched
// exact lookup after the tile's segments; when the queue is full, apply now.
__device__ __forceinline__ void defer_escape(PipeSmem& S, const DevIndex& ix, uint32_t row,
                                             uint64_t gidx, uint32_t term, float c, uint32_t base,
                                             double k1, double b) {
    const uint32_t x = atomicAdd(&S.n_esc, 1u);
    if (x < kEscCap) {
        S.esc_row[x] = row;
        S.esc_gidx[x] = gidx;
        S.esc_term[x] = static_cast<uint16_t>(term);
    } else {
        atomicAdd(&S.acc[row - base], c * esc_w(ix, gidx, row, k1, b));
    }
}

// One long-term segment [lo, hi) of a ring slot.  Warp w takes 256
// consecutive postings (8 per lane, lane-interleaved so consecutive lanes hit
// nearly consecutive rows: conflict-free accumulator banks); warps past the
// segment end skip.  Rows of one term are distinct, so plain RMW is race-free
// (terms are separated by a named barrier).  Escaped codes (and the padding
// entry kMaxCodes) read a zero impact; escapes are then queued.
template <bool CLIP>
__device__ __forceinline__ void accum_long(PipeSmem& S, const DevIndex& ix, const uint32_t* src,
                                           uint32_t lo, uint32_t hi, uint64_t goff, float c,
                                           uint32_t term, uint32_t base, uint32_t rlo, uint32_t rn,
                                           double k1, double b) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t n_codes = ix.n_codes;
    for (uint32_t wb = lo + warp * (kUnroll * 32); wb < hi; wb += kUnroll * kCons) {
        uint32_t p[kUnroll], loc[kUnroll];
        float w[kUnroll], av[kUnroll];
        uint32_t cmax = 0;
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint32_t e = wb + u * 32 + lane;
            p[u] = e < hi ? src[e] : 0u;
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            loc[u] = p[u] >> kCodeBitsLong;
            const uint32_t code = p[u] & kEscLong;
            cmax = max(cmax, code);
            w[u] = S.w32[min(code, static_cast<uint32_t>(kMaxCodes))];
            if (CLIP && loc[u] - rlo >= rn) w[u] = 0.f;
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) av[u] = S.acc[loc[u]];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
            if (wb + u * 32 + lane < hi) S.acc[loc[u]] = __fmaf_rn(c, w[u], av[u]);
        if (__any_sync(0xffffffffu, cmax >= n_codes)) {
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const uint32_t e = wb + u * 32 + lane;
                if (e < hi && (p[u] & kEscLong) >= n_codes && (!CLIP || loc[u] - rlo < rn))
                    defer_escape(S, ix, base + loc[u], goff + e, term, c, base, k1, b);
            }
        }
    }
}

// Short-term segments: same warp mapping, shared-memory atomics (several
// short terms may share a slot and need no barrier between them).
__device__ __forceinline__ void accum_short(PipeSmem& S, const DevIndex& ix, const uint32_t* src,
                                            uint32_t lo, uint32_t hi, uint64_t goff, float c,
                                            uint32_t term, uint32_t base, double k1, double b) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t cb = ix.code_bits, ncs = ix.n_codes_short, escs = ix.esc_short;
    for (uint32_t wb = lo + warp * (kUnroll * 32); wb < hi; wb += kUnroll * kCons) {
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            const uint32_t e = wb + u * 32 + lane;
            if (e < hi) {
                const uint32_t p = src[e];
                const uint32_t row = p >> cb;
                const uint32_t code = p & escs;
                if (code < ncs) atomicAdd(&S.acc[row - base], c * S.w32[code]);
                else defer_escape(S, ix, row, goff + e, term, c, base, k1, b);
            }
        }
    }
}

__global__ void __launch_bounds__(kPipeThreads, 1) search_pipe_kernel(DevIndex ix, BatchArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    PipeSmem& S = *reinterpret_cast<PipeSmem*>(smem_raw);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool producer = warp == kCons / 32;
    auto csync = [] { named_sync<kCons>(); };
    const uint32_t cb = ix.code_bits;
    const uint32_t row_lo = a.row_lo, row_hi = a.row_hi;
    const double k1 = a.k1, bb = a.b;
    const uint32_t stride = a.stab_stride;
    uint32_t* stab = a.stab + static_cast<uint64_t>(blockIdx.x) * kMaxTerms * stride;

    for (int i = tid; i < kTile; i += kPipeThreads) S.acc[i] = 0.f;
    for (int i = tid; i < kMaxCodes + 4; i += kPipeThreads) S.w32[i] = i < kMaxCodes ? a.w32[i] : 0.f;
    if (tid == 0) {
        for (int s = 0; s < kSlots; ++s) {
            mbar_init(&S.full[s], 1);
            mbar_init(&S.empty[s], kCons / 32);
        }
        mbar_init_fence();
        S.n_c = 0;
        S.L = 0.f;
        S.n_esc = 0;
    }
    uint32_t ring_use = 0;  // slot uses so far (identical sequence in both roles)

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
        if (m > kMaxTerms) {
            if (tid == 0) {
                atomicOr(&a.counters[3], kErrTooManyTerms);
                a.out_n[q] = 0;
                if (a.out_post) a.out_post[q] = 0;
                write_decision(a, q, nullptr, 0);
            }
            continue;
        }
        // ---------------- prologue: plan, window bounds
        if (tid < static_cast<int>(m)) {
            uint32_t t = a.plan_tid[poff + tid];
            uint32_t mult = a.plan_mult[poff + tid];
            double idf = ix.idf[t];
            int32_t slot = ix.long_slot[t];
            uint64_t s0 = ix.term_off[t], s1 = ix.term_off[t + 1];
            uint64_t w0 = row_lo > 0 ? first_at_or_after(ix, slot, s0, s1, row_lo) : s0;
            uint64_t w1 = row_hi < ix.n_docs ? first_at_or_after(ix, slot, s0, s1, row_hi) : s1;
            S.t_start[tid] = s0;
            S.t_wlo[tid] = w0;
            S.t_end[tid] = w1;
            S.t_idf[tid] = idf;
            S.t_mult[tid] = mult;
            S.t_c32[tid] = static_cast<float>(static_cast<double>(mult) * idf);
            S.t_slot[tid] = slot;
        }
        __syncthreads();
        if (tid == 0) {
            uint64_t post = 0;
            uint32_t nl = 0, ns = 0, bad = 0;
            for (uint32_t i = 0; i < m; ++i) {
                post += S.t_end[i] - S.t_wlo[i];
                double idf = S.t_idf[i];
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
            S.ovf = 0;
            if (!(a.flags & 2u)) {  // HM_FLAG_DEBUG_NO_RESET skips the sentinel reset
                S.n_c = 0;
                S.L = 0.f;
            }
        }
        __syncthreads();
        if (S.bad || (a.flags & 1u)) {
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
        const uint32_t j0 = row_lo >> kTileShift, j1 = (row_hi - 1) >> kTileShift;
        const uint32_t nt = j1 - j0 + 1;
        // ---------------- short-term tile tables (per CTA scratch)
        if (!producer && n_short) {
            const uint32_t total = S.pref[n_short];
            for (uint32_t f = tid; f < total; f += kCons) {
                uint32_t lo = 0, hi = n_short;  // s: pref[s] <= f < pref[s+1]
                while (hi - lo > 1) {
                    uint32_t mid = (lo + hi) >> 1;
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

        if (producer) {
            // =========================================== producer warp
            uint32_t nb[kMaxTerms / 32], ne[kMaxTerms / 32];
            auto load_bounds = [&](uint32_t j) {
#pragma unroll
                for (int r = 0; r < kMaxTerms / 32; ++r) {
                    const uint32_t x = lane + 32 * r;
                    if (x < m) {
                        if (x < n_long) {
                            const uint32_t* tb = tile_row(ix, S.t_slot[S.order_list[x]]);
                            nb[r] = __ldg(tb + j);
                            ne[r] = __ldg(tb + j + 1);
                        } else {
                            const uint32_t* tab = stab + static_cast<uint64_t>(x - n_long) * stride;
                            nb[r] = tab[j - j0];
                            ne[r] = tab[j - j0 + 1];
                        }
                    }
                }
            };
            auto store_bounds = [&](int buf) {
#pragma unroll
                for (int r = 0; r < kMaxTerms / 32; ++r) {
                    const uint32_t x = lane + 32 * r;
                    if (x < m) {
                        S.pb[buf][x] = nb[r];
                        S.pe[buf][x] = ne[r];
                    }
                }
            };
            load_bounds(j0);
            store_bounds(0);
            __syncwarp();
            bool open = false;
            uint32_t s = 0, fill = 0, nseg = 0;
            auto open_slot = [&] {
                s = ring_use % kSlots;
                mbar_wait(&S.empty[s], ((ring_use / kSlots) & 1u) ^ 1u);
                fill = 0;
                nseg = 0;
                open = true;
            };
            auto close_slot = [&](bool last) {
                S.meta[s].n_seg = nseg;
                S.meta[s].last = last ? 1u : 0u;
                mbar_arrive(&S.full[s]);
                ++ring_use;
                open = false;
            };
            for (uint32_t j = j0; j <= j1; ++j) {
                const int buf = (j - j0) & 1;
                if (j < j1) load_bounds(j + 1);
                if (lane == 0) {
                    for (uint32_t x = 0; x < m; ++x) {
                        const uint32_t i = S.order_list[x];
                        const uint64_t s0 = S.t_start[i];
                        uint64_t b = s0 + S.pb[buf][x];
                        const uint64_t e = s0 + S.pe[buf][x];
                        while (b < e) {
                            if (!open) open_slot();
                            const uint64_t a16 = b & ~3ull;
                            const uint64_t e4 = (e + 3) & ~3ull;
                            const uint64_t cend = min(e4, a16 + (kSlotElems - fill));
                            if (cend <= b) {
                                close_slot(false);
                                continue;
                            }
                            const uint64_t send = min(e, cend);
                            SlotMeta& M = S.meta[s];
                            M.term[nseg] = static_cast<uint16_t>(i);
                            M.lo[nseg] = static_cast<uint16_t>(fill + (b - a16));
                            M.hi[nseg] = static_cast<uint16_t>(fill + (send - a16));
                            M.goff[nseg] = a16 - fill;
                            const uint32_t bytes = static_cast<uint32_t>(cend - a16) * 4u;
                            mbar_expect_tx(&S.full[s], bytes);
                            bulk_g2s(&S.ring[s][fill], ix.post + a16, bytes, &S.full[s]);
                            fill += static_cast<uint32_t>(cend - a16);
                            ++nseg;
                            b = send;
                            if (fill == kSlotElems || nseg == kSegs) close_slot(false);
                        }
                    }
                    if (!open) open_slot();
                    close_slot(true);
                }
                __syncwarp();
                ring_use = __shfl_sync(0xffffffffu, ring_use, 0);
                if (j < j1) store_bounds(buf ^ 1);
                __syncwarp();
            }
            continue;  // wait for the consumers at the top of the loop
        }

        // =============================================== consumer warps
        const float delta = static_cast<float>(m + 10) * 5.9604645e-08f;  // (m+10) * 2^-24
        const float f_slack = 1.0f - 2.5f * delta;
        bool to_exact = false;
        for (uint32_t j = j0; j <= j1; ++j) {
            const uint32_t base = j << kTileShift;
            const uint32_t R0 = max(base, row_lo);
            const uint32_t R1 = min(base + kTile, row_hi);
            const uint32_t rlo = R0 - base, rn = R1 - R0;
            const bool clip = rn != kTile;
            // ---- drain this tile's ring slots
            int cur = -1;
            bool in_short = false;
            for (;;) {
                const uint32_t s = ring_use % kSlots;
                mbar_wait(&S.full[s], (ring_use / kSlots) & 1u);
                const uint32_t nseg = S.meta[s].n_seg;
                const bool last = S.meta[s].last != 0;
                const uint32_t* src = S.ring[s];
                for (uint32_t g = 0; g < nseg && !to_exact; ++g) {
                    const uint32_t i = S.meta[s].term[g];
                    const uint32_t lo = S.meta[s].lo[g], hi = S.meta[s].hi[g];
                    const uint64_t goff = S.meta[s].goff[g];
                    const float c = S.t_c32[i];
                    if (S.t_slot[i] >= 0) {
                        if (cur != static_cast<int>(i)) {
                            if (cur != -1) csync();
                            cur = static_cast<int>(i);
                        }
                        if (clip) accum_long<true>(S, ix, src, lo, hi, goff, c, i, base, rlo, rn, k1, bb);
                        else accum_long<false>(S, ix, src, lo, hi, goff, c, i, base, rlo, rn, k1, bb);
                    } else {
                        if (!in_short) {
                            csync();
                            in_short = true;
                        }
                        accum_short(S, ix, src, lo, hi, goff, c, i, base, k1, bb);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&S.empty[s]);
                ++ring_use;
                if (last) break;
            }
            if (to_exact) continue;  // drain the remaining tiles' slots only
            csync();
            if (S.n_esc) {  // deferred escaped postings: exact (tf, len) lookups, batched
                const uint32_t ne = min(S.n_esc, static_cast<uint32_t>(kEscCap));
                for (uint32_t x = tid; x < ne; x += kCons) {
                    const uint32_t row = S.esc_row[x];
                    const float w = esc_w(ix, S.esc_gidx[x], row, k1, bb);
                    atomicAdd(&S.acc[row - base], S.t_c32[S.esc_term[x]] * w);
                }
                csync();
                if (tid == 0) S.n_esc = 0;
            }
            // ---- scan, with overflow recovery by re-accumulating from HBM/L2
            for (int attempt = 0;; ++attempt) {
                {
                    const float t_emit = S.L * f_slack;
                    const uint32_t v0 = rlo >> 2, v1 = (rlo + rn + 3) >> 2;
                    float4* acc4 = reinterpret_cast<float4*>(S.acc);
                    for (uint32_t vb = v0; vb < v1; vb += kCons) {
                        const uint32_t v = vb + tid;
                        float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
                        if (v < v1) {
                            x = acc4[v];
                            acc4[v] = make_float4(0.f, 0.f, 0.f, 0.f);
                        }
                        const float mx = fmaxf(fmaxf(x.x, x.y), fmaxf(x.z, x.w));
                        if (__ballot_sync(0xffffffffu, mx > 0.f && mx >= t_emit)) {
                            const bool q0 = x.x > 0.f && x.x >= t_emit, q1 = x.y > 0.f && x.y >= t_emit;
                            const bool q2 = x.z > 0.f && x.z >= t_emit, q3 = x.w > 0.f && x.w >= t_emit;
                            const uint32_t cnt = q0 + q1 + q2 + q3;
                            const uint32_t incl = warp_incl_scan(cnt);
                            const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
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
                csync();
                if (!S.ovf) break;
                const uint32_t nc = min(S.n_c, static_cast<uint32_t>(kCap));
                const float nl = block_kth_largest<kCons>(S.cand_a, nc, k, S.hist, S.sel, csync);
                if (attempt >= 3 || !(nl > S.L)) {
                    to_exact = true;
                    break;
                }
                if (warp == 0) {
                    const float thr = nl * f_slack;
                    const uint32_t w = warp_compact(S.cand_row, S.cand_a, nc, [&](uint32_t row, float v) {
                        return (row < R0 || row >= R1) && v >= thr;
                    });
                    if (lane == 0) {
                        S.n_c = w;
                        S.L = nl;
                        S.ovf = 0;
                    }
                }
                // re-accumulate the tile straight from global memory (rare path)
                for (uint32_t x = 0; x < m; ++x) {
                    const uint32_t i = S.order_list[x];
                    const float c = S.t_c32[i];
                    const uint64_t s0 = S.t_start[i];
                    uint64_t b, e;
                    if (x < n_long) {
                        const uint32_t* tb = tile_row(ix, S.t_slot[i]);
                        b = s0 + __ldg(tb + j);
                        e = s0 + __ldg(tb + j + 1);
                    } else {
                        const uint32_t* tab = stab + static_cast<uint64_t>(x - n_long) * stride;
                        b = s0 + tab[j - j0];
                        e = s0 + tab[j - j0 + 1];
                    }
                    csync();
                    for (uint64_t g = b + tid; g < e; g += kCons) {
                        const uint32_t p = __ldg(ix.post + g);
                        if (x < n_long) {
                            const uint32_t local = p >> kCodeBitsLong;
                            if (local - rlo < rn) {
                                const uint32_t code = p & kEscLong;
                                const float w = code < ix.n_codes ? S.w32[code] : esc_w(ix, g, base + local, k1, bb);
                                S.acc[local] = __fmaf_rn(c, w, S.acc[local]);
                            }
                        } else {
                            const uint32_t row = p >> cb;
                            const uint32_t code = p & ix.esc_short;
                            const float w = code < ix.n_codes_short ? S.w32[code] : esc_w(ix, g, row, k1, bb);
                            S.acc[row - base] = __fmaf_rn(c, w, S.acc[row - base]);
                        }
                    }
                }
                csync();
            }
            if (to_exact) continue;
            // ---- keep the list short: raise L and prune
            if (S.n_c > kPruneAt) {
                const uint32_t nc = S.n_c;
                const float nl = block_kth_largest<kCons>(S.cand_a, nc, k, S.hist, S.sel, csync);
                if (warp == 0) {
                    const float L = fmaxf(S.L, nl);
                    const float thr = L * f_slack;
                    const uint32_t w = warp_compact(S.cand_row, S.cand_a, nc,
                                                    [&](uint32_t, float v) { return v >= thr; });
                    if (lane == 0) {
                        S.n_c = w;
                        S.L = L;
                    }
                }
                csync();
            }
        }
        csync();
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
        if (nc >= k) theta = block_kth_largest<kCons>(S.cand_a, nc, k, S.hist, S.sel, csync) * f_slack;
        char* sp = reinterpret_cast<char*>(S.acc);
        SurvView sv{reinterpret_cast<double*>(sp), reinterpret_cast<uint64_t*>(sp + 8 * kSurvCap),
                    reinterpret_cast<uint32_t*>(sp + 16 * kSurvCap)};
        if (warp == 0) {
            uint32_t w = 0;
            for (uint32_t b0 = 0; b0 < nc; b0 += 32) {
                const uint32_t i = b0 + lane;
                const bool keep = i < nc && S.cand_a[i] >= theta;
                const uint32_t bal = __ballot_sync(0xffffffffu, keep);
                const uint32_t pos = w + __popc(bal & ((1u << lane) - 1));
                if (keep && pos < kSurvCap) sv.row[pos] = S.cand_row[i];
                w += __popc(bal);
            }
            if (lane == 0) S.n_surv = w;
        }
        csync();
        const uint32_t ns = S.n_surv;
        if (ns > kSurvCap) {  // near-tie flood: exact kernel takes the query
            for (int i = tid; i < kSurvBytes / 4; i += kCons) S.acc[i] = 0.f;
            if (tid == 0) {
                a.exact_list[atomicAdd(&a.counters[1], 1u)] = q;
                if (a.out_post) a.out_post[q] = S.post;
            }
            continue;
        }
        // warp per survivor, lanes over plan terms; fp64 sum in plan order
        for (uint32_t s = warp; s < ns; s += kCons / 32) {
            const uint32_t row = sv.row[s];
            double E = 0.0;
            for (uint32_t t0 = 0; t0 < m; t0 += 32) {
                const uint32_t t = t0 + lane;
                double val = 0.0;
                bool present = false;
                if (t < m) {
                    double tf, dl;
                    if (find_posting(ix, S.t_slot[t], S.t_wlo[t], S.t_end[t], row, ix.code_tf,
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

static bool g_pipe_attr = false;

cudaError_t launch_search(const DevIndex& ix, const BatchArgs& a, int grid, cudaStream_t st) {
    if (!g_pipe_attr) {
        cudaError_t e = cudaFuncSetAttribute(search_pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(sizeof(PipeSmem)));
        if (e != cudaSuccess) return e;
        g_pipe_attr = true;
    }
    search_pipe_kernel<<<grid, kPipeThreads, sizeof(PipeSmem), st>>>(ix, a);
    return cudaGetLastError();
}

cudaError_t search_occupancy_fast(int* blocks) {
    if (!g_pipe_attr) {
        cudaError_t e = cudaFuncSetAttribute(search_pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(sizeof(PipeSmem)));
        if (e != cudaSuccess) return e;
        g_pipe_attr = true;
    }
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, search_pipe_kernel, kPipeThreads,
                                                         sizeof(PipeSmem));
}

size_t search_smem_bytes() { return sizeof(PipeSmem); }

}  // namespace hm
