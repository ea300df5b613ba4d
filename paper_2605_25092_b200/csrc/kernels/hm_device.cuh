// Device helpers shared by the BM25 search kernels (layout: hm_types.h).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "hm_types.h"

namespace hm {

// exact BM25 in the reference's operation order (src/csr_index.cpp:10-15):
//   norm = avgdl > 0 ? len / avgdl : 1;  denom = tf + k1 * ((1 - b) + b * norm)
//   s = ((idf * tf) * (k1 + 1)) / denom
// Explicit round-to-nearest intrinsics: never contracted into FMAs.
__device__ __forceinline__ double bm25_exact(double tf, double idf, double dl,
                                             double avgdl, double k1, double b) {
    double norm = avgdl > 0.0 ? __ddiv_rn(dl, avgdl) : 1.0;
    double denom = __dadd_rn(tf, __dmul_rn(k1, __dadd_rn(__dsub_rn(1.0, b), __dmul_rn(b, norm))));
    return __ddiv_rn(__dmul_rn(__dmul_rn(idf, tf), __dadd_rn(k1, 1.0)), denom);
}

// idf-free impact tf*(k1+1)/(tf + K_len) evaluated in fp64, rounded once.
__device__ __forceinline__ float impact32(double tf, double dl, double avgdl,
                                          double k1, double b) {
    double norm = avgdl > 0.0 ? dl / avgdl : 1.0;
    double denom = tf + k1 * (1.0 - b + b * norm);
    return static_cast<float>(tf * (k1 + 1.0) / denom);
}

__device__ __forceinline__ uint4 ldg_stream(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t ldg_stream(const uint32_t* p) {
    uint32_t r;
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
    return r;
}

// first index in [lo, hi) whose packed word is >= key
__device__ __forceinline__ uint64_t lower_bound_packed(const uint32_t* post, uint64_t lo,
                                                       uint64_t hi, uint32_t key) {
    while (lo < hi) {
        uint64_t mid = lo + ((hi - lo) >> 1);
        if (__ldg(post + mid) < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
// first posting in [lo, hi) of a SHORT term with global row >= row
__device__ __forceinline__ uint64_t lower_bound_row(const uint32_t* post, uint64_t lo,
                                                    uint64_t hi, uint32_t row, uint32_t cb) {
    while (lo < hi) {
        uint64_t mid = lo + ((hi - lo) >> 1);
        if ((__ldg(post + mid) >> cb) < row) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ const uint32_t* tile_row(const DevIndex& ix, int32_t slot) {
    return ix.tile_tab + static_cast<uint64_t>(slot) * (static_cast<uint64_t>(ix.n_tiles) * kSubPerTile + 1);
}

// First posting of term [s0, s1) whose row is >= row (any format).
__device__ __forceinline__ uint64_t first_at_or_after(const DevIndex& ix, int32_t slot, uint64_t s0,
                                                      uint64_t s1, uint32_t row) {
    if (slot < 0) return lower_bound_row(ix.post, s0, s1, row, ix.code_bits);
    uint32_t j = row >> kSubShift;
    if ((row >> kTileShift) >= ix.n_tiles) return s1;
    const uint32_t* tb = tile_row(ix, slot);
    uint64_t lo = s0 + __ldg(tb + j), hi = s0 + __ldg(tb + j + 1);
    return lower_bound_packed(ix.post, lo, hi, (row & (kTile - 1)) << kCodeBitsLong);
}

// Locate `row` in a term's postings and decode its (tf, doc_len).  s0 is the
// TERM START (long terms index their sub-tile table from it), s1 the end of
// the searched range.  Returns false when the document lacks the term.
__device__ __forceinline__ bool find_posting(const DevIndex& ix, int32_t slot, uint64_t s0,
                                             uint64_t s1, uint32_t row, const uint32_t* code_tf,
                                             const uint32_t* code_len, double* tf, double* dl) {
    uint64_t pos;
    uint32_t p;
    bool hit;
    uint32_t code;
    bool esc;
    if (slot < 0) {
        pos = lower_bound_row(ix.post, s0, s1, row, ix.code_bits);
        if (pos >= s1) return false;
        p = __ldg(ix.post + pos);
        hit = (p >> ix.code_bits) == row;
        code = p & ix.esc_short;
        esc = code >= ix.n_codes_short;
    } else {
        uint32_t j = row >> kSubShift;
        const uint32_t* tb = tile_row(ix, slot);
        uint64_t lo = s0 + __ldg(tb + j), hi = s0 + __ldg(tb + j + 1);
        uint32_t local = row & (kTile - 1);
        pos = lower_bound_packed(ix.post, lo, hi, local << kCodeBitsLong);
        if (pos >= hi) return false;
        p = __ldg(ix.post + pos);
        hit = (p >> kCodeBitsLong) == local;
        code = p & kEscLong;
        esc = code >= ix.n_codes;
    }
    if (!hit) return false;
    if (!esc) {
        *tf = code_tf[code];
        *dl = code_len[code];
    } else {
        *tf = __ldg(ix.tf + pos);
        *dl = __ldg(ix.doc_lens + row);
    }
    return true;
}

// canonical ranking (include/hybrid/types.hpp:21-25): score desc, DocId asc
__device__ __forceinline__ bool better(double sa, uint64_t ia, double sb, uint64_t ib) {
    if (sa != sb) return sa > sb;
    return ia < ib;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

__device__ __forceinline__ uint32_t pow2_ceil(uint32_t x) {
    return x <= 1 ? 1 : 1u << (32 - __clz(x - 1));
}

// k-th largest of n >= k non-negative floats (radix select on the bits),
// executed by the first NT threads, synchronised with SYNC().  LOW > 0 stops
// after the byte at bit LOW: the result is the k-th largest with its LOW low
// bits cleared -- a lower bound (relative error < 2^(LOW - 23)) in fewer passes.
template <int NT, typename Sync>
__device__ float block_kth_largest(const float* v, uint32_t n, uint32_t k, uint32_t* hist,
                                   uint32_t* sh, Sync sync, int low = 0) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t prefix = 0, pmask = 0, kk = k;
    for (int shift = 24; shift >= low; shift -= 8) {
        for (int i = tid; i < 256; i += NT) hist[i] = 0;
        sync();
        for (uint32_t i0 = tid; i0 < n; i0 += 4 * NT) {  // four loads in flight
            uint32_t u[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) u[j] = i0 + j * NT < n ? __float_as_uint(v[i0 + j * NT]) : 0u;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (i0 + j * NT < n && (u[j] & pmask) == prefix) atomicAdd(&hist[(u[j] >> shift) & 255u], 1u);
        }
        sync();
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
        sync();
        prefix = sh[0];
        kk = sh[1];
        pmask |= 255u << shift;
    }
    sync();
    return __uint_as_float(prefix);
}

// In-place bitonic sort, "better" (score desc, id asc) first, by NT threads.
// n is a power of two; entries past the live count hold (-inf, ~0).
template <int NT, typename Row, typename Sync>
__device__ void block_bitonic(double* sc, uint64_t* id, Row* row, uint32_t n, Sync sync) {
    for (uint32_t k = 2; k <= n; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < n; i += NT) {
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
            sync();
        }
    }
}

// The real query and the row window of (slab) query q (BatchArgs::split).
__device__ __forceinline__ void query_window(const BatchArgs& a, uint32_t q, uint32_t& qr, uint32_t& lo,
                                             uint32_t& hi) {
    if (a.split <= 1) {
        qr = q;
        lo = a.row_lo;
        hi = a.row_hi;
        return;
    }
    qr = q % a.nq_real;
    const uint32_t s = q / a.nq_real;
    if (a.slab_row) {
        lo = a.slab_row[s];
        hi = a.slab_row[s + 1];
        return;
    }
    const uint64_t span = a.row_hi - a.row_lo;
    lo = a.row_lo + static_cast<uint32_t>(span * s / a.split);
    hi = a.row_lo + static_cast<uint32_t>(span * (s + 1) / a.split);
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

// warp-0 in-place compaction of (row, score) pairs that satisfy keep(row, v)
template <typename Keep>
__device__ __forceinline__ uint32_t warp_compact(uint32_t* rows, float* vals, uint32_t n, Keep keep) {
    const int lane = threadIdx.x & 31;
    uint32_t w = 0;
    for (uint32_t b0 = 0; b0 < n; b0 += 32) {
        uint32_t i = b0 + lane;
        uint32_t row = 0;
        float v = 0.f;
        bool kp = false;
        if (i < n) {
            row = rows[i];
            v = vals[i];
            kp = keep(row, v);
        }
        uint32_t bal = __ballot_sync(0xffffffffu, kp);
        uint32_t pos = w + __popc(bal & ((1u << lane) - 1));
        __syncwarp();
        if (kp) {
            rows[pos] = row;
            vals[pos] = v;
        }
        w += __popc(bal);
        __syncwarp();
    }
    return w;
}

}  // namespace hm
