// The "wide" path: exhaustive fp64 BM25 for any k and any plan length.
//
// The reference's CsrIndex::bm25_topk takes any k and any number of query
// terms (include/hybrid/csr_index.hpp:72-79; collect_topk has no cap,
// src/csr_index.cpp:50-59).  The fast kernels hold per-query plan state and
// candidate lists in shared memory (k <= 256, <= 256 distinct terms); every
// query beyond that runs here, as a group of G queries at a time:
//
//   wide_init_kernel     per query: postings_touched inside the window (the
//                        reference's sum of df, :100-102) and the selection
//                        state
//   wide_score_kernel    one CTA per (16,384-row tile, query): fp64
//                        accumulators in shared memory, the plan's terms
//                        applied strictly in plan order, each posting added
//                        `mult` times (src/csr_index.cpp:87-101) -- the
//                        reference's bits by construction; the tile's scores
//                        are written to a [G][span] fp64 array in HBM
//   wide_hist/scan       exact radix select of the k-th best document under
//                        the reference's strict order (score desc, DocId asc,
//                        include/hybrid/types.hpp:21-25): the 128-bit key
//                        (score bits, ~DocId) is resolved 8 bits per pass,
//                        most significant first, stopping as soon as the
//                        k-th key's bucket is taken whole
//   wide_compact_kernel  the (at most k) documents with key >= the k-th key
//   DeviceMergeSort      the G x k candidates by (query, score desc, DocId asc)
//   wide_finish_kernel   ranked lists (zero scores dropped), Margin + skip
//
// Bytes per query: the plan's postings once (4 B packed + escapes) plus
// ~3-6 passes over 8 B x span of scores.  Launches per group: ~12 + 2 x passes.
#include <cub/cub.cuh>

#include "hm_device.cuh"
#include "hm_launch.h"

namespace hm {

constexpr int kWideThreads = 512;
constexpr int kWideChunk = 512;  // plan terms whose tile ranges are resolved together

struct WideSmem {
    double acc[kTile];
    uint64_t b[kWideChunk], e[kWideChunk];
    double idf[kWideChunk];
    uint32_t mult[kWideChunk];
    int32_t slot[kWideChunk];
    uint32_t code_tf[kMaxCodes], code_len[kMaxCodes];
};

__global__ void wide_init_kernel(DevIndex ix, BatchArgs a, WideArgs w) {
    const uint32_t g = blockIdx.x;
    const uint32_t q = w.qlist[g];
    const uint32_t poff = a.q_off[q], m = a.plan_len[q];
    __shared__ unsigned long long post;
    if (threadIdx.x == 0) post = 0;
    __syncthreads();
    uint64_t my = 0;
    for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
        const uint32_t t = a.plan_tid[poff + i];
        const int32_t slot = ix.long_slot[t];
        const uint64_t s0 = ix.term_off[t], s1 = ix.term_off[t + 1];
        const uint64_t w0 = a.row_lo > 0 ? first_at_or_after(ix, slot, s0, s1, a.row_lo) : s0;
        const uint64_t w1 = a.row_hi < ix.n_docs ? first_at_or_after(ix, slot, s0, s1, a.row_hi) : s1;
        my += w1 - w0;
    }
    if (my) atomicAdd(&post, static_cast<unsigned long long>(my));
    for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) w.hist[g * 256 + i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) {
        WideState& s = w.st[g];
        s.pre_hi = 0;
        s.pre_lo = 0;
        s.kr = a.k;
        s.done = (m == 0 || a.k == 0 || a.row_hi <= a.row_lo) ? 1u : 0u;
        s.take_all = s.done;
        s.n_c = 0;
        s.post = post;
    }
}

__global__ void __launch_bounds__(kWideThreads, 1) wide_score_kernel(DevIndex ix, BatchArgs a, WideArgs w) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WideSmem& S = *reinterpret_cast<WideSmem*>(smem_raw);
    const uint32_t g = blockIdx.y;
    const uint32_t q = w.qlist[g];
    const uint32_t poff = a.q_off[q], m = a.plan_len[q];
    const int tid = threadIdx.x;
    const uint32_t cb = ix.code_bits;
    const double k1 = a.k1, bb = a.b;
    const uint32_t j = (a.row_lo >> kTileShift) + blockIdx.x;
    const uint32_t base = j << kTileShift;
    const uint32_t R0 = max(base, a.row_lo), R1 = min(base + kTile, a.row_hi);
    if (R0 >= R1) return;
    const uint32_t rlo = R0 - base, rn = R1 - R0;
    for (int i = tid; i < kTile; i += kWideThreads) S.acc[i] = 0.0;
    for (int i = tid; i < kMaxCodes; i += kWideThreads) {
        S.code_tf[i] = ix.code_tf[i];
        S.code_len[i] = ix.code_len[i];
    }
    for (uint32_t c0 = 0; c0 < m; c0 += kWideChunk) {
        const uint32_t cn = min(m - c0, static_cast<uint32_t>(kWideChunk));
        __syncthreads();
        if (static_cast<uint32_t>(tid) < cn) {  // this tile's posting range of each term
            const uint32_t t = a.plan_tid[poff + c0 + tid];
            const int32_t slot = ix.long_slot[t];
            const uint64_t s0 = ix.term_off[t], s1 = ix.term_off[t + 1];
            uint64_t b0, e0;
            if (slot >= 0) {
                const uint32_t* tb = tile_row(ix, slot);
                b0 = s0 + __ldg(tb + static_cast<uint64_t>(j) * kSubPerTile);
                e0 = s0 + __ldg(tb + static_cast<uint64_t>(j + 1) * kSubPerTile);
            } else {
                b0 = lower_bound_row(ix.post, s0, s1, R0, cb);
                e0 = lower_bound_row(ix.post, b0, s1, R1, cb);
            }
            S.b[tid] = b0;
            S.e[tid] = e0;
            S.slot[tid] = slot;
            S.idf[tid] = ix.idf[t];
            S.mult[tid] = a.plan_mult[poff + c0 + tid];
        }
        __syncthreads();
        for (uint32_t i = 0; i < cn; ++i) {  // plan order (src/csr_index.cpp:87-101)
            const uint64_t b0 = S.b[i], e0 = S.e[i];
            const double idf = S.idf[i];
            const uint32_t mu = S.mult[i];
            const bool lng = S.slot[i] >= 0;
            for (uint64_t x = b0 + tid; x < e0; x += kWideThreads) {
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
    }
    __syncthreads();
    double* out = w.scores + static_cast<uint64_t>(g) * w.span + (R0 - a.row_lo);
    for (uint32_t r = tid; r < rn; r += kWideThreads) out[r] = S.acc[rlo + r];
}

// the 128-bit ranking key of a document: (score bits, ~DocId); positive
// doubles order like their bit patterns, so a larger key is a better document
__device__ __forceinline__ uint32_t wide_digit(uint64_t hi, uint64_t lo, int p) {
    return p < 8 ? static_cast<uint32_t>(hi >> (56 - 8 * p)) & 255u
                 : static_cast<uint32_t>(lo >> (56 - 8 * (p - 8))) & 255u;
}
// do the key's first 8p bits equal the prefix?
__device__ __forceinline__ bool wide_match(uint64_t hi, uint64_t lo, const WideState& s, int p) {
    if (p == 0) return true;
    if (p <= 8) return (hi >> (64 - 8 * p)) == (s.pre_hi >> (64 - 8 * p));
    if (hi != s.pre_hi) return false;
    return p == 8 || (lo >> (64 - 8 * (p - 8))) == (s.pre_lo >> (64 - 8 * (p - 8)));
}

__global__ void wide_hist_kernel(DevIndex ix, BatchArgs a, WideArgs w, int p) {
    const uint32_t g = blockIdx.y;
    const WideState s = w.st[g];
    if (s.done) return;
    __shared__ uint32_t h[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const double* sc = w.scores + static_cast<uint64_t>(g) * w.span;
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < w.span; r += gridDim.x * blockDim.x) {
        const double v = sc[r];
        if (!(v > 0.0)) continue;
        const uint64_t hi = static_cast<uint64_t>(__double_as_longlong(v));
        const uint64_t lo = p >= 8 ? ~__ldg(ix.doc_ids + a.row_lo + r) : 0ull;
        if (wide_match(hi, lo, s, p)) atomicAdd(&h[wide_digit(hi, lo, p)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += blockDim.x)
        if (h[i]) atomicAdd(&w.hist[g * 256 + i], h[i]);
}

// one warp per query: pick the digit of the k-th key, narrow the rank
__global__ void wide_scan_kernel(WideArgs w, int p) {
    const uint32_t g = blockIdx.x;
    WideState& s = w.st[g];
    uint32_t* h = w.hist + g * 256;
    if (s.done) return;
    const int lane = threadIdx.x;
    uint32_t loc[8], tot = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        loc[j] = h[lane * 8 + j];
        tot += loc[j];
    }
    uint32_t incl = tot;  // keys in the buckets of lanes >= lane
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t nb = __shfl_down_sync(0xffffffffu, incl, o);
        if (lane + o < 32) incl += nb;
    }
    const uint32_t all = __shfl_sync(0xffffffffu, incl, 0);
    const uint32_t kr = s.kr;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 8; ++j) h[lane * 8 + j] = 0;
    if (p == 0 && all <= kr) {  // at most k positive documents: all of them
        if (lane == 0) {
            s.take_all = 1;
            s.done = 1;
        }
        return;
    }
    const uint32_t above = incl - tot;
    if (above < kr && kr <= incl) {
        uint32_t cum = above;
        for (int j = 7; j >= 0; --j) {
            if (cum + loc[j] >= kr) {
                const uint64_t d = static_cast<uint64_t>(lane * 8 + j);
                if (p < 8) s.pre_hi |= d << (56 - 8 * p);
                else s.pre_lo |= d << (56 - 8 * (p - 8));
                s.kr = kr - cum;
                // the whole bucket is needed: key >= prefix selects exactly k
                if (loc[j] == kr - cum || p == 15) s.done = 1;
                break;
            }
            cum += loc[j];
        }
    }
}

__global__ void wide_compact_kernel(DevIndex ix, BatchArgs a, WideArgs w) {
    const uint32_t g = blockIdx.y;
    const WideState s = w.st[g];
    const double* sc = w.scores + static_cast<uint64_t>(g) * w.span;
    WideCand* out = w.cand + static_cast<uint64_t>(g) * a.k;
    const int lane = threadIdx.x & 31;
    for (uint32_t r0 = blockIdx.x * blockDim.x; r0 < w.span; r0 += gridDim.x * blockDim.x) {
        const uint32_t r = r0 + threadIdx.x;
        bool keep = false;
        uint64_t hi = 0, id = 0;
        if (r < w.span) {
            const double v = sc[r];
            if (v > 0.0) {
                hi = static_cast<uint64_t>(__double_as_longlong(v));
                id = __ldg(ix.doc_ids + a.row_lo + r);
                keep = s.take_all || hi > s.pre_hi || (hi == s.pre_hi && ~id >= s.pre_lo);
            }
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        if (!bal) continue;
        uint32_t pos = 0;
        if (lane == __ffs(bal) - 1) pos = atomicAdd(&w.st[g].n_c, __popc(bal));
        pos = __shfl_sync(0xffffffffu, pos, __ffs(bal) - 1) + __popc(bal & ((1u << lane) - 1u));
        if (keep && pos < a.k) out[pos] = WideCand{g, hi, id};
    }
}

__global__ void wide_fill_kernel(WideCand* c, uint32_t k, uint32_t G) {
    const uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < static_cast<uint64_t>(G) * k) c[i] = WideCand{static_cast<uint32_t>(i / k), 0ull, ~0ull};
}

struct WideLess {
    __device__ bool operator()(const WideCand& x, const WideCand& y) const {
        if (x.g != y.g) return x.g < y.g;
        if (x.bits != y.bits) return x.bits > y.bits;
        return x.id < y.id;
    }
};

__global__ void wide_finish_kernel(BatchArgs a, WideArgs w) {
    const uint32_t g = blockIdx.x;
    const uint32_t q = w.qlist[g];
    const WideCand* c = w.cand + static_cast<uint64_t>(g) * a.k;
    const uint64_t o = static_cast<uint64_t>(q) * a.k;
    __shared__ uint32_t n;
    if (threadIdx.x == 0) n = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < a.k; i += blockDim.x) {
        const double v = __longlong_as_double(static_cast<long long>(c[i].bits));
        if (c[i].bits != 0 && v > 0.0) {
            a.out_ids[o + i] = c[i].id;
            a.out_scores[o + i] = v;
            atomicMax(&n, i + 1);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        a.out_n[q] = n;
        if (a.out_post) a.out_post[q] = w.st[g].post;
        write_decision(a, q, a.out_scores + o, n);
    }
}

static bool g_wide_attr = false;

size_t wide_sort_bytes(uint64_t n_items) {
    size_t bytes = 0;
    cub::DeviceMergeSort::SortKeys(nullptr, bytes, static_cast<WideCand*>(nullptr), static_cast<int64_t>(n_items),
                                   WideLess{});
    return bytes;
}

cudaError_t launch_wide_group(const DevIndex& ix, const BatchArgs& a, const WideArgs& w, void* sort_tmp,
                              size_t sort_bytes, cudaStream_t st) {
    cudaError_t e;
    if (!g_wide_attr) {
        e = cudaFuncSetAttribute(wide_score_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(sizeof(WideSmem)));
        if (e != cudaSuccess) return e;
        g_wide_attr = true;
    }
    if (w.G == 0 || a.k == 0) return cudaSuccess;
    wide_init_kernel<<<w.G, 256, 0, st>>>(ix, a, w);
    if (w.span > 0) {
        const uint32_t tiles = ((a.row_hi - 1) >> kTileShift) - (a.row_lo >> kTileShift) + 1;
        wide_score_kernel<<<dim3(tiles, w.G), kWideThreads, sizeof(WideSmem), st>>>(ix, a, w);
        const uint32_t blocks = min((w.span + 1023u) / 1024u, 1184u);
        for (int p = 0; p < 16; ++p) {
            wide_hist_kernel<<<dim3(blocks, w.G), 256, 0, st>>>(ix, a, w, p);
            wide_scan_kernel<<<w.G, 32, 0, st>>>(w, p);
        }
    }
    const uint64_t n_items = static_cast<uint64_t>(w.G) * a.k;
    wide_fill_kernel<<<static_cast<uint32_t>((n_items + 255) / 256), 256, 0, st>>>(w.cand, a.k, w.G);
    if (w.span > 0) {
        const uint32_t blocks = min((w.span + 1023u) / 1024u, 1184u);
        wide_compact_kernel<<<dim3(blocks, w.G), 256, 0, st>>>(ix, a, w);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    e = cub::DeviceMergeSort::SortKeys(sort_tmp, sort_bytes, w.cand, static_cast<int64_t>(n_items), WideLess{}, st);
    if (e != cudaSuccess) return e;
    wide_finish_kernel<<<w.G, 256, 0, st>>>(a, w);
    return cudaGetLastError();
}

}  // namespace hm
