// bake_kernel: the survey's K0 -- turns the parameter-free
// long-term postings (tile-local row + (tf, len) code) into the streaming
// format of the fused search kernel for one Bm25Params (k1, b):
//
//   bk[i] = (q19 << 13) | ((swz10(r) & 2047) << 2)       (layout: hm_types.h)
//
// with the idf-free impact w = tf*(k1+1)/(tf + k1*(1-b+b*len/avgdl)) -- the
// reference's bm25_score (src/csr_index.cpp:10-15) without the idf factor,
// raw tf (pitfall 1) -- evaluated in fp64, rounded to fp32
// and truncated to 3 exponent + 16 mantissa bits.  Escaped postings (pairs
// outside the code table) read tf[] and doc_lens[] here once, so the search
// kernel never does.  An impact outside the 8 representable binades sets
// *err; the host then serves those parameters with the exact fp64 kernel.
//
// Bank-interleaved order.  Inside one (term, 2048-row unit) range the search
// kernel may apply postings in any order (a term's rows are distinct), so the
// bake permutes each range such that the 32 postings one read-modify-write
// instruction touches sit in distinct shared-memory banks where possible: the
// range's postings are layered (layer k = the k-th posting of every bank,
// banks ascending) and the layers are dealt, in order, into the kernel's
// instruction groups -- first the <= 6 unaligned head/tail words (one
// instruction), then for every block of 32 16-byte chunks its 4 component
// groups (.x of every lane, .y, .z, .w).  A group then spans at most two
// layers, so its conflict degree is 1 or 2 instead of ~3.5 for rows in
// posting order.  post[] keeps the row order (exact rescoring searches it).
//
// One warp per (long term, unit); rows come from the sub-tile table.
#include <cstring>

#include "hm_device.cuh"
#include "hm_launch.h"

namespace hm {

constexpr int kBakeWarps = 8;
constexpr int kUnitShiftB = 11;  // must match search_fast.cu (2048-row warp units)
constexpr int kSubPerUnitB = 1 << (kUnitShiftB - kSubShift);
constexpr int kUnitsPerTile = kTile >> kUnitShiftB;
constexpr int kMaxLayer = (1 << kUnitShiftB) / 32;  // <= 64 rows of a unit per bank

// physical slot (relative to the range start) of logical position `pos`:
// the boundary instruction (h head + tl tail words), then per 32-chunk block
// its 4 component groups
__device__ __forceinline__ uint32_t bake_slot(uint32_t pos, uint32_t h, uint32_t nc, uint32_t tl) {
    const uint32_t nbd = h + tl;
    if (pos < nbd) return pos < h ? pos : h + 4 * nc + (pos - h);
    const uint32_t q = pos - nbd, blk = q >> 7, r = q & 127;
    const uint32_t nb = min(32u, nc - 32 * blk);  // chunks in this block
    const uint32_t f = r / nb, l = r % nb;
    return h + 4 * (32 * blk + l) + f;
}

__global__ void __launch_bounds__(32 * kBakeWarps) bake_kernel(DevIndex ix, const uint32_t* __restrict__ long_terms,
                                                               uint32_t n_long, double k1, double b, uint32_t eb,
                                                               uint32_t* __restrict__ bk, uint32_t* err) {
    __shared__ uint32_t s_S[kBakeWarps][kMaxLayer + 1];
    __shared__ uint32_t s_mask[kBakeWarps][kMaxLayer];
    __shared__ uint32_t s_cnt[kBakeWarps][32];
    const uint32_t wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kBakeWarps + wl;
    const uint64_t units = static_cast<uint64_t>(ix.n_tiles) * kUnitsPerTile;
    if (gw >= static_cast<uint64_t>(n_long) * units) return;
    const uint32_t slot = static_cast<uint32_t>(gw / units);
    const uint32_t unit = static_cast<uint32_t>(gw % units);  // global unit index
    const uint32_t j = unit / kUnitsPerTile;                   // tile
    const uint32_t t = long_terms[slot];
    const uint64_t s0 = ix.term_off[t];
    const uint32_t* tb = tile_row(ix, static_cast<int32_t>(slot));
    const uint64_t B = s0 + tb[static_cast<uint64_t>(unit) * kSubPerUnitB];
    const uint64_t E = s0 + tb[static_cast<uint64_t>(unit + 1) * kSubPerUnitB];
    const uint32_t n = static_cast<uint32_t>(E - B);
    if (n == 0) return;
    // pass 1: postings per bank (smem counters of this warp; lane b reads bank b)
    s_cnt[wl][lane] = 0;
    __syncwarp();
    for (uint32_t i = lane; i < n; i += 32) atomicAdd(&s_cnt[wl][swz10(ix.post[B + i] >> kCodeBitsLong) & 31u], 1u);
    __syncwarp();
    const uint32_t cnt = s_cnt[wl][lane];
    __syncwarp();
    s_cnt[wl][lane] = 0;  // reused below: postings of each bank placed so far
    // layer tables: S[k] = postings in layers < k; mask[k] = banks with > k postings
    uint32_t S = 0;
    for (uint32_t k = 0; k < kMaxLayer; ++k) {
        const uint32_t m = __ballot_sync(0xffffffffu, cnt > k);
        if (lane == 0) {
            s_S[wl][k] = S;
            s_mask[wl][k] = m;
        }
        S += __popc(m);
    }
    __syncwarp();
    const uint32_t h = min(static_cast<uint32_t>((4u - (static_cast<uint32_t>(B) & 3u)) & 3u), n);
    const uint32_t body = n - h, nc = body >> 2, tl = body & 3;
    const uint32_t lim = eb + (static_cast<uint32_t>(kBakeBinades) << 23);
    uint32_t bad = 0;
    for (uint32_t i = lane; i < n; i += 32) {
        const uint32_t p = ix.post[B + i];
        const uint32_t local = p >> kCodeBitsLong;  // row inside the 16K tile
        const uint32_t bank = swz10(local) & 31u;
        const uint32_t k = atomicAdd(&s_cnt[wl][bank], 1u);  // any bijection onto 0..cnt-1 works
        const uint32_t code = p & kEscLong;
        double tf, dl;
        if (code < ix.n_codes) {
            tf = ix.code_tf[code];
            dl = ix.code_len[code];
        } else {
            tf = ix.tf[B + i];
            dl = ix.doc_lens[(j << kTileShift) + local];
        }
        const uint32_t bits = __float_as_uint(impact32(tf, dl, ix.avgdl, k1, b));
        uint32_t q = 0;
        if (bits >= eb && bits < lim) q = (bits - eb) >> (23 - kBakeMantBits);
        else bad = 1;
        const uint32_t pos = s_S[wl][k] + __popc(s_mask[wl][k] & ((1u << bank) - 1u));
        bk[B + bake_slot(pos, h, nc, tl)] = (q << 13) | ((swz10(local) & 2047u) << 2);
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, 1u);
}

// float bits of the lowest binade of the baked range: the top binade holds
// k1 + 1, the largest possible impact (tf -> inf, or b = 1 and len = 0)
uint32_t bake_eb(double k1) {
    const float top = static_cast<float>(k1 + 1.0);
    uint32_t bits;
    memcpy(&bits, &top, 4);
    const uint32_t e = bits >> 23;
    const uint32_t e_lo = e >= kBakeBinades ? e - (kBakeBinades - 1) : 1;
    return e_lo << 23;
}

cudaError_t launch_bake(const DevIndex& ix, const uint32_t* long_terms, uint32_t n_long, double k1,
                        double b, uint32_t eb, uint32_t* bk, uint32_t* err, cudaStream_t st) {
    const uint64_t warps = static_cast<uint64_t>(n_long) * ix.n_tiles * kUnitsPerTile;
    if (warps == 0) return cudaSuccess;
    const uint64_t blocks = (warps + kBakeWarps - 1) / kBakeWarps;
    bake_kernel<<<static_cast<unsigned>(blocks), 32 * kBakeWarps, 0, st>>>(ix, long_terms, n_long, k1, b, eb, bk, err);
    return cudaGetLastError();
}

}  // namespace hm
