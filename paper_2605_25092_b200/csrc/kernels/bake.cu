// bake_kernel: the survey's K0 -- turns the parameter-free
// long-term postings (tile-local row + (tf, len) code) into the streaming
// format of the fused search kernel for one Bm25Params (k1, b) (layout:
// hm_types.h): one word per posting carrying the accumulator offset and the
// idf-free impact w = tf*(k1+1)/(tf + k1*(1-b+b*len/avgdl)) -- the
// reference's bm25_score (src/csr_index.cpp:10-15) without the idf factor,
// raw tf (pitfall 1) -- evaluated in fp64, rounded to fp32,
// scaled by 2^-ks and truncated to 16 mantissa bits.  Escaped postings (pairs
// outside the code table) read tf[] and doc_lens[] here once, so the search
// kernel never does.  An impact outside the 7 representable binades sets
// *err; the host then serves those parameters with the exact fp64 kernel.
//
// Each (term, 2048-row unit) range is padded to a multiple of 4 words with
// NULL postings (impact 0) that point at rows the term does NOT contain in the
// unit: adding or storing 0 there is harmless and cannot race with the term's
// real postings.  The search kernel then reads whole 16-byte chunks only.
//
// Bank-interleaved order.  Inside a range the kernel may apply postings in any
// order (a term's rows are distinct), so the bake permutes each range such
// that the 32 postings one read-modify-write instruction touches sit in
// distinct shared-memory banks where possible: postings are layered (layer k
// = the k-th posting of every bank, banks ascending), the NULLs go last, and
// the sequence is dealt into the kernel's instruction groups -- per block of
// 32 chunks its 4 component groups (.x of every lane, .y, .z, .w).  A group
// then spans at most two layers: conflict degree 1-2 instead of ~3.5 for rows
// in posting order.  post[] keeps the row order (exact rescoring searches it).
//
// One warp per (long term, unit); rows come from the sub-tile table.
#include <cstring>

#include "hm_device.cuh"
#include "hm_launch.h"

namespace hm {

constexpr int kBakeWarps = 8;
constexpr int kUnitRows = 1 << kUnitShift;
constexpr int kMaxLayer = kUnitRows / 32;  // a unit has exactly 64 rows per bank

// physical slot (relative to the padded range) of logical position `pos`:
// block = pos / 128 (32 chunks), inside it component group f, lane l
__device__ __forceinline__ uint32_t bake_slot(uint32_t pos, uint32_t nch) {
    const uint32_t blk = pos >> 7, r = pos & 127;
    const uint32_t nb = min(32u, nch - 32 * blk);  // chunks in this block
    const uint32_t f = r / nb, l = r % nb;
    return 4 * (32 * blk + l) + f;
}

__global__ void __launch_bounds__(32 * kBakeWarps) bake_kernel(DevIndex ix, const uint32_t* __restrict__ long_terms,
                                                               uint32_t n_long, double k1, double b, uint32_t ks,
                                                               uint32_t* __restrict__ bk, uint32_t* err) {
    __shared__ uint32_t s_S[kBakeWarps][kMaxLayer + 1];
    __shared__ uint32_t s_mask[kBakeWarps][kMaxLayer];
    __shared__ uint32_t s_cnt[kBakeWarps][32];
    __shared__ uint32_t s_have[kBakeWarps][kUnitRows / 32];  // rows of the unit the term contains
    const uint32_t wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t gw = static_cast<uint64_t>(blockIdx.x) * kBakeWarps + wl;
    const uint64_t units = ix.n_units;
    if (gw >= static_cast<uint64_t>(n_long) * units) return;
    const uint32_t slot = static_cast<uint32_t>(gw / units);
    const uint32_t unit = static_cast<uint32_t>(gw % units);  // global unit index
    const uint32_t j = unit / kUnitsPerTile;                   // tile
    const uint32_t t = long_terms[slot];
    const uint64_t s0 = ix.term_off[t];
    const uint32_t* tb = tile_row(ix, static_cast<int32_t>(slot));
    const uint64_t B = s0 + tb[static_cast<uint64_t>(unit) * kSubPerUnit];
    const uint64_t E = s0 + tb[static_cast<uint64_t>(unit + 1) * kSubPerUnit];
    const uint32_t n = static_cast<uint32_t>(E - B);
    if (n == 0) return;
    const uint32_t* uo = ix.bk_uoff + static_cast<uint64_t>(slot) * (units + 1);
    uint32_t* dst = bk + ix.bk_base[slot] + uo[unit];
    const uint32_t n_pad = uo[unit + 1] - uo[unit], nch = n_pad >> 2;
    // pass 1: postings per bank, presence bitmap
    s_cnt[wl][lane] = 0;
    s_have[wl][lane] = 0;
    s_have[wl][lane + 32] = 0;
    __syncwarp();
    for (uint32_t i = lane; i < n; i += 32) {
        const uint32_t r = (ix.post[B + i] >> kCodeBitsLong) & (kUnitRows - 1);
        atomicAdd(&s_cnt[wl][swz10(r) & 31u], 1u);
        atomicOr(&s_have[wl][r >> 5], 1u << (r & 31));
    }
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
    const uint32_t lo = (ks + 1) << 23, hi = (ks + 1 + kBakeBinades) << 23;  // exponent fields 1..7 after scaling
    uint32_t bad = 0;
    float wmax = 0.f;
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
        const float w = impact32(tf, dl, ix.avgdl, k1, b);
        wmax = fmaxf(wmax, w);
        const uint32_t bits = __float_as_uint(w);
        uint32_t q = 0;
        if (bits >= lo && bits < hi) q = (bits - (ks << 23)) >> (23 - kBakeMantBits);
        else bad = 1;
        const uint32_t pos = s_S[wl][k] + __popc(s_mask[wl][k] & ((1u << bank) - 1u));
        dst[bake_slot(pos, nch)] = (q << 13) | ((swz10(local) & (kUnitRows - 1)) << 2);
    }
    // NULL padding (<= 3 words): impact 0 on rows the term lacks in this unit
    if (lane == 0) {
        uint32_t pos = n, w = 0;
        while (pos < n_pad) {
            const uint32_t miss = ~s_have[wl][w];
            if (miss == 0) {
                ++w;
                continue;
            }
            const uint32_t bit = __ffs(miss) - 1;
            s_have[wl][w] |= 1u << bit;
            const uint32_t r = (w << 5) | bit;
            dst[bake_slot(pos, nch)] = swz10(r) << 2;
            ++pos;
        }
    }
    // the term's max impact (non-negative floats order like their bit patterns)
    for (int o = 16; o > 0; o >>= 1) wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
    if (lane == 0) atomicMax(reinterpret_cast<unsigned int*>(const_cast<float*>(ix.tmax) + t), __float_as_uint(wmax));
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, 1u);
}

// Max impact of every SHORT term (long terms get theirs in bake_kernel).
__global__ void tmax_short_kernel(DevIndex ix, double k1, double b, float* __restrict__ tmax) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ix.n_terms || ix.long_slot[t] >= 0) return;
    const uint32_t cb = ix.code_bits;
    float m = 0.f;
    for (uint64_t i = ix.term_off[t]; i < ix.term_off[t + 1]; ++i) {
        const uint32_t p = ix.post[i], code = p & ix.esc_short;
        double tf, dl;
        if (code < ix.n_codes_short) {
            tf = ix.code_tf[code];
            dl = ix.code_len[code];
        } else {
            tf = ix.tf[i];
            dl = ix.doc_lens[p >> cb];
        }
        m = fmaxf(m, impact32(tf, dl, ix.avgdl, k1, b));
    }
    tmax[t] = m;
}

// impact scale: float(k1 + 1), the largest possible impact (tf -> inf, or
// b = 1 and len = 0), lands in exponent field 7 once multiplied by 2^-ks
uint32_t bake_ks(double k1) {
    const float top = static_cast<float>(k1 + 1.0);
    uint32_t bits;
    memcpy(&bits, &top, 4);
    const uint32_t e = bits >> 23;
    return e > static_cast<uint32_t>(kBakeBinades) ? e - kBakeBinades : 0u;
}

cudaError_t launch_bake(const DevIndex& ix, const uint32_t* long_terms, uint32_t n_long, double k1,
                        double b, uint32_t ks, uint32_t* bk, uint32_t* err, cudaStream_t st) {
    const uint64_t warps = static_cast<uint64_t>(n_long) * ix.n_units;
    if (warps) {
        const uint64_t blocks = (warps + kBakeWarps - 1) / kBakeWarps;
        bake_kernel<<<static_cast<unsigned>(blocks), 32 * kBakeWarps, 0, st>>>(ix, long_terms, n_long, k1, b, ks, bk, err);
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (ix.n_terms)
        tmax_short_kernel<<<(ix.n_terms + 255) / 256, 256, 0, st>>>(ix, k1, b, const_cast<float*>(ix.tmax));
    return cudaGetLastError();
}

}  // namespace hm
