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
// One warp per (long term, 16K-row tile): the tile's postings come from the
// sub-tile table, the tile index restores the global row of escapes.
#include <cstring>

#include "hm_device.cuh"
#include "hm_launch.h"

namespace hm {

__global__ void bake_kernel(DevIndex ix, const uint32_t* __restrict__ long_terms, uint32_t n_long,
                            double k1, double b, uint32_t eb, uint32_t* __restrict__ bk,
                            uint32_t* err) {
    const uint64_t gw = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (gw >= static_cast<uint64_t>(n_long) * ix.n_tiles) return;
    const uint32_t slot = static_cast<uint32_t>(gw / ix.n_tiles);
    const uint32_t j = static_cast<uint32_t>(gw % ix.n_tiles);
    const uint32_t t = long_terms[slot];
    const uint64_t s0 = ix.term_off[t];
    const uint32_t* tb = tile_row(ix, static_cast<int32_t>(slot));
    const uint64_t lo = s0 + tb[static_cast<uint64_t>(j) * kSubPerTile];
    const uint64_t hi = s0 + tb[static_cast<uint64_t>(j + 1) * kSubPerTile];
    const uint32_t lim = eb + (static_cast<uint32_t>(kBakeBinades) << 23);
    uint32_t bad = 0;
    for (uint64_t i = lo + lane; i < hi; i += 32) {
        const uint32_t p = ix.post[i];
        const uint32_t local = p >> kCodeBitsLong;  // row inside the 16K tile
        const uint32_t code = p & kEscLong;
        double tf, dl;
        if (code < ix.n_codes) {
            tf = ix.code_tf[code];
            dl = ix.code_len[code];
        } else {
            tf = ix.tf[i];
            dl = ix.doc_lens[(j << kTileShift) + local];
        }
        const uint32_t bits = __float_as_uint(impact32(tf, dl, ix.avgdl, k1, b));
        uint32_t q = 0;
        if (bits >= eb && bits < lim) q = (bits - eb) >> (23 - kBakeMantBits);
        else bad = 1;
        bk[i] = (q << 13) | ((swz10(local) & 2047u) << 2);
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
    const uint64_t warps = static_cast<uint64_t>(n_long) * ix.n_tiles;
    if (warps == 0) return cudaSuccess;
    const uint64_t blocks = (warps * 32 + 255) / 256;
    bake_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(ix, long_terms, n_long, k1, b, eb, bk, err);
    return cudaGetLastError();
}

}  // namespace hm
