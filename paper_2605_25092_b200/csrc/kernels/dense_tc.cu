// Dense escalate channel, tensor-core path: candidate generation with
// tcgen05 TF32 MMAs, exact fp64 rescoring of the candidates.
//
// S = Q E^T is a GEMM (queries x rows x dim).  The 5th-generation tensor
// cores compute it in TF32 with fp32 accumulation into TMEM; the reference's
// scores are fp64 sums (src/dense.cpp:95-97), so the GEMM only SELECTS:
//
//   |S~ - S| <= err = 1.25 (2^-9 + 2^-20 + dim 2^-22) ||q|| max_r ||r||
//
// (TF32 keeps 10 of the 23 mantissa bits of each input: relative error
// < 2^-10 per factor; fp32 accumulation adds at most one rounding per
// product).  Each epilogue thread owns one query row of the accumulator tile
// and keeps the best KT approximate scores of its slab in registers; once it
// holds k, every row with S~ >= kth - 2 err is a candidate (k rows with
// S >= kth - err exist, so the exact k-th score is >= kth - err, and a row of
// the exact top-k has S~ >= S - err >= kth - 2 err).  The bound is published
// per query (atomicMax) so every slab of the query filters with the best one.  dense_rescore_kernel
// then scores the candidates exactly -- the reference's fp64 chain -- and
// ranks them by (score desc, DocId asc): bit-identical output.  A query whose
// candidate list overflows is rescored over every row instead.
//
// Kernel anatomy (one CTA per SM, persistent over (query tile, row slab)):
//   warp 0   TMA producer: per 32-wide K chunk, the 128-query A tile and the
//            256-row B tile (fp32, 128B-swizzled K-major) into a 4-stage ring
//   warp 1   TMEM owner + MMA issuer: 4 x tcgen05.mma.kind::tf32 (M128 N256
//            K8) per chunk into one of two 256-column TMEM accumulators
//   warps 2-9  epilogue (two per TMEM lane quarter, each on half of the 256
//            columns): tcgen05.ld 32x32b.x32, filter, candidate emission
#include <cstdint>

#include <cuda.h>

#include "hm_dense.h"
#include "hm_ptx.cuh"

namespace hm {
namespace {

#ifndef HM_TC_N
#define HM_TC_N 256
#endif
constexpr int kTcM = 128, kTcN = HM_TC_N, kTcKc = 32;  // tile rows, tile columns, K elements per stage
constexpr int kTcAcc = 512 / kTcN;                   // TMEM accumulators (512 columns)
constexpr int kTcStages = 192 * 1024 / (kTcM * 128 + kTcN * 128);
constexpr uint32_t kABytes = kTcM * 128;  // 16 KB: 128 rows x 128 B
constexpr uint32_t kBBytes = kTcN * 128;  // 32 KB
constexpr int kEpiWarps = 8;  // two warps per TMEM lane quarter, each on half the columns
constexpr int kTcThreads = 64 + 32 * kEpiWarps;
constexpr int kEpiCols = kTcN * 4 / kEpiWarps;  // accumulator columns per epilogue warp
constexpr uint32_t kTmemCols = 512;  // kTcAcc accumulators of kTcN columns

struct __align__(1024) TcSmem {
    uint8_t a[kTcStages][kABytes];
    uint8_t b[kTcStages][kBBytes];
    uint64_t full[kTcStages], empty[kTcStages], tfull[kTcAcc], tempty[kTcAcc];
    uint32_t tmem_base;
};

__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_addr(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_addr(bar))
        : "memory");
}

// UMMA shared-memory descriptor: K-major, 128B swizzle, 8-row groups 1024 B
// apart (SBO), version 1 (sm_100)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    uint64_t d = static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
    d |= static_cast<uint64_t>(1) << 16;             // LBO (unused for swizzled K-major)
    d |= static_cast<uint64_t>(1024 >> 4) << 32;     // SBO
    d |= static_cast<uint64_t>(1) << 46;             // descriptor version
    d |= static_cast<uint64_t>(2) << 61;             // SWIZZLE_128B
    return d;
}

// instruction descriptor: D f32, A/B tf32, both K-major, M = 128, N = 256
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((kTcN >> 3) << 17) | ((kTcM >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(kIdesc), "r"(accum)
        : "memory");
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// order-preserving float <-> int (atomicMax on the shared per-query bound)
__device__ __forceinline__ int f2key(float f) {
    const int i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float key2f(int k) { return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff); }

template <int KT>
__global__ void __launch_bounds__(kTcThreads, 1)
    dense_tc_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_e,
                    DenseTcArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // the swizzled stages need 1024-byte alignment
    TcSmem& S = *reinterpret_cast<TcSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t n_kc = a.dim / kTcKc;
    const uint32_t n_qt = (a.nq + kTcM - 1) / kTcM;
    const uint32_t n_tiles = (a.n_rows + kTcN - 1) / kTcN;
    const uint32_t n_items = n_qt * a.n_slabs;
    auto slab_tiles = [&](uint32_t s, uint32_t& t0, uint32_t& t1) {
        t0 = static_cast<uint32_t>((static_cast<uint64_t>(n_tiles) * s) / a.n_slabs);
        t1 = static_cast<uint32_t>((static_cast<uint64_t>(n_tiles) * (s + 1)) / a.n_slabs);
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            mbar_init(&S.full[s], 1);
            mbar_init(&S.empty[s], 1);
        }
        for (int s = 0; s < kTcAcc; ++s) {
            mbar_init(&S.tfull[s], 1);
            mbar_init(&S.tempty[s], kEpiWarps * 32);
        }
        mbar_init_fence();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&S.tmem_base)),
                     "n"(kTmemCols)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = S.tmem_base;

    if (warp == 0) {
        // ================= TMA producer
        if (lane == 0) {
            uint32_t stage = 0, phase = 0;
            for (uint32_t it = blockIdx.x; it < n_items; it += gridDim.x) {
                const uint32_t qt = it % n_qt, slab = it / n_qt;
                uint32_t t0, t1;
                slab_tiles(slab, t0, t1);
                for (uint32_t t = t0; t < t1; ++t)
                    for (uint32_t kc = 0; kc < n_kc; ++kc) {
                        mbar_wait(&S.empty[stage], phase ^ 1);
                        mbar_arrive_tx(&S.full[stage], kABytes + kBBytes);
                        tma_2d(S.a[stage], &map_q, kc * kTcKc, qt * kTcM, &S.full[stage]);
                        tma_2d(S.b[stage], &map_e, kc * kTcKc, t * kTcN, &S.full[stage]);
                        if (++stage == kTcStages) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
            }
        }
    } else if (warp == 1) {
        // ================= MMA issuer
        if (lane == 0) {
            uint32_t stage = 0, phase = 0, acc = 0, aphase = 0;
            for (uint32_t it = blockIdx.x; it < n_items; it += gridDim.x) {
                const uint32_t slab = it / n_qt;
                uint32_t t0, t1;
                slab_tiles(slab, t0, t1);
                for (uint32_t t = t0; t < t1; ++t) {
                    mbar_wait(&S.tempty[acc], aphase ^ 1);  // the epilogue drained this accumulator
                    tc_fence_after();
                    const uint32_t d = tmem + acc * kTcN;
                    for (uint32_t kc = 0; kc < n_kc; ++kc) {
                        mbar_wait(&S.full[stage], phase);
                        tc_fence_after();
                        const uint64_t ad = umma_desc(smem_addr(S.a[stage]));
                        const uint64_t bd = umma_desc(smem_addr(S.b[stage]));
#pragma unroll
                        for (uint32_t kk = 0; kk < kTcKc / 8; ++kk)  // K = 8 tf32 = 32 B per MMA
                            mma_tf32(d, ad + 2 * kk, bd + 2 * kk, (kc | kk) != 0);
                        mma_commit(&S.empty[stage]);  // frees the stage when these MMAs complete
                        if (++stage == kTcStages) {
                            stage = 0;
                            phase ^= 1;
                        }
                    }
                    mma_commit(&S.tfull[acc]);
                    if (++acc == kTcAcc) {
                        acc = 0;
                        aphase ^= 1;
                    }
                }
            }
        }
    } else {
        // ================= epilogue: one query row per thread
        const uint32_t quarter = static_cast<uint32_t>(warp & 3);  // TMEM lanes 32*quarter .. +31
        const uint32_t row = quarter * 32 + lane;
        const uint32_t col0 = static_cast<uint32_t>((warp - 2) / 4) * kEpiCols;  // my half of the columns
        uint32_t acc = 0, aphase = 0;
        for (uint32_t it = blockIdx.x; it < n_items; it += gridDim.x) {
            const uint32_t qt = it % n_qt, slab = it / n_qt;
            uint32_t t0, t1;
            slab_tiles(slab, t0, t1);
            const uint32_t q = qt * kTcM + row;
            const bool valid = q < a.nq;
            float err = 0.f;
            if (valid) {
                double nq2 = 0.0;
                const float* qv = a.q + static_cast<uint64_t>(q) * a.dim;
                for (uint32_t j = 0; j < a.dim; ++j) nq2 += static_cast<double>(qv[j]) * qv[j];
                err = static_cast<float>(sqrt(nq2) * a.err_scale) * 1.0001f;
            }
            float top[KT];
#pragma unroll
            for (int i = 0; i < KT; ++i) top[i] = -__int_as_float(0x7f800000);
            float thr = -__int_as_float(0x7f800000);
            for (uint32_t t = t0; t < t1; ++t) {
                mbar_wait(&S.tfull[acc], aphase);
                tc_fence_after();
                const uint32_t taddr = tmem + ((quarter * 32) << 16) + acc * kTcN + col0;
                // pass 1: each 32-column chunk's maximum (FMNMX3 tree); only a
                // chunk that beats the running KT-th value is walked to update
                // the running best KT (and so the bound) -- rare after the
                // first tiles, so a tile costs ~25 instructions per chunk
                const bool tail = t * kTcN + col0 + kEpiCols > a.n_rows;
                float cmax[kEpiCols / 32];
#pragma unroll 1
                for (uint32_t c = 0; c < static_cast<uint32_t>(kEpiCols / 32); ++c) {
                    uint32_t v[32];
                    tmem_ld32(taddr + 32 * c, v);
                    if (tail) {
                        const uint32_t base = t * kTcN + col0 + 32 * c;
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            if (base + i >= a.n_rows) v[i] = 0xff800000u;  // -inf: past the last row
                    }
                    float m = fmaxf(fmaxf(__uint_as_float(v[0]), __uint_as_float(v[1])), __uint_as_float(v[2]));
#pragma unroll
                    for (int i = 3; i < 31; i += 2)
                        m = fmaxf(fmaxf(m, __uint_as_float(v[i])), __uint_as_float(v[i + 1]));
                    m = fmaxf(m, __uint_as_float(v[31]));
                    cmax[c] = m;
                    if (valid && m > top[KT - 1]) {
                        if (t - t0 < 2) {  // warm-up tiles: every value (a tight bound early)
#pragma unroll
                            for (int i = 0; i < 32; ++i) {
                                float x = __uint_as_float(v[i]);
                                if (x > top[KT - 1]) {
#pragma unroll
                                    for (int j = 0; j < KT; ++j)
                                        if (x > top[j]) {
                                            const float y = top[j];
                                            top[j] = x;
                                            x = y;
                                        }
                                }
                            }
                        } else {  // then only the chunk maximum: still real rows' values
                            // (a valid bound; the top-k values of a slab almost never
                            // share a 32-row chunk), and the insertion network runs once
                            // per chunk instead of per value -- per value it cost ~2x the
                            // epilogue, since some lane of the warp nearly always inserts
                            float x = m;
#pragma unroll
                            for (int j = 0; j < KT; ++j)
                                if (x > top[j]) {
                                    const float y = top[j];
                                    top[j] = x;
                                    x = y;
                                }
                        }
                    }
                }
                if (valid) {
                    float kth = top[0];
#pragma unroll
                    for (int j = 0; j < KT; ++j)
                        if (static_cast<uint32_t>(j) + 1 == a.k) kth = top[j];
                    const float t2 = kth - 2.f * err;
                    if (t2 > thr) {
                        thr = t2;
                        atomicMax(a.thr_key + q, f2key(t2));
                    }
                    // the bound other slabs of this query proved (valid for
                    // every slab: it comes from k real rows)
                    thr = fmaxf(thr, key2f(*reinterpret_cast<volatile int*>(a.thr_key + q)));
                }
                // pass 2: candidates, from the chunks whose maximum reaches the bound
#pragma unroll 1
                for (uint32_t c = 0; c < static_cast<uint32_t>(kEpiCols / 32); ++c) {
                    if (!__any_sync(0xffffffffu, valid && cmax[c] >= thr)) continue;
                    uint32_t v[32];
                    tmem_ld32(taddr + 32 * c, v);
                    const uint32_t base = t * kTcN + col0 + 32 * c;
                    if (valid && cmax[c] >= thr) {
#pragma unroll
                        for (int i = 0; i < 32; ++i) {
                            const float x = __uint_as_float(v[i]);
                            if (x >= thr && base + i < a.n_rows) {
                                const uint32_t p = atomicAdd(a.cand_n + q, 1u);
                                if (p < a.cand_cap) a.cand_rows[static_cast<uint64_t>(q) * a.cand_cap + p] = base + i;
                            }
                        }
                    }
                }
                tc_fence_before();
                mbar_arrive(&S.tempty[acc]);
                if (++acc == kTcAcc) {
                    acc = 0;
                    aphase ^= 1;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kTmemCols) : "memory");
    }
}

constexpr int kRsThreads = 256;
constexpr int kRsCap = 8192;  // candidates rescored in shared memory (128 KB)

__device__ __forceinline__ bool better(double sa, uint64_t ia, double sb, uint64_t ib) {
    return sa > sb || (sa == sb && ia < ib);
}

// One CTA per query: exact fp64 scores of the candidates (the reference's
// chain, DFMA: the float x float products are exact), ranked by a bitonic
// sort.  Overflowed lists: every row is scored, keeping a running best list.
__global__ void __launch_bounds__(kRsThreads) dense_rescore_kernel(DenseDev ix, DenseTcArgs a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    double* s = reinterpret_cast<double*>(smem_raw);
    uint64_t* id = reinterpret_cast<uint64_t*>(smem_raw + sizeof(double) * kRsCap);
    __shared__ uint32_t n_sh;
    __shared__ double L_sh;
    const uint32_t q = blockIdx.x, k = a.k, dim = ix.dim;
    const float* qv = a.q + static_cast<uint64_t>(q) * dim;
    auto exact = [&](uint32_t row) {
        const float* r = ix.E + static_cast<uint64_t>(row) * dim;
        double acc = 0.0;
        for (uint32_t j = 0; j < dim; ++j) acc = __fma_rn(static_cast<double>(__ldg(r + j)), static_cast<double>(qv[j]), acc);
        return acc;
    };
    auto sort_n = [&](uint32_t n) {  // bitonic over pow2 >= n, padded with -inf
        uint32_t n2 = 1;
        while (n2 < n) n2 <<= 1;
        for (uint32_t i = n + threadIdx.x; i < n2; i += kRsThreads) {
            s[i] = -__longlong_as_double(0x7ff0000000000000ll);
            id[i] = ~0ull;
        }
        __syncthreads();
        for (uint32_t size = 2; size <= n2; size <<= 1)
            for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                for (uint32_t t = threadIdx.x; t < n2 / 2; t += kRsThreads) {
                    const uint32_t i = 2 * t - (t & (stride - 1)), j = i + stride;
                    const double si = s[i], sj = s[j];
                    const uint64_t ii = id[i], ij = id[j];
                    if ((i & size) == 0 ? better(sj, ij, si, ii) : better(si, ii, sj, ij)) {
                        s[i] = sj;
                        s[j] = si;
                        id[i] = ij;
                        id[j] = ii;
                    }
                }
                __syncthreads();
            }
    };
    const uint32_t nc = a.cand_n[q];
    if (nc <= a.cand_cap && nc <= static_cast<uint32_t>(kRsCap)) {
        for (uint32_t i = threadIdx.x; i < nc; i += kRsThreads) {
            const uint32_t row = a.cand_rows[static_cast<uint64_t>(q) * a.cand_cap + i];
            s[i] = exact(row);
            id[i] = __ldg(ix.ids + row);
        }
        __syncthreads();
        sort_n(nc);
    } else {
        // overflow: every row, a running best list of 2048 (k <= 32 here)
        if (threadIdx.x == 0) {
            n_sh = 0;
            L_sh = -__longlong_as_double(0x7ff0000000000000ll);
        }
        __syncthreads();
        for (uint32_t r0 = 0; r0 < ix.n; r0 += kRsThreads) {
            const uint32_t row = r0 + threadIdx.x;
            if (row < ix.n) {
                const double x = exact(row);
                if (x >= L_sh) {
                    const uint32_t p = atomicAdd(&n_sh, 1u);
                    s[p] = x;
                    id[p] = __ldg(ix.ids + row);
                }
            }
            __syncthreads();
            if (n_sh + kRsThreads > static_cast<uint32_t>(kRsCap) || r0 + kRsThreads >= ix.n) {
                const uint32_t n = n_sh;
                sort_n(n);
                if (threadIdx.x == 0) {
                    n_sh = min(n, k);
                    if (n >= k) L_sh = s[k - 1];
                }
                __syncthreads();
            }
        }
    }
    const uint32_t n_out = min(nc <= a.cand_cap && nc <= static_cast<uint32_t>(kRsCap) ? nc : n_sh, k);
    for (uint32_t i = threadIdx.x; i < n_out; i += kRsThreads) {
        a.out_ids[static_cast<uint64_t>(q) * k + i] = id[i];
        a.out_scores[static_cast<uint64_t>(q) * k + i] = s[i];
    }
    if (threadIdx.x == 0) a.out_n[q] = n_out;
}

template <int KT>
cudaError_t launch_tc(const CUtensorMap& mq, const CUtensorMap& me, const DenseTcArgs& a, int grid, cudaStream_t st) {
    const size_t smem = sizeof(TcSmem) + 1024;
    cudaError_t e = cudaFuncSetAttribute(dense_tc_kernel<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    dense_tc_kernel<KT><<<grid, kTcThreads, smem, st>>>(mq, me, a);
    return cudaGetLastError();
}

}  // namespace

uint32_t dense_tc_max_k() { return 32; }
uint32_t dense_tc_tile_rows() { return kTcN; }

cudaError_t launch_dense_tc(const DenseDev& ix, const void* map_q, const void* map_e, const DenseTcArgs& a, int sms,
                            cudaStream_t st) {
    if (a.nq == 0) return cudaSuccess;
    const CUtensorMap& mq = *static_cast<const CUtensorMap*>(map_q);
    const CUtensorMap& me = *static_cast<const CUtensorMap*>(map_e);
    const uint32_t n_qt = (a.nq + kTcM - 1) / kTcM;
    const uint32_t items = n_qt * a.n_slabs;
    const int grid = static_cast<int>(items < static_cast<uint32_t>(sms) ? items : static_cast<uint32_t>(sms));
    cudaError_t e = a.k <= 16 ? launch_tc<16>(mq, me, a, grid, st) : launch_tc<32>(mq, me, a, grid, st);
    if (e != cudaSuccess) return e;
    const size_t rs_smem = (sizeof(double) + sizeof(uint64_t)) * kRsCap;
    e = cudaFuncSetAttribute(dense_rescore_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(rs_smem));
    if (e != cudaSuccess) return e;
    dense_rescore_kernel<<<a.nq, kRsThreads, rs_smem, st>>>(ix, a);
    return cudaGetLastError();
}

uint32_t dense_tc_slabs(uint32_t nq, uint32_t n_rows, int sms) {
    const uint32_t n_qt = (nq + kTcM - 1) / kTcM;
    const uint32_t n_tiles = (n_rows + kTcN - 1) / kTcN;
    uint32_t s = static_cast<uint32_t>(sms) / n_qt;
    // every slab starts its own bound (~k first-tile candidates each): keep
    // slabs long enough that the bound, not the start-up, dominates
    s = s > n_tiles / 64 ? n_tiles / 64 : s;
    s = s < 1 ? 1 : s;
    return s > n_tiles ? (n_tiles ? n_tiles : 1) : s;
}

}  // namespace hm
