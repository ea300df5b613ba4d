// Probes of one plan term for given rows (the seeded MaxScore pass and the
// essential-term sweep): the term's contribution in the selection-score
// domain (score * 2^-61) from the dense per-row code array, the term's
// 1,024-row sub-tile range (long terms) or its tile segment (short terms).
#pragma once
#include "search_common.cuh"

namespace hm {

template <class Sm>
struct ProbeCtx {
    const DevIndex& ix;
    const BatchArgs& a;
    Sm& S;
    const uint32_t* stab;
    uint32_t stride, j0, cb;
    double k1, b;
};

// impact of a (tf, len) code: the first kShortCodes from shared memory
template <class Sm>
__device__ __forceinline__ float code_w(const ProbeCtx<Sm>& c, uint32_t code) {
    return code < static_cast<uint32_t>(kShortCodes) ? c.S.w32s[code] : __ldg(c.a.w32 + code);
}

// Contribution of plan term i (selection-score domain: score * 2^-61) to a row.
template <class Sm>
__device__ __noinline__ float seed_probe(const ProbeCtx<Sm>& c, uint32_t i, uint32_t row) {
    const DevIndex& ix = c.ix;
    const int32_t slot = c.S.t_slot[i];
    float w;
    if (slot >= 0) {
        const int32_t d = c.S.t_dense[i];
        if (d >= 0) {
            const uint16_t code = __ldg(ix.dense + static_cast<uint64_t>(d) * ix.n_docs + row);
            if (code == kDenseAbsent) return 0.f;
            if (code != kDenseEscape) return c.S.t_cu[i] * code_w(c, code);
        }
        const uint32_t* tb = tile_row(ix, slot);
        const uint32_t sub = row >> kSubShift;
        const uint64_t s0 = c.S.t_start[i];
        const uint64_t lo = s0 + __ldg(tb + sub), hi = s0 + __ldg(tb + sub + 1);
        const uint32_t local = row & (kTile - 1);
        const uint64_t pos = lower_bound_packed(ix.post, lo, hi, local << kCodeBitsLong);
        if (pos >= hi) return 0.f;
        const uint32_t p = __ldg(ix.post + pos);
        if ((p >> kCodeBitsLong) != local) return 0.f;
        const uint32_t code = p & kEscLong;
        w = code < ix.n_codes ? code_w(c, code)
                              : impact32(static_cast<double>(__ldg(ix.tf + pos)),
                                         static_cast<double>(__ldg(ix.doc_lens + row)), ix.avgdl, c.k1, c.b);
    } else {
        const uint32_t* tab = c.stab + static_cast<uint64_t>(c.S.t_spos[i]) * c.stride;
        const uint32_t jj = (row >> kTileShift) - c.j0;
        const uint64_t s0 = c.S.t_start[i];
        const uint64_t lo = s0 + tab[jj], hi = s0 + tab[jj + 1];
        const uint64_t pos = lower_bound_row(ix.post, lo, hi, row, c.cb);
        if (pos >= hi) return 0.f;
        const uint32_t p = __ldg(ix.post + pos);
        if ((p >> c.cb) != row) return 0.f;
        const uint32_t code = p & ix.esc_short;
        w = code < ix.n_codes_short ? c.S.w32s[code]
                                    : impact32(static_cast<double>(__ldg(ix.tf + pos)),
                                               static_cast<double>(__ldg(ix.doc_lens + row)), ix.avgdl, c.k1, c.b);
    }
    return c.S.t_cu[i] * w;
}

// seed_probe for N rows at once (rows whose bit is clear in vmask are not
// needed): all N dense loads / range loads / search steps are in flight
// together.  Escaped dense codes (rare) fall back to the scalar probe.
template <int N>
struct RowsN {
    uint32_t r[N];
};
template <int N>
struct ValsN {
    float v[N];
};
template <class Sm, int N>  // vmask != 0
__device__ __noinline__ ValsN<N> seed_probeN(const ProbeCtx<Sm>& c, uint32_t i, RowsN<N> rw, uint32_t vmask) {
    const DevIndex& ix = c.ix;
    const int32_t slot = c.S.t_slot[i];
    const float cu = c.S.t_cu[i];
    ValsN<N> out;
    // rows not needed take a needed row's value (every probe stays in the window)
    const uint32_t fill = rw.r[__ffs(vmask) - 1];
#pragma unroll
    for (int u = 0; u < N; ++u)
        if (!((vmask >> u) & 1u)) rw.r[u] = fill;
    if (slot >= 0) {
        const int32_t d = c.S.t_dense[i];
        if (d >= 0) {
            const uint16_t* col = ix.dense + static_cast<uint64_t>(d) * ix.n_docs;
            uint16_t code[N];
#pragma unroll
            for (int u = 0; u < N; ++u) code[u] = __ldg(col + rw.r[u]);
#pragma unroll
            for (int u = 0; u < N; ++u)
                out.v[u] = code[u] == kDenseAbsent ? 0.f
                           : code[u] == kDenseEscape ? seed_probe(c, i, rw.r[u])
                                                     : cu * code_w(c, code[u]);
            return out;
        }
        const uint32_t* tb = tile_row(ix, slot);
        const uint64_t s0 = c.S.t_start[i];
        uint64_t lo[N], hi[N], end[N];
#pragma unroll
        for (int u = 0; u < N; ++u) {
            lo[u] = s0 + __ldg(tb + (rw.r[u] >> kSubShift));
            hi[u] = s0 + __ldg(tb + (rw.r[u] >> kSubShift) + 1);
            end[u] = hi[u];
        }
        for (;;) {
            bool any = false;
            uint32_t p[N];
#pragma unroll
            for (int u = 0; u < N; ++u) {
                const uint64_t mid = lo[u] + ((hi[u] - lo[u]) >> 1);
                p[u] = lo[u] < hi[u] ? __ldg(ix.post + mid) : 0u;
            }
#pragma unroll
            for (int u = 0; u < N; ++u) {
                if (lo[u] < hi[u]) {
                    const uint64_t mid = lo[u] + ((hi[u] - lo[u]) >> 1);
                    if ((p[u] >> kCodeBitsLong) < (rw.r[u] & (kTile - 1))) lo[u] = mid + 1;
                    else hi[u] = mid;
                }
                any |= lo[u] < hi[u];
            }
            if (!any) break;
        }
#pragma unroll
        for (int u = 0; u < N; ++u) {
            float w = 0.f;
            if (lo[u] < end[u]) {
                const uint32_t pp = __ldg(ix.post + lo[u]);
                if ((pp >> kCodeBitsLong) == (rw.r[u] & (kTile - 1))) {
                    const uint32_t code = pp & kEscLong;
                    w = code < ix.n_codes ? code_w(c, code)
                                          : impact32(static_cast<double>(__ldg(ix.tf + lo[u])),
                                                     static_cast<double>(__ldg(ix.doc_lens + rw.r[u])), ix.avgdl,
                                                     c.k1, c.b);
                }
            }
            out.v[u] = cu * w;
        }
        return out;
    }
    const uint32_t* tab = c.stab + static_cast<uint64_t>(c.S.t_spos[i]) * c.stride;
    const uint64_t s0 = c.S.t_start[i];
    const uint32_t cb = c.cb;
    uint64_t lo[N], hi[N], end[N];
#pragma unroll
    for (int u = 0; u < N; ++u) {
        const uint32_t jj = (rw.r[u] >> kTileShift) - c.j0;
        lo[u] = s0 + tab[jj];
        hi[u] = s0 + tab[jj + 1];
        end[u] = hi[u];
    }
    for (;;) {
        bool any = false;
        uint32_t p[N];
#pragma unroll
        for (int u = 0; u < N; ++u) {
            const uint64_t mid = lo[u] + ((hi[u] - lo[u]) >> 1);
            p[u] = lo[u] < hi[u] ? __ldg(ix.post + mid) : 0u;
        }
#pragma unroll
        for (int u = 0; u < N; ++u) {
            if (lo[u] < hi[u]) {
                const uint64_t mid = lo[u] + ((hi[u] - lo[u]) >> 1);
                if ((p[u] >> cb) < rw.r[u]) lo[u] = mid + 1;
                else hi[u] = mid;
            }
            any |= lo[u] < hi[u];
        }
        if (!any) break;
    }
#pragma unroll
    for (int u = 0; u < N; ++u) {
        float w = 0.f;
        if (lo[u] < end[u]) {
            const uint32_t pp = __ldg(ix.post + lo[u]);
            if ((pp >> cb) == rw.r[u]) {
                const uint32_t code = pp & ix.esc_short;
                w = code < ix.n_codes_short ? c.S.w32s[code]
                                            : impact32(static_cast<double>(__ldg(ix.tf + lo[u])),
                                                       static_cast<double>(__ldg(ix.doc_lens + rw.r[u])), ix.avgdl,
                                                       c.k1, c.b);
            }
        }
        out.v[u] = cu * w;
    }
    return out;
}

}  // namespace hm
