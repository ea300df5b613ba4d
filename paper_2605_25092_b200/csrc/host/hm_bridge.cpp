// C-ABI of the learned-sparse bridge path (include/hm_b200.h, hm_bridge_*):
// upload of a Bridge-mode CsrIndex and batch top-k on kernels/bridge.cu.
//
// The device copy keeps the reference's layout (term_offsets u64, rows u32,
// weights f64: 12 B per posting) because the scores must be the reference's
// fp64 bits (src/bridge.cpp:127): there is no (tf, len) structure to compress.
// Search is one persistent kernel per batch; no CPU scoring path exists.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "hm_b200.h"
#include "hm_bridge.h"
#include "hm_host.h"
#include "hm_launch.h"

using hm_host::ck;
using hm_host::guard;

namespace {

thread_local float g_ms_bridge = 0.f;

// device buffers + stream of one in-flight batch
struct BridgeWs {
    cudaStream_t st = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    uint32_t nq_cap = 0, k_cap = 0;
    uint64_t nnz_cap = 0, scratch_cap = 0;
    uint64_t *q_off = nullptr, *out_ids = nullptr, *out_post = nullptr, *scratch = nullptr;
    uint32_t *q_idx = nullptr, *out_n = nullptr, *counters = nullptr;
    double *q_val = nullptr, *out_scores = nullptr;
    // slab-query results of a split batch (merged into the final outputs)
    uint64_t *v_ids = nullptr, *v_post = nullptr;
    double* v_scores = nullptr;
    uint32_t* v_n = nullptr;
    uint64_t v_cap = 0, vk_cap = 0;

    BridgeWs() {
        ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "bridge stream");
        ck(cudaEventCreate(&ev[0]), "event");
        ck(cudaEventCreate(&ev[1]), "event");
        ck(cudaMalloc(&counters, 4 * sizeof(uint32_t)), "cudaMalloc(counters)");
    }
    ~BridgeWs() {
        void* ps[] = {q_off, out_ids, out_post, scratch, q_idx, out_n, counters, q_val, out_scores,
                      v_ids, v_post, v_scores, v_n};
        for (void* p : ps)
            if (p) cudaFree(p);
        cudaEventDestroy(ev[0]);
        cudaEventDestroy(ev[1]);
        cudaStreamDestroy(st);
    }
    template <typename T>
    static void grow(T*& p, uint64_t n) {
        if (p) cudaFree(p);
        p = nullptr;
        ck(cudaMalloc(&p, std::max<uint64_t>(n, 1) * sizeof(T)), "cudaMalloc(bridge workspace)");
    }
    void ensure_slabs(uint64_t nv, uint32_t k) {
        if (nv <= v_cap && k <= vk_cap) return;
        const uint64_t NV = std::max(nv, v_cap), K = std::max<uint64_t>(k, vk_cap);
        grow(v_ids, NV * K);
        grow(v_scores, NV * K);
        grow(v_n, NV);
        grow(v_post, NV);
        v_cap = NV;
        vk_cap = K;
    }
    void ensure(uint32_t nq, uint64_t nnz, uint32_t k, uint64_t scratch_words) {
        if (nq > nq_cap || k > k_cap) {
            const uint32_t NQ = std::max(nq, nq_cap), K = std::max(std::max(k, k_cap), 1u);
            grow(q_off, NQ + 1ull);
            grow(out_n, NQ);
            grow(out_post, NQ);
            grow(out_ids, static_cast<uint64_t>(NQ) * K);
            grow(out_scores, static_cast<uint64_t>(NQ) * K);
            nq_cap = NQ;
            k_cap = K;
        }
        if (nnz > nnz_cap) {
            grow(q_idx, nnz);
            grow(q_val, nnz);
            nnz_cap = nnz;
        }
        if (scratch_words > scratch_cap) {
            grow(scratch, scratch_words);
            scratch_cap = scratch_words;
        }
    }
};

}  // namespace

struct hm_bridge {
    int device = 0;
    int sms = 0;
    hm::BridgeDev dev{};
    std::vector<void*> allocs;
    uint64_t bytes = 0;
    std::mutex mu;
    std::vector<BridgeWs*> pool;

    ~hm_bridge() {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        for (auto* w : pool) delete w;
        for (void* p : allocs) cudaFree(p);
        cudaSetDevice(prev);
    }
    BridgeWs* acquire() {
        std::lock_guard<std::mutex> lk(mu);
        if (!pool.empty()) {
            BridgeWs* w = pool.back();
            pool.pop_back();
            return w;
        }
        return new BridgeWs();
    }
    void release(BridgeWs* w) {
        std::lock_guard<std::mutex> lk(mu);
        pool.push_back(w);
    }
};

namespace {

template <typename T>
const T* upload(hm_bridge* X, const T* host, uint64_t n) {
    void* p = nullptr;
    const uint64_t sz = std::max<uint64_t>(n, 1) * sizeof(T);
    ck(cudaMalloc(&p, sz), "cudaMalloc(bridge index)");
    X->allocs.push_back(p);
    X->bytes += sz;
    if (n) ck(cudaMemcpy(p, host, n * sizeof(T), cudaMemcpyHostToDevice), "cudaMemcpy(bridge index)");
    return static_cast<const T*>(p);
}

// The CsrIndex invariants the kernel relies on (csr_index.hpp:50-60).
void check_view(const hm_bridge_view* v) {
    if (!v->term_offsets) throw std::invalid_argument("term_offsets is required");
    const uint64_t P = v->term_offsets[v->n_terms];
    if ((P && (!v->posting_rows || !v->posting_weights)) || (v->n_docs && !v->doc_ids))
        throw std::invalid_argument("null index array");
    if (v->term_offsets[0] != 0) throw std::invalid_argument("term_offsets[0] must be 0");
    for (uint32_t t = 0; t < v->n_terms; ++t) {
        const uint64_t b = v->term_offsets[t], e = v->term_offsets[t + 1];
        if (e < b) throw std::invalid_argument("term_offsets not monotone");
        for (uint64_t i = b; i < e; ++i) {
            if (v->posting_rows[i] >= v->n_docs) throw std::invalid_argument("posting row out of range");
            if (i > b && v->posting_rows[i] <= v->posting_rows[i - 1])
                throw std::invalid_argument("posting rows must be strictly increasing per term");
        }
    }
}

// SparseVector::validate (src/bridge.cpp:10-20), same messages
void validate_queries(const hm_bridge_batch* b, uint32_t* max_nnz) {
    uint32_t mx = 0;
    for (uint32_t q = 0; q < b->n_queries; ++q) {
        const uint64_t o0 = b->q_off[q], o1 = b->q_off[q + 1];
        if (o1 < o0) throw std::invalid_argument("q_off not monotone");
        for (uint64_t i = o0; i < o1; ++i) {
            if (i > o0 && b->q_idx[i] <= b->q_idx[i - 1])
                throw std::invalid_argument("sparse vector indices must be strictly increasing");
            if (!(b->q_val[i] > 0.0)) throw std::invalid_argument("sparse vector values must be > 0");
        }
        mx = std::max<uint32_t>(mx, static_cast<uint32_t>(o1 - o0));
    }
    *max_nnz = mx;
}

hm::BridgeArgs make_args(const hm_bridge* X, const hm_bridge_batch* b, BridgeWs* w, uint32_t m_max) {
    hm::BridgeArgs a{};
    a.nq = b->n_queries;
    a.k = b->k;
    a.row_lo = b->row_lo;
    a.row_hi = b->row_hi == 0 ? X->dev.n_docs : std::min(b->row_hi, X->dev.n_docs);
    a.m_max = std::max(m_max, 1u);
    a.scratch = w->scratch;
    a.counters = w->counters;
    return a;
}

uint64_t scratch_words(const hm_bridge* X, uint32_t k, uint32_t m_max) {
    return static_cast<uint64_t>(hm::bridge_grid(k, X->sms)) * (3 + 2 * 8) * std::max(m_max, 1u);
}

// Small batches: each query split into row slabs (the BM25 path's policy,
// hm_index.cpp split_for): slab queries in one launch, merged like doc shards.
uint32_t bridge_split(const hm_bridge* X, const hm::BridgeArgs& a, uint32_t flags) {
    if ((flags & HM_FLAG_NO_SPLIT) || a.k == 0 || a.nq == 0) return 1;
    const uint64_t resident = hm::bridge_grid(a.k, X->sms);
    const uint64_t target = a.nq < 32 ? resident : a.nq < 256 ? 4 * resident : 8 * resident;
    const uint32_t span = a.row_hi > a.row_lo ? a.row_hi - a.row_lo : 0;
    uint64_t S = std::min<uint64_t>(target / a.nq, 64);
    S = std::min<uint64_t>(S, 2048 / a.k);  // merge_kernel holds split x k candidates
    S = std::min<uint64_t>(S, span / 8192);  // >= one 1,024-row unit per warp
    return S >= 2 ? static_cast<uint32_t>(S) : 1;
}

// one batch: a.out_* are the final outputs; split batches write slab results
// to the workspace and merge them there
void run(hm_bridge* X, hm::BridgeArgs a, BridgeWs* w, cudaStream_t st, bool timing, uint32_t flags) {
    const uint32_t nq = a.nq, split = bridge_split(X, a, flags);
    uint64_t* fin_ids = a.out_ids;
    double* fin_scores = a.out_scores;
    uint32_t* fin_n = a.out_n;
    uint64_t* fin_post = a.out_post;
    if (split > 1) {
        w->ensure_slabs(static_cast<uint64_t>(nq) * split, a.k);
        a.nq = nq * split;
        a.split = split;
        a.nq_real = nq;
        a.out_ids = w->v_ids;
        a.out_scores = w->v_scores;
        a.out_n = w->v_n;
        a.out_post = w->v_post;
    }
    ck(cudaMemsetAsync(w->counters, 0, 4 * sizeof(uint32_t), st), "memset counters");
    if (timing) ck(cudaEventRecord(w->ev[0], st), "event");
    ck(hm::launch_bridge(X->dev, a, X->sms, st), "bridge kernel");
    if (split > 1) {
        ck(hm::launch_merge(split, nq, a.k, w->v_ids, w->v_scores, w->v_n, nullptr, 0.0, 1e-9, fin_ids, fin_scores,
                            fin_n, nullptr, nullptr, st),
           "slab merge");
        ck(hm::launch_sum_slab_postings(nq, split, w->v_post, fin_post, st), "slab postings");
    }
    if (timing) ck(cudaEventRecord(w->ev[1], st), "event");
}

}  // namespace

extern "C" {

int hm_bridge_create(const hm_bridge_view* view, int device, hm_bridge** out) {
    return guard([&] {
        if (!view || !out) throw std::invalid_argument("null argument");
        check_view(view);
        hm_host::use_device(device);
        auto* X = new hm_bridge();
        try {
            X->device = device;
            cudaDeviceProp prop{};
            ck(cudaGetDeviceProperties(&prop, device), "device properties");
            X->sms = prop.multiProcessorCount;
            const uint64_t P = view->term_offsets[view->n_terms];
            X->dev.term_off = upload(X, view->term_offsets, view->n_terms + 1ull);
            X->dev.rows = upload(X, view->posting_rows, P);
            X->dev.w = upload(X, view->posting_weights, P);
            X->dev.doc_ids = upload(X, view->doc_ids, view->n_docs);
            X->dev.n_terms = view->n_terms;
            X->dev.n_docs = view->n_docs;
        } catch (...) {
            delete X;
            throw;
        }
        *out = X;
    });
}

int hm_bridge_destroy(hm_bridge* bridge) {
    return guard([&] { delete bridge; });
}

int hm_bridge_search_batch(hm_bridge* X, const hm_bridge_batch* b, hm_results* out) {
    return guard([&] {
        if (!X || !b || !out) throw std::invalid_argument("null argument");
        const uint32_t nq = b->n_queries;
        if (nq == 0) return;
        if (!b->q_off || !out->ids || !out->scores || !out->n) throw std::invalid_argument("null batch buffer");
        const uint64_t nnz = b->q_off[nq];
        if (nnz && (!b->q_idx || !b->q_val)) throw std::invalid_argument("q_idx and q_val are required");
        if (b->k > hm::bridge_max_k())
            throw std::invalid_argument("k exceeds the supported maximum of " + std::to_string(hm::bridge_max_k()));
        uint32_t m_max = 0;
        validate_queries(b, &m_max);
        ck(cudaSetDevice(X->device), "cudaSetDevice");
        BridgeWs* w = X->acquire();
        try {
            const uint32_t kk = std::max(b->k, 1u);
            w->ensure(nq, nnz, kk, scratch_words(X, b->k, m_max));
            cudaStream_t st = w->st;
            ck(cudaMemcpyAsync(w->q_off, b->q_off, (nq + 1ull) * 8, cudaMemcpyHostToDevice, st), "H2D q_off");
            if (nnz) {
                ck(cudaMemcpyAsync(w->q_idx, b->q_idx, nnz * 4, cudaMemcpyHostToDevice, st), "H2D q_idx");
                ck(cudaMemcpyAsync(w->q_val, b->q_val, nnz * 8, cudaMemcpyHostToDevice, st), "H2D q_val");
            }
            hm::BridgeArgs a = make_args(X, b, w, m_max);
            a.q_off = w->q_off;
            a.q_idx = w->q_idx;
            a.q_val = w->q_val;
            a.out_ids = w->out_ids;
            a.out_scores = w->out_scores;
            a.out_n = w->out_n;
            a.out_post = w->out_post;
            // row stride of the results is k (the caller's layout)
            const bool timing = (b->flags & HM_FLAG_TIMING) != 0;
            run(X, a, w, st, timing, b->flags);
            if (b->k) {
                ck(cudaMemcpyAsync(out->ids, w->out_ids, static_cast<uint64_t>(nq) * b->k * 8, cudaMemcpyDeviceToHost, st),
                   "D2H ids");
                ck(cudaMemcpyAsync(out->scores, w->out_scores, static_cast<uint64_t>(nq) * b->k * 8,
                                   cudaMemcpyDeviceToHost, st),
                   "D2H scores");
            }
            ck(cudaMemcpyAsync(out->n, w->out_n, nq * 4ull, cudaMemcpyDeviceToHost, st), "D2H n");
            if (out->postings)
                ck(cudaMemcpyAsync(out->postings, w->out_post, nq * 8ull, cudaMemcpyDeviceToHost, st), "D2H postings");
            ck(cudaStreamSynchronize(st), "bridge sync");
            if (timing) ck(cudaEventElapsedTime(&g_ms_bridge, w->ev[0], w->ev[1]), "elapsed");
        } catch (...) {
            X->release(w);
            throw;
        }
        X->release(w);
    });
}

int hm_bridge_search_batch_device(hm_bridge* X, const hm_bridge_batch* b, hm_results* out, void* stream) {
    return guard([&] {
        if (!X || !b || !out) throw std::invalid_argument("null argument");
        const uint32_t nq = b->n_queries;
        if (nq == 0) return;
        if (!b->q_off || !out->ids || !out->scores || !out->n) throw std::invalid_argument("null batch buffer");
        if (b->k > hm::bridge_max_k())
            throw std::invalid_argument("k exceeds the supported maximum of " + std::to_string(hm::bridge_max_k()));
        if (b->max_nnz == 0) throw std::invalid_argument("max_nnz is required for device batches");
        ck(cudaSetDevice(X->device), "cudaSetDevice");
        BridgeWs* w = X->acquire();
        try {
            w->ensure(0, 0, 0, scratch_words(X, b->k, b->max_nnz));
            cudaStream_t st = static_cast<cudaStream_t>(stream);
            hm::BridgeArgs a = make_args(X, b, w, b->max_nnz);
            a.q_off = b->q_off;
            a.q_idx = b->q_idx;
            a.q_val = b->q_val;
            a.out_ids = out->ids;
            a.out_scores = out->scores;
            a.out_n = out->n;
            a.out_post = out->postings;
            const bool timing = (b->flags & HM_FLAG_TIMING) != 0;
            run(X, a, w, st, timing, b->flags);
            // the workspace (scratch, counters) is reusable once the kernel ends
            ck(cudaStreamSynchronize(st), "bridge sync");
            if (timing) ck(cudaEventElapsedTime(&g_ms_bridge, w->ev[0], w->ev[1]), "elapsed");
        } catch (...) {
            X->release(w);
            throw;
        }
        X->release(w);
    });
}

int hm_bridge_last_timing(float* ms_kernel) {
    if (ms_kernel) *ms_kernel = g_ms_bridge;
    return HM_OK;
}

}  // extern "C"
