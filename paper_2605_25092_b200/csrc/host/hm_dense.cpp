// C-ABI of the dense escalate channel (include/hm_b200.h, hm_dense_*):
// upload of an EmbeddingMatrix and batched exact inner-product top-k on
// kernels/dense.cu.  The matrix stays in the reference's layout (row-major
// fp32, src/dense.cpp / include/hybrid/dense.hpp:13-22); no CPU scoring path.
#include <algorithm>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <cmath>

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include "hm_b200.h"
#include "hm_dense.h"
#include "hm_host.h"

using hm_host::ck;
using hm_host::guard;

namespace {

thread_local float g_ms_dense = 0.f;
thread_local uint32_t g_dense_overflow = 0;
thread_local uint64_t g_dense_candidates = 0;
thread_local uint32_t g_dense_path = 0;  // 1 tensor cores, 2 fp64 lists, 3 fp64 sort (large k)
constexpr uint32_t kCandCap = 8192;  // tensor-core path: candidates per query (= rescoring capacity)
constexpr uint32_t kTcChunk = 16384;  // queries per tensor-core launch (candidate lists: 512 MB)

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled is unavailable");
    return fn;
}

// fp32 [rows x dim] row-major as a 2-D TMA map: 32-element (128 B) K boxes,
// box_rows rows, 128-byte swizzle (the UMMA K-major SW128 layout)
void encode_map(CUtensorMap* m, const float* ptr, uint32_t rows, uint32_t dim, uint32_t box_rows) {
    const cuuint64_t gdim[2] = {dim, rows};
    const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(dim) * 4};
    const cuuint32_t box[2] = {32, box_rows};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(ptr), gdim, gstride, box,
                                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(r));
}

struct DenseWs {
    cudaStream_t st = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    uint64_t q_cap = 0, part_cap = 0, lists_cap = 0, out_cap = 0, nq_cap = 0, big_cap = 0, cand_cap = 0;
    uint32_t *cand_n = nullptr, *cand_rows = nullptr;
    int* thr_key = nullptr;
    void* big = nullptr;  // large-k scratch (scores, sort keys, CUB temp)
    float* q_in = nullptr;
    double *q64 = nullptr, *part_scores = nullptr, *out_scores = nullptr;
    uint64_t *part_ids = nullptr, *out_ids = nullptr;
    uint32_t *part_n = nullptr, *out_n = nullptr;

    DenseWs() {
        ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "dense stream");
        ck(cudaEventCreate(&ev[0]), "event");
        ck(cudaEventCreate(&ev[1]), "event");
    }
    ~DenseWs() {
        void* ps[] = {q_in, q64, part_scores, out_scores, part_ids, out_ids, part_n, out_n, big, cand_n, cand_rows,
                      thr_key};
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
        ck(cudaMalloc(&p, std::max<uint64_t>(n, 1) * sizeof(T)), "cudaMalloc(dense workspace)");
    }
    void ensure(uint64_t q_el, uint64_t part_el, uint64_t part_lists, uint64_t out_el, uint64_t nq) {
        if (q_el > q_cap) {
            grow(q_in, q_el);
            grow(q64, q_el);
            q_cap = q_el;
        }
        if (part_el > part_cap) {
            grow(part_scores, part_el);
            grow(part_ids, part_el);
            part_cap = part_el;
        }
        if (part_lists > lists_cap) {
            grow(part_n, part_lists);
            lists_cap = part_lists;
        }
        if (out_el > out_cap) {
            grow(out_scores, out_el);
            grow(out_ids, out_el);
            out_cap = out_el;
        }
        if (nq > nq_cap) {
            grow(out_n, nq);
            nq_cap = nq;
        }
    }
};

}  // namespace

struct hm_dense {
    int device = 0, sms = 0;
    hm::DenseDev dev{};
    bool tc = false;            // dim % 32 == 0: the tensor-core candidate path applies
    alignas(64) CUtensorMap map_e{};
    float err_scale = 0.f;      // TF32 selection bound per unit ||q|| (dense_tc.cu)
    std::vector<void*> allocs;
    std::mutex mu;
    std::vector<DenseWs*> pool;

    ~hm_dense() {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        for (auto* w : pool) delete w;
        for (void* p : allocs) cudaFree(p);
        cudaSetDevice(prev);
    }
    DenseWs* acquire() {
        std::lock_guard<std::mutex> lk(mu);
        if (!pool.empty()) {
            DenseWs* w = pool.back();
            pool.pop_back();
            return w;
        }
        return new DenseWs();
    }
    void release(DenseWs* w) {
        std::lock_guard<std::mutex> lk(mu);
        pool.push_back(w);
    }
};

namespace {

template <typename T>
const T* upload(hm_dense* X, const T* host, uint64_t n) {
    void* p = nullptr;
    ck(cudaMalloc(&p, std::max<uint64_t>(n, 1) * sizeof(T)), "cudaMalloc(embeddings)");
    X->allocs.push_back(p);
    if (n) ck(cudaMemcpy(p, host, n * sizeof(T), cudaMemcpyHostToDevice), "cudaMemcpy(embeddings)");
    return static_cast<const T*>(p);
}

void check_batch(const hm_dense* X, const hm_dense_batch* b) {
    if (b->dim != X->dev.dim) throw std::invalid_argument("query dimension mismatch");  // dense.cpp:88-89
}

// one batch on the workspace's device buffers (queries already in w->q_in
// or at q_dev); results into w->out_* or the caller's device buffers
void run(hm_dense* X, DenseWs* w, uint32_t nq, uint32_t k, const float* q_dev, uint64_t* out_ids, double* out_scores,
         uint32_t* out_n, cudaStream_t st, bool timing, uint32_t flags) {
    if (timing) ck(cudaEventRecord(w->ev[0], st), "event");
    if (X->tc && k <= hm::dense_tc_max_k() && !(flags & HM_FLAG_FORCE_EXACT)) {
        // tensor cores select candidates (TF32), fp64 rescoring decides; the
        // candidate lists (8,192 rows per query) bound a launch to kTcChunk queries
        const uint32_t chunk = std::min<uint32_t>(nq, kTcChunk);
        if (static_cast<uint64_t>(chunk) > w->cand_cap) {
            DenseWs::grow(w->cand_n, chunk);
            DenseWs::grow(w->cand_rows, static_cast<uint64_t>(chunk) * kCandCap);
            DenseWs::grow(w->thr_key, chunk);
            w->cand_cap = chunk;
        }
        if (timing) {
            g_dense_overflow = 0;
            g_dense_candidates = 0;
        }
        for (uint32_t q0 = 0; q0 < nq; q0 += chunk) {
            const uint32_t nc = std::min(chunk, nq - q0);
            const float* qd = q_dev + static_cast<uint64_t>(q0) * X->dev.dim;
            alignas(64) CUtensorMap map_q{};
            encode_map(&map_q, qd, nc, X->dev.dim, 128);
            ck(cudaMemsetAsync(w->cand_n, 0, nc * 4ull, st), "memset candidates");
            ck(cudaMemsetAsync(w->thr_key, 0x80, nc * 4ull, st), "memset bounds");
            hm::DenseTcArgs a{};
            a.nq = nc;
            a.dim = X->dev.dim;
            a.n_rows = X->dev.n;
            a.k = k;
            a.n_slabs = hm::dense_tc_slabs(nc, X->dev.n, X->sms);
            a.q = qd;
            a.err_scale = X->err_scale;
            a.cand_n = w->cand_n;
            a.thr_key = w->thr_key;
            a.cand_rows = w->cand_rows;
            a.cand_cap = kCandCap;
            a.out_ids = out_ids + static_cast<uint64_t>(q0) * k;
            a.out_scores = out_scores + static_cast<uint64_t>(q0) * k;
            a.out_n = out_n + q0;
            ck(hm::launch_dense_tc(X->dev, &map_q, &X->map_e, a, X->sms, st), "dense tensor-core kernels");
            if (timing) {  // candidate statistics (test / bench evidence of the selection's tightness)
                std::vector<uint32_t> cn(nc);
                ck(cudaMemcpyAsync(cn.data(), w->cand_n, nc * 4ull, cudaMemcpyDeviceToHost, st), "D2H candidates");
                ck(cudaStreamSynchronize(st), "sync");
                for (uint32_t c : cn) {
                    g_dense_candidates += c;
                    g_dense_overflow += c > kCandCap;
                }
            }
        }
        g_dense_path = 1;
    } else if (k > hm::dense_max_k()) {
        // k beyond the shared-memory lists: per query, every row scored and
        // sorted on the device (rare: the reference callers use k = 10)
        const uint32_t kk = std::min<uint32_t>(k, X->dev.n);
        const size_t bytes = hm::dense_large_k_bytes(X->dev.n);
        w->ensure(static_cast<uint64_t>(nq) * X->dev.dim, 0, 0, 0, 0);
        if (bytes > w->big_cap) {
            if (w->big) cudaFree(w->big);
            w->big = nullptr;
            ck(cudaMalloc(&w->big, bytes), "cudaMalloc(dense large-k scratch)");
            w->big_cap = bytes;
        }
        for (uint32_t q = 0; q < nq; ++q) {
            double* q64 = w->q64 + static_cast<uint64_t>(q) * X->dev.dim;
            ck(hm::launch_dense_widen(q_dev + static_cast<uint64_t>(q) * X->dev.dim, q64, X->dev.dim, st), "widen");
            ck(hm::launch_dense_large_k(X->dev, q64, kk, w->big, bytes, out_ids + static_cast<uint64_t>(q) * k,
                                        out_scores + static_cast<uint64_t>(q) * k, out_n + q, st),
               "dense large-k");
        }
        g_dense_path = 3;
    } else {
        hm::DenseArgs a{};
        a.nq = nq;
        a.k = k;
        a.n_slabs = hm::dense_slabs(nq, X->dev.n, X->sms);
        w->ensure(static_cast<uint64_t>(nq) * X->dev.dim, static_cast<uint64_t>(a.n_slabs) * nq * k,
                  static_cast<uint64_t>(a.n_slabs) * nq, 0, 0);
        a.q_in = q_dev;
        a.q64 = w->q64;
        a.part_ids = w->part_ids;
        a.part_scores = w->part_scores;
        a.part_n = w->part_n;
        a.out_ids = out_ids;
        a.out_scores = out_scores;
        a.out_n = out_n;
        ck(hm::launch_dense(X->dev, a, st), "dense kernels");
        g_dense_path = 2;
    }
    if (timing) ck(cudaEventRecord(w->ev[1], st), "event");
}

}  // namespace

extern "C" {

int hm_dense_create(const hm_dense_view* view, int device, hm_dense** out) {
    return guard([&] {
        if (!view || !out) throw std::invalid_argument("null argument");
        if (view->count && (!view->data || !view->doc_ids)) throw std::invalid_argument("null embedding array");
        if (view->count && view->dim == 0) throw std::invalid_argument("embedding dimension must be > 0");
        hm_host::use_device(device);
        auto* X = new hm_dense();
        try {
            X->device = device;
            cudaDeviceProp prop{};
            ck(cudaGetDeviceProperties(&prop, device), "device properties");
            X->sms = prop.multiProcessorCount;
            X->dev.E = upload(X, view->data, static_cast<uint64_t>(view->count) * view->dim);
            X->dev.ids = upload(X, view->doc_ids, view->count);
            X->dev.n = view->count;
            X->dev.dim = view->dim;
            if (view->dim % 32 == 0 && view->count > 0) {
                // selection bound: 1.25 (2^-9 + 2^-20 + dim 2^-22) max_r ||r|| (dense_tc.cu)
                double mx = 0.0;
                for (uint64_t r = 0; r < view->count; ++r) {
                    double s2 = 0.0;
                    const float* row = view->data + r * view->dim;
                    for (uint32_t j = 0; j < view->dim; ++j) s2 += static_cast<double>(row[j]) * row[j];
                    mx = std::max(mx, s2);
                }
                const double c = 1.25 * (std::ldexp(1.0, -9) + std::ldexp(1.0, -20) + view->dim * std::ldexp(1.0, -22));
                X->err_scale = static_cast<float>(c * std::sqrt(mx) * 1.0001);
                encode_map(&X->map_e, X->dev.E, view->count, view->dim, hm::dense_tc_tile_rows());
                X->tc = std::isfinite(X->err_scale);
            }
        } catch (...) {
            delete X;
            throw;
        }
        *out = X;
    });
}

int hm_dense_destroy(hm_dense* dense) {
    return guard([&] { delete dense; });
}

int hm_dense_search_batch(hm_dense* X, const hm_dense_batch* b, hm_results* out) {
    return guard([&] {
        if (!X || !b || !out) throw std::invalid_argument("null argument");
        check_batch(X, b);
        const uint32_t nq = b->n_queries;
        if (nq == 0) return;
        if (!b->queries || !out->n || (b->k && (!out->ids || !out->scores)))
            throw std::invalid_argument("null batch buffer");
        if (b->k == 0 || X->dev.n == 0) {
            std::fill(out->n, out->n + nq, 0u);
            return;
        }
        ck(cudaSetDevice(X->device), "cudaSetDevice");
        DenseWs* w = X->acquire();
        try {
            const uint64_t q_el = static_cast<uint64_t>(nq) * X->dev.dim;
            w->ensure(q_el, 0, 0, static_cast<uint64_t>(nq) * b->k, nq);
            cudaStream_t st = w->st;
            ck(cudaMemcpyAsync(w->q_in, b->queries, q_el * 4, cudaMemcpyHostToDevice, st), "H2D queries");
            const bool timing = (b->flags & HM_FLAG_TIMING) != 0;
            run(X, w, nq, b->k, w->q_in, w->out_ids, w->out_scores, w->out_n, st, timing, b->flags);
            ck(cudaMemcpyAsync(out->ids, w->out_ids, static_cast<uint64_t>(nq) * b->k * 8, cudaMemcpyDeviceToHost, st),
               "D2H ids");
            ck(cudaMemcpyAsync(out->scores, w->out_scores, static_cast<uint64_t>(nq) * b->k * 8,
                               cudaMemcpyDeviceToHost, st),
               "D2H scores");
            ck(cudaMemcpyAsync(out->n, w->out_n, nq * 4ull, cudaMemcpyDeviceToHost, st), "D2H n");
            ck(cudaStreamSynchronize(st), "dense sync");
            if (timing) ck(cudaEventElapsedTime(&g_ms_dense, w->ev[0], w->ev[1]), "elapsed");
        } catch (...) {
            X->release(w);
            throw;
        }
        X->release(w);
    });
}

int hm_dense_search_batch_device(hm_dense* X, const hm_dense_batch* b, hm_results* out, void* stream) {
    return guard([&] {
        if (!X || !b || !out) throw std::invalid_argument("null argument");
        check_batch(X, b);
        const uint32_t nq = b->n_queries;
        if (nq == 0) return;
        if (b->k == 0 || X->dev.n == 0) throw std::invalid_argument("device batches need k > 0 and rows");
        ck(cudaSetDevice(X->device), "cudaSetDevice");
        DenseWs* w = X->acquire();
        try {
            w->ensure(static_cast<uint64_t>(nq) * X->dev.dim, 0, 0, 0, 0);
            cudaStream_t st = static_cast<cudaStream_t>(stream);
            const bool timing = (b->flags & HM_FLAG_TIMING) != 0;
            run(X, w, nq, b->k, b->queries, out->ids, out->scores, out->n, st, timing, b->flags);
            ck(cudaStreamSynchronize(st), "dense sync");  // the workspace is reusable afterwards
            if (timing) ck(cudaEventElapsedTime(&g_ms_dense, w->ev[0], w->ev[1]), "elapsed");
        } catch (...) {
            X->release(w);
            throw;
        }
        X->release(w);
    });
}

int hm_dense_last_timing(float* ms) {
    if (ms) *ms = g_ms_dense;
    return HM_OK;
}

int hm_dense_last_stats(uint32_t* path, uint32_t* n_overflow, uint64_t* n_candidates) {
    if (path) *path = g_dense_path;
    if (n_overflow) *n_overflow = g_dense_overflow;
    if (n_candidates) *n_candidates = g_dense_candidates;
    return HM_OK;
}

}  // extern "C"
