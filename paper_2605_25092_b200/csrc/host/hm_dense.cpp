// C-ABI of the dense escalate channel (include/hm_b200.h, hm_dense_*):
// upload of an EmbeddingMatrix and batched exact inner-product top-k on
// kernels/dense.cu.  The matrix stays in the reference's layout (row-major
// fp32, src/dense.cpp / include/hybrid/dense.hpp:13-22); no CPU scoring path.
#include <algorithm>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "hm_b200.h"
#include "hm_dense.h"
#include "hm_host.h"

using hm_host::ck;
using hm_host::guard;

namespace {

thread_local float g_ms_dense = 0.f;

struct DenseWs {
    cudaStream_t st = nullptr;
    cudaEvent_t ev[2] = {nullptr, nullptr};
    uint64_t q_cap = 0, part_cap = 0, lists_cap = 0, out_cap = 0, nq_cap = 0, big_cap = 0;
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
        void* ps[] = {q_in, q64, part_scores, out_scores, part_ids, out_ids, part_n, out_n, big};
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
         uint32_t* out_n, cudaStream_t st, bool timing) {
    if (timing) ck(cudaEventRecord(w->ev[0], st), "event");
    if (k > hm::dense_max_k()) {
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
            run(X, w, nq, b->k, w->q_in, w->out_ids, w->out_scores, w->out_n, st, timing);
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
            run(X, w, nq, b->k, b->queries, out->ids, out->scores, out->n, st, timing);
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

}  // extern "C"
