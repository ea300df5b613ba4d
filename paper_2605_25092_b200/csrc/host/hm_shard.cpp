// Doc-sharded search behind the C ABI (hm_sharded_*, include/hm_b200.h): one
// process driving several devices, for C++ callers of the reference API
// (the reference defers sharding; its precedent for
// shard-local scoring with global statistics is SharedStats,
// proj/include/hybrid/csr_index.hpp:28-35, used by build_temporal_index,
// proj/src/temporal_index.cpp:136-142).
//
//   * create: rows split into G contiguous ranges; shard g is the sub-CSR of
//     its rows (rows renumbered from 0) with the flat index's idf, order keys
//     and avgdl -- every local score is the flat score bit for bit -- uploaded
//     to devices[g] as an ordinary hm_index.  Peer access root -> g is
//     enabled where the devices allow it (NVLink / NVSwitch).
//   * search: one host thread per shard uploads the batch to its device and
//     runs the single-device launch sequence (hm_search_batch_device) with
//     the window clipped to the shard -- for batches of 256+ queries after an
//     exchange of bounds (every shard's k best seed scores, their k-th largest
//     per query computed on the root: bound_kth_kernel), so each shard prunes
//     against the union's threshold; each
//     leaves its list of the documents that can be in the union's top-k in
//     its own HBM.  The root device then runs gather_merge_kernel
//     (kernels/shard_merge.cu): it reads every shard's lists over peer memory
//     and merges them by rank in the same kernel -- the all-gather and the
//     k-way merge fused, no separate collective.  Shards whose device the
//     root cannot address are copied to the root first (cudaMemcpyPeerAsync).
#include <algorithm>
#include <cstring>
#include <exception>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "hm_b200.h"
#include "hm_host.h"
#include "hm_launch.h"

using hm_host::ck;
using hm_host::guard;

namespace {

// an hm_* status from a call made on a worker thread -> the exception the
// caller's guard maps back to the same status (the message travels with it)
void rethrow_status(int st, const char* what) {
    if (st == HM_OK) return;
    const std::string msg = std::string(hm_last_error());
    switch (st) {
        case HM_ERR_INVALID: throw std::invalid_argument(msg);
        case HM_ERR_RANGE: throw std::out_of_range(msg);
        case HM_ERR_NO_DEVICE: throw hm_host::no_device_error(msg);
        default: throw std::runtime_error(std::string(what) + ": " + msg);
    }
}

// batches from this size on exchange the shards' bounds before the search
constexpr uint32_t kBoundMinQueries = 256;

template <typename T>
void grow(T*& p, uint64_t& cap, uint64_t n) {
    if (n <= cap && p) return;
    if (p) cudaFree(p);
    p = nullptr;
    void* v = nullptr;
    ck(cudaMalloc(&v, std::max<uint64_t>(n, 1) * sizeof(T)), "cudaMalloc(shard buffers)");
    p = static_cast<T*>(v);
    cap = std::max<uint64_t>(n, 1);
}

template <typename F>
void run_parallel(uint32_t n, F&& f) {
    std::vector<std::exception_ptr> err(n);
    auto body = [&](uint32_t g) {
        try {
            f(g);
        } catch (...) {
            err[g] = std::current_exception();
        }
    };
    if (n == 1) {
        body(0);
    } else {
        std::vector<std::thread> th;
        for (uint32_t g = 0; g < n; ++g) th.emplace_back(body, g);
        for (auto& t : th) t.join();
    }
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
}

struct Shard {
    int device = 0;
    uint32_t row0 = 0, row1 = 0;
    hm_index* index = nullptr;
    bool p2p = false;  // the root device addresses this shard's memory directly
    cudaStream_t stream = nullptr;
    uint32_t *q_off = nullptr, *q_tid = nullptr, *n = nullptr;
    uint64_t *ids = nullptr, *post = nullptr;
    double* scores = nullptr;
    float* bound = nullptr;  // [nq][k] this shard's k best seed scores (the bound pass)
    float* ext = nullptr;    // [nq] the union's k-th-score bound
    uint64_t off_cap = 0, tid_cap = 0, n_cap = 0, ids_cap = 0, post_cap = 0, sc_cap = 0, bound_cap = 0, ext_cap = 0;
    float* r_bound = nullptr;  // root-side copy of `bound` for a shard the root cannot address
    uint64_t rbound_cap = 0;
    // root-side copies for a shard the root cannot address
    uint32_t* r_n = nullptr;
    uint64_t *r_ids = nullptr, *r_post = nullptr;
    double* r_scores = nullptr;
    uint64_t rn_cap = 0, rids_cap = 0, rpost_cap = 0, rsc_cap = 0;
};

}  // namespace

struct hm_sharded {
    std::vector<Shard> shards;
    uint32_t n_docs = 0, n_terms = 0;
    std::mutex mu;  // one batch at a time per sharded index
    // root (devices[0]) merge buffers
    cudaStream_t root_stream = nullptr;
    double* tau = nullptr;
    uint64_t* ids = nullptr;
    double *scores = nullptr, *conf = nullptr;
    uint32_t* n = nullptr;
    uint8_t* skip = nullptr;
    uint64_t* post = nullptr;
    float* ext = nullptr;  // the union's bounds, computed on the root
    uint64_t tau_cap = 0, ids_cap = 0, sc_cap = 0, conf_cap = 0, n_cap = 0, skip_cap = 0, post_cap = 0, ext_cap = 0;

    ~hm_sharded() {
        for (auto& s : shards) {
            if (s.index) hm_index_destroy(s.index);
            cudaSetDevice(s.device);
            void* ps[] = {s.q_off, s.q_tid, s.n, s.ids, s.post, s.scores, s.bound, s.ext};
            for (void* p : ps)
                if (p) cudaFree(p);
            if (s.stream) cudaStreamDestroy(s.stream);
        }
        if (!shards.empty()) {
            cudaSetDevice(shards[0].device);
            for (auto& s : shards) {
                void* ps[] = {s.r_n, s.r_ids, s.r_post, s.r_scores, s.r_bound};
                for (void* p : ps)
                    if (p) cudaFree(p);
            }
            void* ps[] = {tau, ids, scores, conf, n, skip, post, ext};
            for (void* p : ps)
                if (p) cudaFree(p);
            if (root_stream) cudaStreamDestroy(root_stream);
        }
    }
};

namespace {

// shard g's sub-CSR: rows [r0, r1) renumbered from 0, the flat index's
// statistics (idf, order keys, avgdl) unchanged
void build_shard(const hm_csr_view* v, Shard& s) {
    const uint32_t V = v->n_terms, r0 = s.row0, r1 = s.row1;
    std::vector<uint64_t> lo(V), off(V + 1ull, 0);
    for (uint32_t t = 0; t < V; ++t) {
        const uint32_t* b = v->posting_rows + v->term_offsets[t];
        const uint32_t* e = v->posting_rows + v->term_offsets[t + 1];
        const uint32_t* a = std::lower_bound(b, e, r0);
        const uint32_t* z = std::lower_bound(a, e, r1);
        lo[t] = static_cast<uint64_t>(a - v->posting_rows);
        off[t + 1] = off[t] + static_cast<uint64_t>(z - a);
    }
    const uint64_t P = off[V];
    std::vector<uint32_t> rows(P);
    std::vector<uint32_t> tf(v->posting_tf ? P : 0);
    std::vector<double> w(v->posting_tf ? 0 : P);
    for (uint32_t t = 0; t < V; ++t) {
        const uint64_t n = off[t + 1] - off[t];
        for (uint64_t i = 0; i < n; ++i) rows[off[t] + i] = v->posting_rows[lo[t] + i] - r0;
        if (v->posting_tf) std::memcpy(tf.data() + off[t], v->posting_tf + lo[t], n * 4);
        else if (n) std::memcpy(w.data() + off[t], v->posting_weights + lo[t], n * 8);
    }
    hm_csr_view sv = *v;
    sv.term_offsets = off.data();
    sv.posting_rows = rows.data();
    sv.posting_tf = v->posting_tf ? tf.data() : nullptr;
    sv.posting_weights = v->posting_tf ? nullptr : w.data();
    sv.n_docs = r1 - r0;
    sv.doc_lens = v->doc_lens + r0;
    sv.doc_ids = v->doc_ids + r0;
    rethrow_status(hm_index_create(&sv, s.device, &s.index), "hm_index_create(shard)");
}

void search(hm_sharded* H, const hm_query_batch* b, hm_results* out) {
    if (!H || !b || !out) throw std::invalid_argument("null argument");
    const uint32_t nq = b->n_queries;
    if (nq == 0) return;
    if (!b->q_off) throw std::invalid_argument("q_off is required");
    if (!out->ids || !out->scores || !out->n) throw std::invalid_argument("null result buffer");
    if (b->ext_bound || b->out_bound || (b->flags & HM_FLAG_BOUND_ONLY))
        throw std::invalid_argument("the sharded search exchanges the shards' bounds itself");
    for (uint32_t i = 0; i < nq; ++i)
        if (b->q_off[i + 1] < b->q_off[i]) throw std::invalid_argument("q_off not monotone");
    const uint32_t ntid = b->q_off[nq];
    if (ntid && !b->q_tid) throw std::invalid_argument("q_tid is required");
    for (uint32_t i = 0; i < ntid; ++i)
        if (b->q_tid[i] != hm::kNoTerm && b->q_tid[i] >= H->n_terms) throw std::out_of_range("term id out of range");
    const uint32_t row_lo = b->row_lo, row_hi = b->row_hi ? b->row_hi : H->n_docs;
    if (row_hi > H->n_docs) throw std::out_of_range("row window beyond the index's rows");
    const uint32_t k = b->k, kk = std::max(k, 1u);
    const uint32_t G = static_cast<uint32_t>(H->shards.size());
    std::lock_guard<std::mutex> lk(H->mu);

    // 1. every shard: its top-k over its part of the window.  Batches of
    // kBoundMinQueries queries or more first exchange the shards' k-th-score
    // bounds (the seeded pass's k best seed scores, HM_FLAG_BOUND_ONLY; the
    // k-th largest over the shards on the root): each shard then prunes
    // against the union's bound and keeps
    // only documents that can be in the union's top-k -- the merge below is
    // still exact, and a shard's work shrinks like its share of the corpus.
    // (Smaller batches keep row slabs, which the bounds would disable.)
    const bool bounded = G > 1 && nq >= kBoundMinQueries && k > 0 && k <= static_cast<uint32_t>(hm::kMaxK);
    auto prepare = [&](uint32_t g) {
        Shard& s = H->shards[g];
        ck(cudaSetDevice(s.device), "cudaSetDevice");
        grow(s.q_off, s.off_cap, nq + 1ull);
        grow(s.q_tid, s.tid_cap, ntid);
        grow(s.ids, s.ids_cap, static_cast<uint64_t>(nq) * kk);
        grow(s.scores, s.sc_cap, static_cast<uint64_t>(nq) * kk);
        grow(s.n, s.n_cap, nq);
        grow(s.post, s.post_cap, nq);
        grow(s.bound, s.bound_cap, static_cast<uint64_t>(nq) * kk);
        grow(s.ext, s.ext_cap, nq);
    };
    auto window = [&](const Shard& s, hm_query_batch& sb) {
        const uint32_t lo = std::max(row_lo, s.row0), hi = std::min(row_hi, s.row1);
        sb = *b;
        sb.q_off = s.q_off;
        sb.q_tid = s.q_tid;
        sb.tau = nullptr;  // decisions are taken after the merge
        sb.ext_bound = nullptr;
        sb.out_bound = nullptr;
        sb.row_lo = lo < hi ? lo - s.row0 : 0;
        sb.row_hi = lo < hi ? hi - s.row0 : 0;
        return lo < hi;
    };
    if (bounded) {
        run_parallel(G, [&](uint32_t g) {
            prepare(g);
            Shard& s = H->shards[g];
            hm_query_batch sb;
            if (!window(s, sb)) {  // the window misses this shard: no seeds
                ck(cudaMemsetAsync(s.bound, 0, static_cast<uint64_t>(nq) * kk * 4, s.stream), "memset");
                ck(cudaStreamSynchronize(s.stream), "shard sync");
                return;
            }
            ck(cudaMemcpyAsync(s.q_off, b->q_off, (nq + 1ull) * 4, cudaMemcpyHostToDevice, s.stream), "H2D q_off");
            if (ntid)
                ck(cudaMemcpyAsync(s.q_tid, b->q_tid, ntid * 4ull, cudaMemcpyHostToDevice, s.stream), "H2D q_tid");
            sb.flags |= HM_FLAG_BOUND_ONLY;
            sb.out_bound = s.bound;
            hm_results r{s.ids, s.scores, s.n, nullptr, nullptr, s.post};
            rethrow_status(hm_search_batch_device(s.index, &sb, &r, s.stream), "shard bounds");
            ck(cudaStreamSynchronize(s.stream), "shard sync");
        });
        // the root: per query the k-th largest of every shard's k values (over peer
        // memory), then the bound to every shard
        Shard& root = H->shards[0];
        ck(cudaSetDevice(root.device), "cudaSetDevice");
        grow(H->ext, H->ext_cap, nq);
        hm::BoundLists BL{};
        BL.G = G;
        for (uint32_t g = 0; g < G; ++g) {
            Shard& s = H->shards[g];
            if (s.p2p) {
                BL.b[g] = s.bound;
                continue;
            }
            grow(s.r_bound, s.rbound_cap, static_cast<uint64_t>(nq) * kk);
            ck(cudaMemcpyPeerAsync(s.r_bound, root.device, s.bound, s.device, static_cast<uint64_t>(nq) * kk * 4,
                                   H->root_stream),
               "peer copy");
            BL.b[g] = s.r_bound;
        }
        ck(hm::launch_bound_kth(BL, nq, kk, H->ext, H->root_stream), "bound_kth_kernel");
        for (uint32_t g = 0; g < G; ++g) {
            Shard& s = H->shards[g];
            ck(cudaMemcpyPeerAsync(s.ext, s.device, H->ext, root.device, nq * 4ull, H->root_stream), "peer copy");
        }
        ck(cudaStreamSynchronize(H->root_stream), "bound exchange");
    }
    run_parallel(G, [&](uint32_t g) {
        Shard& s = H->shards[g];
        if (!bounded) prepare(g);
        ck(cudaSetDevice(s.device), "cudaSetDevice");
        hm_query_batch sb;
        if (!window(s, sb)) {  // the window misses this shard: empty lists
            ck(cudaMemsetAsync(s.n, 0, nq * 4ull, s.stream), "memset");
            ck(cudaMemsetAsync(s.post, 0, nq * 8ull, s.stream), "memset");
            ck(cudaStreamSynchronize(s.stream), "shard sync");
            return;
        }
        if (bounded) {
            sb.ext_bound = s.ext;
        } else {
            ck(cudaMemcpyAsync(s.q_off, b->q_off, (nq + 1ull) * 4, cudaMemcpyHostToDevice, s.stream), "H2D q_off");
            if (ntid)
                ck(cudaMemcpyAsync(s.q_tid, b->q_tid, ntid * 4ull, cudaMemcpyHostToDevice, s.stream), "H2D q_tid");
        }
        hm_results r{s.ids, s.scores, s.n, nullptr, nullptr, s.post};
        rethrow_status(hm_search_batch_device(s.index, &sb, &r, s.stream), "shard search");
        ck(cudaStreamSynchronize(s.stream), "shard sync");
    });

    // 2. root: all-gather over peer memory fused with the k-way merge
    Shard& root = H->shards[0];
    ck(cudaSetDevice(root.device), "cudaSetDevice");
    cudaStream_t st = H->root_stream;
    grow(H->ids, H->ids_cap, static_cast<uint64_t>(nq) * kk);
    grow(H->scores, H->sc_cap, static_cast<uint64_t>(nq) * kk);
    grow(H->n, H->n_cap, nq);
    grow(H->conf, H->conf_cap, nq);
    grow(H->skip, H->skip_cap, nq);
    grow(H->post, H->post_cap, nq);
    if (b->tau) {
        grow(H->tau, H->tau_cap, nq);
        ck(cudaMemcpyAsync(H->tau, b->tau, nq * 8ull, cudaMemcpyHostToDevice, st), "H2D tau");
    }
    hm::ShardLists L{};
    L.G = G;
    for (uint32_t g = 0; g < G; ++g) {
        Shard& s = H->shards[g];
        if (s.p2p) {
            L.ids[g] = s.ids;
            L.scores[g] = s.scores;
            L.n[g] = s.n;
            L.post[g] = s.post;
            continue;
        }
        grow(s.r_ids, s.rids_cap, static_cast<uint64_t>(nq) * kk);
        grow(s.r_scores, s.rsc_cap, static_cast<uint64_t>(nq) * kk);
        grow(s.r_n, s.rn_cap, nq);
        grow(s.r_post, s.rpost_cap, nq);
        const uint64_t nk = static_cast<uint64_t>(nq) * kk;
        ck(cudaMemcpyPeerAsync(s.r_ids, root.device, s.ids, s.device, nk * 8, st), "peer copy");
        ck(cudaMemcpyPeerAsync(s.r_scores, root.device, s.scores, s.device, nk * 8, st), "peer copy");
        ck(cudaMemcpyPeerAsync(s.r_n, root.device, s.n, s.device, nq * 4ull, st), "peer copy");
        ck(cudaMemcpyPeerAsync(s.r_post, root.device, s.post, s.device, nq * 8ull, st), "peer copy");
        L.ids[g] = s.r_ids;
        L.scores[g] = s.r_scores;
        L.n[g] = s.r_n;
        L.post[g] = s.r_post;
    }
    ck(hm::launch_gather_merge(L, nq, kk, b->tau ? H->tau : nullptr, b->tau_default, b->epsilon_guard, H->ids,
                               H->scores, H->n, H->conf, H->skip, H->post, st),
       "gather_merge_kernel");
    if (k == 0) ck(cudaMemsetAsync(H->n, 0, nq * 4ull, st), "memset");
    // 3. results to the caller (stride k)
    std::vector<uint64_t> rids(static_cast<uint64_t>(nq) * kk);
    std::vector<double> rsc(static_cast<uint64_t>(nq) * kk);
    std::vector<uint32_t> rn(nq);
    ck(cudaMemcpyAsync(rids.data(), H->ids, rids.size() * 8, cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaMemcpyAsync(rsc.data(), H->scores, rsc.size() * 8, cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaMemcpyAsync(rn.data(), H->n, nq * 4ull, cudaMemcpyDeviceToHost, st), "D2H");
    if (out->conf) ck(cudaMemcpyAsync(out->conf, H->conf, nq * 8ull, cudaMemcpyDeviceToHost, st), "D2H");
    if (out->skip) ck(cudaMemcpyAsync(out->skip, H->skip, nq, cudaMemcpyDeviceToHost, st), "D2H");
    if (out->postings) ck(cudaMemcpyAsync(out->postings, H->post, nq * 8ull, cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "merge");
    for (uint32_t i = 0; i < nq; ++i) {
        out->n[i] = rn[i];
        for (uint32_t j = 0; j < rn[i]; ++j) {
            out->ids[static_cast<uint64_t>(i) * k + j] = rids[static_cast<uint64_t>(i) * kk + j];
            out->scores[static_cast<uint64_t>(i) * k + j] = rsc[static_cast<uint64_t>(i) * kk + j];
        }
    }
}

}  // namespace

extern "C" {

int hm_sharded_create(const hm_csr_view* view, const int* devices, uint32_t n_shards, hm_sharded** out) {
    return guard([&] {
        if (!view || !devices || !out) throw std::invalid_argument("null argument");
        if (n_shards == 0 || n_shards > static_cast<uint32_t>(hm::kMaxShards))
            throw std::invalid_argument("n_shards must be in [1, 16]");
        if (view->n_docs < n_shards) throw std::invalid_argument("fewer documents than shards");
        if (!view->term_offsets || (view->term_offsets[view->n_terms] && !view->posting_rows))
            throw std::invalid_argument("hm_csr_view: missing array");
        for (uint32_t g = 0; g < n_shards; ++g) hm_host::use_device(devices[g]);
        auto* H = new hm_sharded();
        try {
            H->n_docs = view->n_docs;
            H->n_terms = view->n_terms;
            H->shards.resize(n_shards);
            for (uint32_t g = 0; g < n_shards; ++g) {
                Shard& s = H->shards[g];
                s.device = devices[g];
                s.row0 = static_cast<uint32_t>(static_cast<uint64_t>(view->n_docs) * g / n_shards);
                s.row1 = static_cast<uint32_t>(static_cast<uint64_t>(view->n_docs) * (g + 1) / n_shards);
            }
            run_parallel(n_shards, [&](uint32_t g) {
                Shard& s = H->shards[g];
                ck(cudaSetDevice(s.device), "cudaSetDevice");
                ck(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking), "stream");
                build_shard(view, s);
            });
            const int root = devices[0];
            ck(cudaSetDevice(root), "cudaSetDevice");
            ck(cudaStreamCreateWithFlags(&H->root_stream, cudaStreamNonBlocking), "stream");
            for (auto& s : H->shards) {
                if (s.device == root) {
                    s.p2p = true;
                    continue;
                }
                int can = 0;
                ck(cudaDeviceCanAccessPeer(&can, root, s.device), "cudaDeviceCanAccessPeer");
                if (can) {
                    const cudaError_t e = cudaDeviceEnablePeerAccess(s.device, 0);
                    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                    else ck(e, "cudaDeviceEnablePeerAccess");
                    s.p2p = true;
                }
            }
        } catch (...) {
            delete H;
            throw;
        }
        *out = H;
    });
}

int hm_sharded_destroy(hm_sharded* s) {
    return guard([&] { delete s; });
}

int hm_sharded_info(const hm_sharded* H, uint32_t* n_shards, uint32_t* shard_row, int* devices, uint32_t* p2p_mask) {
    return guard([&] {
        if (!H) throw std::invalid_argument("null index");
        const uint32_t G = static_cast<uint32_t>(H->shards.size());
        if (n_shards) *n_shards = G;
        uint32_t mask = 0;
        for (uint32_t g = 0; g < G; ++g) {
            if (shard_row) shard_row[g] = H->shards[g].row0;
            if (devices) devices[g] = H->shards[g].device;
            if (H->shards[g].p2p) mask |= 1u << g;
        }
        if (shard_row) shard_row[G] = H->n_docs;
        if (p2p_mask) *p2p_mask = mask;
    });
}

int hm_sharded_search_batch(hm_sharded* H, const hm_query_batch* b, hm_results* out) {
    return guard([&] { search(H, b, out); });
}

}  // extern "C"
