#include <cstdlib>
// C-ABI implementation (include/hm_b200.h): device index build/upload, the
// per-call workspace pool, batch orchestration and error mapping.
//
// Index build (once, at hm_index_create):
//   * raw tf per posting (from the reference's posting_weights doubles or a
//     u32 array) and doc length per row define a (tf, len) pair; the 2^cb - 1
//     most frequent pairs get codes, the rest use the escape code;
//   * packed posting: long terms (local row << 18) | code18, short terms
//     (row << cb) | code_cb, cb = min(8, 32 - row_bits) (see kernels/hm_types.h);
//   * long terms (df > 32 * n_tiles) get a tile-boundary table;
//   * everything is uploaded once and stays resident in HBM.
// Search (per batch): upload query tids, plan kernel, LPT sort, persistent
// selection kernel, persistent exact kernel (takes only flagged queries),
// download results.  No CPU scoring path exists.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <shared_mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include <cuda_runtime.h>

#include "hm_b200.h"
#include "hm_host.h"
#include "hm_launch.h"

namespace {

thread_local uint32_t g_last_exact = 0, g_last_launches = 0, g_last_handed = 0, g_last_graph = 0, g_last_wide = 0;
thread_local float g_ms_plan = 0.f, g_ms_search = 0.f, g_ms_exact = 0.f, g_ms_seed = 0.f;
thread_local bool g_last_seeded = false;
thread_local uint32_t g_last_split = 1;
thread_local std::vector<uint32_t> g_handover;  // HM_FLAG_TIMING batches: fb_list of the seeded pass

using hm_host::ck;
using hm_host::guard;
using hm_host::no_device_error;

int hw_threads() {
    unsigned h = std::thread::hardware_concurrency();
    return h ? static_cast<int>(std::min(h, 64u)) : 1;
}

template <typename F>
void par_for(uint64_t n, F&& f) {
    int T = static_cast<int>(std::min<uint64_t>(hw_threads(), std::max<uint64_t>(n / 65536, 1)));
    if (T <= 1) {
        f(0, 0, n);
        return;
    }
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t)
        pool.emplace_back([&, t] { f(t, n * t / T, n * (t + 1) / T); });
    for (auto& th : pool) th.join();
}

template <typename T>
T* dev_upload(const T* host, uint64_t n, std::vector<void*>& allocs, uint64_t& bytes) {
    void* p = nullptr;
    uint64_t sz = std::max<uint64_t>(n, 1) * sizeof(T);
    ck(cudaMalloc(&p, sz), "cudaMalloc(index)");
    allocs.push_back(p);
    bytes += sz;
    if (n) ck(cudaMemcpy(p, host, n * sizeof(T), cudaMemcpyHostToDevice), "cudaMemcpy(index)");
    return static_cast<T*>(p);
}

// device scratch + stream + pinned staging for one in-flight batch
struct Workspace {
    cudaStream_t stream = nullptr;
    uint32_t nq_cap = 0, tid_cap = 0, k_cap = 0;
    size_t sort_bytes = 0;
    // device
    uint32_t *q_off = nullptr, *q_tid = nullptr, *plan_tid = nullptr, *plan_mult = nullptr,
             *plan_len = nullptr, *order_in = nullptr, *order = nullptr, *counters = nullptr,
             *exact_list = nullptr, *out_n = nullptr, *fb_list = nullptr, *wide_list = nullptr,
             *order_seed = nullptr;
    uint64_t *cost = nullptr, *cost_sorted = nullptr, *out_ids = nullptr, *out_post = nullptr, *cost_seed = nullptr;
    double *tau = nullptr, *out_scores = nullptr, *out_conf = nullptr;
    float* w32 = nullptr;
    uint8_t* out_skip = nullptr;
    void* sort_tmp = nullptr;
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    uint32_t* stab = nullptr;  // per-CTA short-term tile tables
    uint64_t stab_words = 0;
    uint32_t* seed_scratch = nullptr;  // per-CTA seeded-pass scratch
    uint64_t* ne_pend = nullptr;       // per-CTA/warp pending rows of the essential-term sweep
    uint32_t* slab_row = nullptr;      // part boundaries of hm_search_batch_parts
    uint32_t slab_cap = 0;
    // pinned host staging
    unsigned char* pin = nullptr;
    size_t pin_bytes = 0;
    // slab-query results of a split batch (merged into the caller's outputs)
    uint64_t *v_ids = nullptr, *v_post = nullptr;
    double* v_scores = nullptr;
    uint32_t* v_n = nullptr;
    uint64_t v_cap = 0, vk_cap = 0;
    // the wide path (kernels/wide.cu): k > 256 or > 256 distinct terms
    double* wd_scores = nullptr;
    uint64_t wd_scores_cap = 0;
    uint32_t* wd_hist = nullptr;
    hm::WideState* wd_st = nullptr;
    uint32_t wd_g_cap = 0;
    hm::WideCand* wd_cand = nullptr;
    uint64_t wd_cand_cap = 0;
    void* wd_sort = nullptr;
    size_t wd_sort_bytes = 0;
    uint32_t* wd_iota = nullptr;
    uint32_t wd_iota_cap = 0;
    // CUDA graph of the batch's launch sequence, replayed while a batch's
    // arguments repeat (serving loops): captured on the second identical batch
    cudaGraphExec_t gexec = nullptr;
    unsigned char gkey[512] = {}, pkey[512] = {};
    bool gvalid = false, pvalid = false;
    void drop_graph() {
        if (gexec) cudaGraphExecDestroy(gexec);
        gexec = nullptr;
        gvalid = pvalid = false;
    }

    void free_dev() {
        drop_graph();
        void* ps[] = {q_off, q_tid, plan_tid, plan_mult, plan_len, order_in, order, counters,
                      exact_list, fb_list, wide_list, out_n, cost, cost_sorted, out_ids, out_post, tau,
                      order_seed, cost_seed,
                      out_scores, out_conf, w32, out_skip, sort_tmp};
        for (void* p : ps)
            if (p) cudaFree(p);
        q_off = q_tid = plan_tid = plan_mult = plan_len = order_in = order = counters = exact_list =
            out_n = fb_list = wide_list = order_seed = nullptr;
        cost = cost_sorted = out_ids = out_post = cost_seed = nullptr;
        tau = out_scores = out_conf = nullptr;
        w32 = nullptr;
        out_skip = nullptr;
        sort_tmp = nullptr;
    }
    ~Workspace() {
        drop_graph();
        free_dev();
        void* vs[] = {v_ids, v_post, v_scores, v_n, wd_scores, wd_hist, wd_st, wd_cand, wd_sort, wd_iota};
        for (void* p : vs)
            if (p) cudaFree(p);
        if (stab) cudaFree(stab);
        if (seed_scratch) cudaFree(seed_scratch);
        if (ne_pend) cudaFree(ne_pend);
        if (slab_row) cudaFree(slab_row);
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
        if (pin) cudaFreeHost(pin);
        if (stream) cudaStreamDestroy(stream);
    }
};

template <typename T>
void dalloc(T*& p, uint64_t n) {
    void* v = nullptr;
    ck(cudaMalloc(&v, std::max<uint64_t>(n, 1) * sizeof(T)), "cudaMalloc(workspace)");
    p = static_cast<T*>(v);
}

}  // namespace

struct hm_index {
    int device = 0;
    hm::DevIndex dev{};
    std::vector<void*> allocs;
    uint64_t bytes = 0;
    uint32_t row_bits = 0, code_bits = 0, n_codes = 0;
    uint64_t n_escaped = 0;
    uint64_t n_postings = 0;  // a query's cost (postings of its terms) never exceeds it: LPT key bits
    std::vector<uint32_t> code_tf, code_len;
    int grid_search = 0, grid_exact = 0;
    // baked long-term postings (kernels/bake.cu) for one (k1, b)
    uint32_t* d_long_terms = nullptr;
    uint32_t n_long = 0;
    uint32_t* d_bk = nullptr;
    uint32_t* d_bake_err = nullptr;
    std::shared_mutex bake_mu;
    bool bake_valid = false, bake_ok = false;
    double bake_k1 = 0.0, bake_b = 0.0;
    std::mutex mu;
    std::vector<Workspace*> pool;

    ~hm_index() {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        for (auto* w : pool) delete w;
        for (void* p : allocs) cudaFree(p);
        cudaSetDevice(prev);
    }
};

namespace {

using hm_host::use_device;

void build_index(const hm_csr_view* v, hm_index* X) {
    const uint32_t V = v->n_terms, N = v->n_docs;
    if (!v->term_offsets) throw std::invalid_argument("term_offsets is required");
    const uint64_t P = v->term_offsets[V];
    X->n_postings = P;
    if ((P && !v->posting_rows) || (N && (!v->doc_lens || !v->doc_ids)) ||
        (V && (!v->term_idfs || !v->term_order_keys)))
        throw std::invalid_argument("hm_csr_view: missing array");
    if (P && !v->posting_weights == !v->posting_tf)
        throw std::invalid_argument("exactly one of posting_weights / posting_tf must be set");
    // packed row width
    uint32_t row_bits = N <= 1 ? 1 : 32 - __builtin_clz(N - 1);
    if (row_bits > 28)
        throw std::invalid_argument("more than 2^28 rows per index: shard the corpus across devices");
    uint32_t cb = std::min<uint32_t>(8, 32 - row_bits);
    uint32_t esc = (1u << cb) - 1;
    X->row_bits = row_bits;
    X->code_bits = cb;
    // raw tf per posting (BM25 mode: integral, >= 1)
    std::vector<uint32_t> tf(P);
    std::atomic<int> bad{0};
    par_for(P, [&](int, uint64_t a, uint64_t b) {
        for (uint64_t i = a; i < b; ++i) {
            uint32_t t;
            if (v->posting_tf) {
                t = v->posting_tf[i];
            } else {
                double w = v->posting_weights[i];
                if (!(w >= 1.0 && w < 4294967296.0) || w != std::floor(w)) {
                    bad = 1;
                    t = 1;
                } else {
                    t = static_cast<uint32_t>(w);
                }
            }
            if (t == 0) bad = 1;
            if (v->posting_rows[i] >= N) bad = 2;
            tf[i] = t;
        }
    });
    if (bad == 1)
        throw std::runtime_error("BM25 scoring requires a BM25-mode index (raw integral tf weights)");
    if (bad == 2) throw std::out_of_range("posting row out of range");
    // rows strictly increasing per term
    par_for(V, [&](int, uint64_t a, uint64_t b) {
        for (uint64_t t = a; t < b; ++t) {
            uint64_t lo = v->term_offsets[t], hi = v->term_offsets[t + 1];
            if (hi < lo || hi > P) {
                bad = 3;
                return;
            }
            for (uint64_t i = lo + 1; i < hi; ++i)
                if (v->posting_rows[i] <= v->posting_rows[i - 1]) bad = 4;
        }
    });
    if (bad == 3) throw std::invalid_argument("term_offsets not monotone");
    if (bad == 4) throw std::invalid_argument("posting rows must be strictly increasing per term");
    // (tf, len) pair histogram: dense for small pairs, hashed otherwise
    constexpr uint32_t kTfD = 64, kLenD = 4096;
    const int T = hw_threads();
    std::vector<std::vector<uint64_t>> dense(T);
    std::vector<std::unordered_map<uint64_t, uint64_t>> sparse(T);
    auto key = [](uint64_t t, uint64_t l) { return (t << 32) | l; };
    {
        std::vector<std::thread> pool;
        for (int t = 0; t < T; ++t)
            pool.emplace_back([&, t] {
                dense[t].assign(static_cast<size_t>(kTfD) * kLenD, 0);
                uint64_t a = P * t / T, b = P * (t + 1) / T;
                for (uint64_t i = a; i < b; ++i) {
                    uint32_t f = tf[i], l = v->doc_lens[v->posting_rows[i]];
                    if (f < kTfD && l < kLenD) ++dense[t][static_cast<size_t>(f) * kLenD + l];
                    else ++sparse[t][key(f, l)];
                }
            });
        for (auto& th : pool) th.join();
    }
    std::vector<std::pair<uint64_t, uint64_t>> pairs;  // (count, key)
    {
        std::vector<uint64_t> dsum(static_cast<size_t>(kTfD) * kLenD, 0);
        std::unordered_map<uint64_t, uint64_t> ssum;
        for (int t = 0; t < T; ++t) {
            for (size_t i = 0; i < dsum.size(); ++i) dsum[i] += dense[t][i];
            for (auto& kv : sparse[t]) ssum[kv.first] += kv.second;
            std::vector<uint64_t>().swap(dense[t]);
        }
        for (size_t i = 0; i < dsum.size(); ++i)
            if (dsum[i]) pairs.emplace_back(dsum[i], key(i / kLenD, i % kLenD));
        for (auto& kv : ssum) pairs.emplace_back(kv.second, kv.first);
    }
    std::sort(pairs.begin(), pairs.end(), [](const auto& x, const auto& y) {
        if (x.first != y.first) return x.first > y.first;
        return x.second < y.second;
    });
    // code table: the kMaxCodes most frequent pairs; short-term postings can
    // only address the first esc_short of them (their code field is cb bits)
    // (code kCodeMask is reserved: a long escape masked to 12 bits lands on it, and its impact is 0)
    const uint32_t n_codes = static_cast<uint32_t>(std::min<size_t>(pairs.size(), hm::kCodeMask));
    const uint32_t n_codes_short = std::min(n_codes, esc);
    X->n_codes = n_codes;
    X->code_tf.assign(hm::kMaxCodes, 0);
    X->code_len.assign(hm::kMaxCodes, 0);
    std::vector<uint16_t> dense_code(static_cast<size_t>(kTfD) * kLenD, 0xFFFF);
    std::unordered_map<uint64_t, uint32_t> sparse_code;
    for (uint32_t c = 0; c < n_codes; ++c) {
        uint64_t kk = pairs[c].second;
        uint32_t f = static_cast<uint32_t>(kk >> 32), l = static_cast<uint32_t>(kk);
        X->code_tf[c] = f;
        X->code_len[c] = l;
        if (f < kTfD && l < kLenD) dense_code[static_cast<size_t>(f) * kLenD + l] = static_cast<uint16_t>(c);
        else sparse_code[kk] = c;
    }
    // long terms (tile table) vs short terms
    const uint32_t n_tiles = std::max<uint32_t>(1, (N + hm::kTile - 1) / hm::kTile);
    std::vector<int32_t> slot(V, -1);
    std::vector<uint32_t> long_terms;
    for (uint32_t t = 0; t < V; ++t) {
        uint64_t df = v->term_offsets[t + 1] - v->term_offsets[t];
        if (df > static_cast<uint64_t>(hm::kLongFactor) * n_tiles) {
            slot[t] = static_cast<int32_t>(long_terms.size());
            long_terms.push_back(t);
        }
    }
    // short terms' tile tables (hm_types.h short_tab): one pass over each
    // such term's rows
    // (terms with fewer postings than half the tiles cost less to scan per query
    // than their table's n_tiles + 1 entries to fill: none kept for them)
    std::vector<uint32_t> stab_row(std::max<uint32_t>(V, 1), hm::kNoTabRow);
    uint64_t n_stab = 0;
    const uint64_t stab_min = std::max<uint64_t>(hm::kShortTabMinDf, n_tiles / 2);
    for (uint32_t t = 0; t < V; ++t) {
        const uint64_t df = v->term_offsets[t + 1] - v->term_offsets[t];
        if (slot[t] < 0 && df >= stab_min) stab_row[t] = static_cast<uint32_t>(n_stab++);
    }
    std::vector<uint32_t> stab_all(std::max<uint64_t>(n_stab, 1) * (n_tiles + 1));
    par_for(V, [&](int, uint64_t a, uint64_t b) {
        for (uint64_t t = a; t < b; ++t) {
            if (stab_row[t] == hm::kNoTabRow) continue;
            const uint64_t o = v->term_offsets[t], df = v->term_offsets[t + 1] - o;
            uint32_t* T = stab_all.data() + static_cast<uint64_t>(stab_row[t]) * (n_tiles + 1);
            uint64_t i = 0;
            for (uint32_t j = 0; j <= n_tiles; ++j) {
                const uint64_t r0 = static_cast<uint64_t>(j) << hm::kTileShift;
                while (i < df && v->posting_rows[o + i] < r0) ++i;
                T[j] = static_cast<uint32_t>(i);
            }
        }
    });
    // packed postings (+8 words of padding for 16-byte bulk copies)
    std::vector<uint32_t> packed(P + 8, 0);
    std::atomic<uint64_t> escaped{0};
    par_for(V, [&](int, uint64_t a, uint64_t b) {
        uint64_t esc_local = 0;
        for (uint64_t t = a; t < b; ++t) {
            const bool lng = slot[t] >= 0;
            for (uint64_t i = v->term_offsets[t]; i < v->term_offsets[t + 1]; ++i) {
                uint32_t r = v->posting_rows[i], f = tf[i], l = v->doc_lens[r];
                uint32_t code = 0xFFFFFFFFu;
                if (f < kTfD && l < kLenD) {
                    uint16_t c16 = dense_code[static_cast<size_t>(f) * kLenD + l];
                    if (c16 != 0xFFFF) code = c16;
                } else {
                    auto it = sparse_code.find(key(f, l));
                    if (it != sparse_code.end()) code = it->second;
                }
                if (lng) {
                    if (code >= n_codes) {
                        code = hm::kEscLong;
                        ++esc_local;
                    }
                    packed[i] = ((r & (hm::kTile - 1)) << hm::kCodeBitsLong) | code;
                } else {
                    if (code >= n_codes_short) {
                        code = esc;
                        ++esc_local;
                    }
                    packed[i] = (r << cb) | code;
                }
            }
        }
        escaped += esc_local;
    });
    X->n_escaped = escaped;
    std::vector<uint8_t> long_esc(std::max<size_t>(long_terms.size(), 1), 0);
    par_for(long_terms.size(), [&](int, uint64_t a, uint64_t b) {
        for (uint64_t s = a; s < b; ++s) {
            uint32_t t = long_terms[s];
            for (uint64_t i = v->term_offsets[t]; i < v->term_offsets[t + 1]; ++i)
                if ((packed[i] & hm::kEscLong) == hm::kEscLong) {
                    long_esc[s] = 1;
                    break;
                }
        }
    });
    // long-term sub-tile tables (1024-row granularity; tile j starts at 16*j)
    const uint64_t n_sub = static_cast<uint64_t>(n_tiles) * hm::kSubPerTile;
    std::vector<uint32_t> tab(long_terms.size() * (n_sub + 1));
    par_for(long_terms.size(), [&](int, uint64_t a, uint64_t b) {
        for (uint64_t s = a; s < b; ++s) {
            uint32_t t = long_terms[s];
            uint64_t lo = v->term_offsets[t], hi = v->term_offsets[t + 1];
            uint32_t* row = tab.data() + s * (n_sub + 1);
            uint64_t i = lo;
            for (uint64_t j = 0; j <= n_sub; ++j) {
                uint64_t lim = j << hm::kSubShift;
                while (i < hi && v->posting_rows[i] < lim) ++i;
                row[j] = static_cast<uint32_t>(i - lo);
            }
            row[n_sub] = static_cast<uint32_t>(hi - lo);
        }
    });
    // dense probe arrays (seeded kernel): the most frequent long terms get a
    // per-row u16 (tf, len) code so a probe is one load
    std::vector<int32_t> dense_of(std::max<size_t>(long_terms.size(), 1), -1);
    std::vector<uint32_t> dense_slots;
    if (N >= 65536) {
        std::vector<uint32_t> cand;
        auto dfs = [&](uint32_t s) { return v->term_offsets[long_terms[s] + 1] - v->term_offsets[long_terms[s]]; };
        for (size_t s = 0; s < long_terms.size(); ++s)
            if (dfs(static_cast<uint32_t>(s)) >= N / hm::kDenseMinDiv) cand.push_back(static_cast<uint32_t>(s));
        std::sort(cand.begin(), cand.end(),
                  [&](uint32_t a, uint32_t b) { return dfs(a) > dfs(b) || (dfs(a) == dfs(b) && a < b); });
        if (cand.size() > static_cast<size_t>(hm::kMaxDense)) cand.resize(hm::kMaxDense);
        dense_slots = cand;
        for (size_t dd = 0; dd < cand.size(); ++dd) dense_of[cand[dd]] = static_cast<int32_t>(dd);
    }
    std::vector<float> idf32(V);
    for (uint32_t t = 0; t < V; ++t) idf32[t] = static_cast<float>(v->term_idfs[t]);
    // upload
    auto& A = X->allocs;
    auto& B = X->bytes;
    hm::DevIndex& d = X->dev;
    d.post = dev_upload(packed.data(), P + 8, A, B);
    d.tf = dev_upload(tf.data(), P, A, B);
    std::vector<uint32_t>().swap(tf);
    d.term_off = dev_upload(v->term_offsets, static_cast<uint64_t>(V) + 1, A, B);
    d.idf = dev_upload(v->term_idfs, V, A, B);
    d.idf32 = dev_upload(idf32.data(), V, A, B);
    d.order_key = dev_upload(v->term_order_keys, V, A, B);
    d.long_slot = dev_upload(slot.data(), V, A, B);
    d.tile_tab = dev_upload(tab.data(), tab.size(), A, B);
    d.short_tab = dev_upload(stab_all.data(), stab_all.size(), A, B);
    d.short_tab_row = dev_upload(stab_row.data(), std::max<uint64_t>(V, 1), A, B);
    std::vector<uint32_t>().swap(stab_all);
    d.long_esc = dev_upload(long_esc.data(), long_esc.size(), A, B);
    d.doc_lens = dev_upload(v->doc_lens, N, A, B);
    d.doc_ids = dev_upload(v->doc_ids, N, A, B);
    d.code_tf = dev_upload(X->code_tf.data(), hm::kMaxCodes, A, B);
    d.code_len = dev_upload(X->code_len.data(), hm::kMaxCodes, A, B);
    {
        d.dense_of_slot = dev_upload(dense_of.data(), dense_of.size(), A, B);
        const uint64_t nd = dense_slots.size();
        void* p = nullptr;
        ck(cudaMalloc(&p, std::max<uint64_t>(nd * N, 1) * 2), "cudaMalloc(dense)");
        A.push_back(p);
        B += std::max<uint64_t>(nd * N, 1) * 2;
        d.dense = static_cast<const uint16_t*>(p);
        std::vector<uint16_t> col(N);
        for (uint64_t dd = 0; dd < nd; ++dd) {
            const uint32_t s = dense_slots[dd], t = long_terms[s];
            std::fill(col.begin(), col.end(), hm::kDenseAbsent);
            for (uint64_t i = v->term_offsets[t]; i < v->term_offsets[t + 1]; ++i) {
                const uint32_t code = packed[i] & hm::kEscLong;
                col[v->posting_rows[i]] = code < n_codes ? static_cast<uint16_t>(code) : hm::kDenseEscape;
            }
            ck(cudaMemcpy(static_cast<uint16_t*>(p) + dd * N, col.data(), N * 2ull, cudaMemcpyHostToDevice),
               "cudaMemcpy(dense)");
        }
        ck(cudaMalloc(&p, std::max<uint64_t>(V, 1) * 4), "cudaMalloc(tmax)");
        A.push_back(p);
        B += std::max<uint64_t>(V, 1) * 4;
        d.tmax = static_cast<const float*>(p);
    }
    std::vector<uint32_t>().swap(packed);
    X->n_long = static_cast<uint32_t>(long_terms.size());
    X->d_long_terms = dev_upload(long_terms.data(), long_terms.size(), A, B);
    // baked-posting index space: every (long term, 2048-row unit) range padded
    // to a multiple of 4 words and 16-byte aligned (kernels/bake.cu)
    {
        const uint64_t n_units = static_cast<uint64_t>(n_tiles) * hm::kUnitsPerTile;
        std::vector<uint64_t> base(std::max<size_t>(long_terms.size(), 1), 0);
        std::vector<uint32_t> uoff(long_terms.size() * (n_units + 1));
        uint64_t tot = 0;
        for (size_t s = 0; s < long_terms.size(); ++s) {
            const uint32_t* row = tab.data() + s * (n_sub + 1);
            uint32_t* uo = uoff.data() + s * (n_units + 1);
            base[s] = tot;
            uint32_t acc = 0;
            for (uint64_t u = 0; u < n_units; ++u) {
                uo[u] = acc;
                const uint32_t n = row[(u + 1) * hm::kSubPerUnit] - row[u * hm::kSubPerUnit];
                acc += (n + 3) & ~3u;
            }
            uo[n_units] = acc;
            tot += acc;
        }
        d.bk_base = dev_upload(base.data(), base.size(), A, B);
        d.bk_uoff = dev_upload(uoff.data(), uoff.size(), A, B);
        d.n_units = static_cast<uint32_t>(n_units);
        void* p = nullptr;
        ck(cudaMalloc(&p, std::max<uint64_t>(tot, 4) * 4), "cudaMalloc(bk)");
        A.push_back(p);
        B += std::max<uint64_t>(tot, 4) * 4;
        X->d_bk = static_cast<uint32_t*>(p);
        ck(cudaMalloc(&p, 16), "cudaMalloc(bake err)");
        A.push_back(p);
        X->d_bake_err = static_cast<uint32_t*>(p);
    }
    d.bk = X->d_bk;
    d.bk_ks = 0;
    d.n_terms = V;
    d.n_docs = N;
    d.n_tiles = n_tiles;
    d.code_bits = cb;
    d.esc_short = esc;
    d.n_codes = n_codes;
    d.n_codes_short = n_codes_short;
    d.avgdl = v->avgdl;
    int sb = 0, eb = 0, sms = 0;
    ck(hm::search_occupancy(&sb, &eb), "occupancy");
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, X->device), "SM count");
    if (sb < 1 || eb < 1) throw std::runtime_error("search kernels do not fit on this device");
    X->grid_search = sb * sms;
    X->grid_exact = eb * sms;
}

Workspace* acquire(hm_index* X) {
    {
        std::lock_guard<std::mutex> lk(X->mu);
        if (!X->pool.empty()) {
            Workspace* w = X->pool.back();
            X->pool.pop_back();
            return w;
        }
    }
    auto* w = new Workspace();
    ck(cudaStreamCreateWithFlags(&w->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    return w;
}

void release(hm_index* X, Workspace* w) {
    std::lock_guard<std::mutex> lk(X->mu);
    X->pool.push_back(w);
}

void ensure(Workspace* w, uint32_t nq, uint32_t ntid, uint32_t k, bool need_io) {
    if (nq > w->nq_cap || ntid > w->tid_cap || k > w->k_cap || !w->counters) {
        cudaStreamSynchronize(w->stream);
        w->free_dev();
        uint32_t NQ = std::max(nq, std::max(w->nq_cap, 1u));
        uint32_t NT = std::max(ntid, std::max(w->tid_cap, 1u));
        uint32_t K = std::max(k, std::max(w->k_cap, 1u));
        dalloc(w->q_off, NQ + 1ull);
        dalloc(w->q_tid, NT);
        dalloc(w->plan_tid, NT);
        dalloc(w->plan_mult, NT);
        dalloc(w->plan_len, NQ);
        dalloc(w->order_in, NQ);
        dalloc(w->order, NQ);
        dalloc(w->counters, 16);
        dalloc(w->exact_list, NQ);
        dalloc(w->fb_list, NQ);
        dalloc(w->wide_list, NQ);
        dalloc(w->cost, NQ);
        dalloc(w->cost_sorted, NQ);
        dalloc(w->cost_seed, NQ);
        dalloc(w->order_seed, NQ);
        dalloc(w->tau, NQ);
        dalloc(w->w32, hm::kMaxCodes);
        dalloc(w->out_ids, static_cast<uint64_t>(NQ) * K);
        dalloc(w->out_scores, static_cast<uint64_t>(NQ) * K);
        dalloc(w->out_n, NQ);
        dalloc(w->out_conf, NQ);
        dalloc(w->out_skip, NQ);
        dalloc(w->out_post, NQ);
        ck(hm::lpt_sort_bytes(NQ, &w->sort_bytes), "cub sort sizing");
        void* t = nullptr;
        ck(cudaMalloc(&t, std::max<size_t>(w->sort_bytes, 16)), "cudaMalloc(sort)");
        w->sort_tmp = t;
        w->nq_cap = NQ;
        w->tid_cap = NT;
        w->k_cap = K;
    }
    // pinned staging: inputs (q_off, q_tid, tau, w32) + outputs
    size_t need = 1024 + hm::kMaxCodes * 4;
    if (need_io)
        need += (nq + 1ull) * 4 + ntid * 4ull + nq * 8ull +
                static_cast<size_t>(nq) * k * 16 + nq * (4ull + 8 + 1 + 8) + 64;
    if (need > w->pin_bytes) {
        cudaStreamSynchronize(w->stream);
        if (w->pin) cudaFreeHost(w->pin);
        w->pin = nullptr;
        ck(cudaMallocHost(&w->pin, need * 2), "cudaMallocHost");
        w->pin_bytes = need * 2;
    }
}

bool needs_exact(double k1, double b) { return !(k1 >= 0.0 && b >= 0.0 && b <= 1.0); }

// impact table of the codes for (k1, b): tf*(k1+1)/(tf + k1*(1-b+b*len/avgdl))
void fill_w32(const hm_index* X, double k1, double b, float* w) {
    const double avgdl = X->dev.avgdl;
    for (uint32_t c = 0; c < hm::kMaxCodes; ++c) {
        if (c >= X->n_codes) {
            w[c] = 0.f;
            continue;
        }
        double tf = X->code_tf[c], dl = X->code_len[c];
        double norm = avgdl > 0.0 ? dl / avgdl : 1.0;
        double denom = tf + k1 * (1.0 - b + b * norm);
        w[c] = static_cast<float>(tf * (k1 + 1.0) / denom);
    }
}

// enqueue the whole batch on w->stream; batch arrays already on the device
// Small batches leave most CTAs idle (one CTA per query): each query is then
// split into row slabs served as separate "slab queries" -- exact per-slab
// top-k lists, merged by merge_kernel exactly like doc shards (§4).  The
// intra-query data parallelism of PAPER.md:616.
// the seeded pass runs on row windows of at least this many rows (8 tiles)
constexpr uint32_t kSeedMinRows = 1u << 17;

uint32_t split_for(const hm_index* X, const hm_query_batch& hb) {
    if ((hb.flags & (HM_FLAG_NO_SPLIT | HM_FLAG_FORCE_EXACT | HM_FLAG_BOUND_ONLY)) || needs_exact(hb.k1, hb.b) ||
        hb.n_queries == 0 || hb.k == 0 || hb.ext_bound || hb.out_bound)
        return 1;  // (the fp64 fallback path keeps one CTA per query; shard bounds are per real query)
    const uint32_t nq = hb.n_queries, k = hb.k;
    // resident sweep CTAs (launch_search runs 2 per unit of grid_search); the
    // batch is split while the heaviest query, not the total work, would set
    // the time
    const uint64_t resident = 2ull * static_cast<uint64_t>(X->grid_search);
    const uint32_t hi = hb.row_hi == 0 ? X->dev.n_docs : std::min(hb.row_hi, X->dev.n_docs);
    const uint32_t span = hi > hb.row_lo ? hi - hb.row_lo : 0;
    // slab queries per resident CTA, measured on C2 (profiles/r01_latency.md):
    // tiny batches one (per-slab overheads dominate thin slabs), 32-255
    // queries four, 256+ eight (LPT then evens out the heaviest queries)
    const uint64_t target = nq < 32 ? resident : nq < 256 ? 4 * resident : 8 * resident;
#ifndef HM_MAX_SLABS
#define HM_MAX_SLABS 64
#endif
    uint32_t S = static_cast<uint32_t>(std::min<uint64_t>(target / nq, HM_MAX_SLABS));
    S = std::min<uint32_t>(S, 2048 / k);  // merge_kernel holds split x k candidates
    S = std::min<uint32_t>(S, span / hm::kTile);  // at least a tile per slab
    return S >= 2 ? S : 1;
}

// d_slab_row (n_parts + 1 device boundaries): every query is searched inside
// each part separately; the per-part lists stay in the workspace's v_* arrays
// ([part][query][k]) instead of being merged (hm_search_batch_parts)
void run_batch(hm_index* X, Workspace* w, const hm_query_batch& hb, const uint32_t* d_off,
               const uint32_t* d_tid, const double* d_tau, const hm_results& out, float* pin_w32,
               uint32_t n_parts = 0, const uint32_t* d_slab_row = nullptr) {
    const uint32_t nq = hb.n_queries;
    hm::BatchArgs a{};
    a.nq = nq;
    a.k = hb.k;
    a.q_off = d_off;
    a.q_tid = d_tid;
    a.k1 = hb.k1;
    a.b = hb.b;
    a.tau = d_tau;
    a.tau_default = hb.tau_default;
    a.eps = hb.epsilon_guard;
    a.row_lo = hb.row_lo;
    a.row_hi = hb.row_hi == 0 ? X->dev.n_docs : std::min(hb.row_hi, X->dev.n_docs);
    a.flags = hb.flags | (needs_exact(hb.k1, hb.b) ? HM_FLAG_FORCE_EXACT : 0u);
    a.w32 = w->w32;
    a.plan_tid = w->plan_tid;
    a.plan_mult = w->plan_mult;
    a.plan_len = w->plan_len;
    a.cost = w->cost;
    a.order = w->order;
    a.counters = w->counters;
    a.exact_list = w->exact_list;
    a.wide_list = w->wide_list;
    a.stab_stride = X->dev.n_tiles + 2;
    const uint64_t words = 2ull * X->grid_search * hm::kMaxTerms * a.stab_stride;  // up to 2 CTAs per SM
    if (w->stab_words < words) {
        ck(cudaStreamSynchronize(w->stream), "sync");
        if (w->stab) cudaFree(w->stab);
        w->stab = nullptr;
        w->stab_words = 0;
        dalloc(w->stab, words);
        w->stab_words = words;
    }
    a.stab = w->stab;
    a.seed_half = std::max<uint32_t>(1, std::min<uint32_t>(hm::kSeedScratch / 2, X->dev.n_docs));
    a.seed_scratch = w->seed_scratch;  // allocated below when the seeded pass runs
    a.out_ids = out.ids;
    a.out_scores = out.scores;
    a.out_n = out.n;
    a.out_conf = out.conf;
    a.out_skip = out.skip;
    a.out_post = out.postings;
    a.ext_bound = hb.ext_bound;
    a.out_bound = hb.out_bound;
    const uint32_t split = d_slab_row ? n_parts : split_for(X, hb);
    a.split = split;
    a.nq_real = nq;
    a.slab_row = d_slab_row;
    const bool merge = split > 1 && !d_slab_row;
    if (split > 1 || d_slab_row) {  // slab queries: results into the workspace, decisions at the merge
        const uint64_t nv = static_cast<uint64_t>(nq) * split;
        if (nv > w->v_cap || hb.k > w->vk_cap) {
            ck(cudaStreamSynchronize(w->stream), "sync");
            void* vs[] = {w->v_ids, w->v_post, w->v_scores, w->v_n};
            for (void* p : vs)
                if (p) cudaFree(p);
            const uint64_t NV = std::max(nv, w->v_cap);
            const uint64_t K = std::max<uint64_t>(hb.k, w->vk_cap);
            dalloc(w->v_ids, NV * K);
            dalloc(w->v_scores, NV * K);
            dalloc(w->v_n, NV);
            dalloc(w->v_post, NV);
            w->v_cap = NV;
            w->vk_cap = K;
        }
        a.nq = static_cast<uint32_t>(nv);
        a.tau = nullptr;
        a.out_ids = w->v_ids;
        a.out_scores = w->v_scores;
        a.out_n = w->v_n;
        a.out_conf = nullptr;
        a.out_skip = nullptr;
        a.out_post = w->v_post;
    }
    fill_w32(X, hb.k1, hb.b, pin_w32);
    cudaStream_t st = w->stream;
    const bool timing = (hb.flags & HM_FLAG_TIMING) != 0;
    if (timing && !w->ev[0])
        for (auto& e : w->ev) ck(cudaEventCreate(&e), "event");
    // seeded MaxScore first (exact; serves the queries with a rare term), the
    // exhaustive kernel for the rest; HM_FLAG_EXHAUSTIVE skips the seeded pass
    // (a narrow row window -- a recency window of the temporal index -- keeps
    // every query cheap on the exhaustive kernel: no seeded pass)
    // (and an index of a few tiles -- C1's 100K docs -- sweeps every query faster
    // than the pass's fixed per-query work: 0.58 vs 0.94 ms per 1K queries)
    const bool seeded = !(a.flags & (HM_FLAG_EXHAUSTIVE | HM_FLAG_FORCE_EXACT)) &&
                        ((a.flags & HM_FLAG_SEED_ALL) || (4ull * (a.row_hi - a.row_lo) >= X->dev.n_docs &&
                                                          a.row_hi - a.row_lo >= kSeedMinRows));
    if (seeded && split == 1) {  // the seeded pass walks its own LPT order (its cost is not the sweep's)
        a.cost_seed = w->cost_seed;
        a.order_seed = w->order_seed;
    }
    if (seeded) {
        a.fb_list = w->fb_list;
        if (!w->seed_scratch) dalloc(w->seed_scratch, 2ull * X->grid_search * 2ull * a.seed_half);  // up to 2 CTAs per SM
        a.seed_scratch = w->seed_scratch;
    }
    a.ne_pend = nullptr;
    if (hm::sweep_ne_launched(a)) {  // up to 2 sweep CTAs per SM, 8 warps each
        if (!w->ne_pend) dalloc(w->ne_pend, 2ull * X->grid_search * 8ull * hm::kNePendCap);
        a.ne_pend = w->ne_pend;
    }
    g_last_seeded = seeded;
    g_last_split = split;
    g_last_launches = (seeded ? 4 : 3) + (split > 1 ? 1 : 0) + (merge ? 2 : 0) +  // ours: plan, [seeded,] exhaustive, exact
                      (hm::sweep_ne_launched(a) ? 1 : 0);                      // [+ essential-term sweep]
                                                             // [+ expand, merge, postings] (plus CUB's sort)
    auto enqueue = [&] {
        ck(cudaMemcpyAsync(w->w32, pin_w32, hm::kMaxCodes * sizeof(float), cudaMemcpyHostToDevice, st),
           "upload w32");
        ck(cudaMemsetAsync(w->counters, 0, 16 * sizeof(uint32_t), st), "memset counters");
        if (timing) ck(cudaEventRecord(w->ev[0], st), "event");
        // the costs are postings counts <= the index's: radix passes over those bits only
        const int key_bits = X->n_postings ? 64 - __builtin_clzll(X->n_postings) : 1;
        if (split > 1) {  // plan + LPT over the real queries, then every slab of each
            hm::BatchArgs ap = a;
            ap.nq = nq;
            ap.order = w->exact_list;  // scratch until the sweep appends to it
            ck(hm::launch_plan(X->dev, ap, w->order_in, st), "plan kernel");
            ck(hm::launch_lpt_sort(w->sort_tmp, w->sort_bytes, ap, w->cost_sorted, w->order_in, key_bits, st),
               "lpt sort");
            ck(hm::launch_expand_order(nq, split, w->exact_list, w->order, st), "expand order");
        } else {
            ck(hm::launch_plan(X->dev, a, w->order_in, st), "plan kernel");
            ck(hm::launch_lpt_sort(w->sort_tmp, w->sort_bytes, a, w->cost_sorted, w->order_in, key_bits, st),
               "lpt sort");
            if (a.order_seed)  // the seeded pass's own LPT order
                ck(hm::launch_seed_sort(w->sort_tmp, w->sort_bytes, a, w->cost_sorted, w->order_in, w->order_seed,
                                        key_bits, st),
                   "seed lpt sort");
        }
        if (timing) ck(cudaEventRecord(w->ev[1], st), "event");
        if (a.flags & HM_FLAG_BOUND_ONLY) {  // doc shards' bound pass: the seeded pass's L per query
            if (seeded) {
                ck(cudaMemsetAsync(w->fb_list, 0, static_cast<uint64_t>(a.nq) * sizeof(uint32_t), st), "memset");
                ck(hm::launch_search_seed(X->dev, a, 2 * X->grid_search, st), "seeded search kernel (bounds)");
            } else {
                ck(cudaMemsetAsync(a.out_bound, 0, static_cast<uint64_t>(nq) * hb.k * sizeof(float), st),
                   "memset bounds");
            }
            if (timing) {
                ck(cudaEventRecord(w->ev[4], st), "event");
                ck(cudaEventRecord(w->ev[2], st), "event");
                ck(cudaEventRecord(w->ev[3], st), "event");
            }
            return;
        }
        if (seeded) {
            ck(cudaMemsetAsync(w->fb_list, 0, static_cast<uint64_t>(a.nq) * sizeof(uint32_t), st), "memset hand-over flags");
            ck(hm::launch_search_seed(X->dev, a, 2 * X->grid_search, st), "seeded search kernel");
        }
        if (timing) ck(cudaEventRecord(w->ev[4], st), "event");
        ck(hm::launch_search(X->dev, a, X->grid_search, st), "search kernel");
        if (timing) ck(cudaEventRecord(w->ev[2], st), "event");
        ck(hm::launch_exact(X->dev, a, X->grid_exact, st), "exact kernel");
        if (merge) {  // the slabs' exact lists -> the real queries' top-k, Margin, skip
            ck(hm::launch_merge(split, nq, hb.k, w->v_ids, w->v_scores, w->v_n, d_tau, hb.tau_default,
                                hb.epsilon_guard, out.ids, out.scores, out.n, out.conf, out.skip, st),
               "slab merge");
            ck(hm::launch_sum_slab_postings(nq, split, w->v_post, out.postings, st), "slab postings");
        }
        if (timing) ck(cudaEventRecord(w->ev[3], st), "event");
    };
    g_last_graph = 0;
    if (timing) {  // per-kernel events: run eagerly
        enqueue();
        return;
    }
    // the launch sequence depends only on the arguments below: a batch equal
    // to the previous one is captured into a graph, later equal batches
    // replay it (one launch instead of eight stream operations)
    unsigned char key[512] = {};
    static_assert(sizeof(hm::BatchArgs) + 4 * sizeof(int) + 2 * sizeof(void*) + sizeof(size_t) <= sizeof(key),
                  "graph key");
    {
        unsigned char* k = key;
        std::memcpy(k, &a, sizeof a);  // value-initialised: padding is zero
        k += sizeof a;
        const int ints[4] = {seeded ? 1 : 0, X->grid_search, X->grid_exact, static_cast<int>(nq)};
        std::memcpy(k, ints, sizeof ints);
        k += sizeof ints;
        std::memcpy(k, &w->sort_tmp, sizeof(void*));
        k += sizeof(void*);
        std::memcpy(k, &pin_w32, sizeof(void*));
        k += sizeof(void*);
        std::memcpy(k, &w->sort_bytes, sizeof(size_t));
    }
    if (w->gvalid && std::memcmp(key, w->gkey, sizeof key) == 0) {
        ck(cudaGraphLaunch(w->gexec, st), "graph launch");
        g_last_graph = 2;
        return;
    }
    if (!(w->pvalid && std::memcmp(key, w->pkey, sizeof key) == 0)) {  // first sighting: eager
        enqueue();
        std::memcpy(w->pkey, key, sizeof key);
        w->pvalid = true;
        return;
    }
    ck(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "begin capture");
    cudaGraph_t g = nullptr;
    try {
        enqueue();
    } catch (...) {
        cudaStreamEndCapture(st, &g);
        if (g) cudaGraphDestroy(g);
        throw;
    }
    ck(cudaStreamEndCapture(st, &g), "end capture");
    if (w->gexec) cudaGraphExecDestroy(w->gexec);
    w->gexec = nullptr;
    w->gvalid = false;
    const cudaError_t ie = cudaGraphInstantiate(&w->gexec, g, 0);
    cudaGraphDestroy(g);
    ck(ie, "graph instantiate");
    std::memcpy(w->gkey, key, sizeof key);
    w->gvalid = true;
    ck(cudaGraphLaunch(w->gexec, st), "graph launch");
    g_last_graph = 1;
}

// Arguments of the wide path for a planned batch (plan arrays in w).
hm::BatchArgs wide_args(const hm_index* X, const Workspace* w, const hm_query_batch& hb, const uint32_t* d_off,
                        const uint32_t* d_tid, const double* d_tau, const hm_results& out) {
    hm::BatchArgs a{};
    a.nq = hb.n_queries;
    a.k = hb.k;
    a.q_off = d_off;
    a.q_tid = d_tid;
    a.k1 = hb.k1;
    a.b = hb.b;
    a.tau = d_tau;
    a.tau_default = hb.tau_default;
    a.eps = hb.epsilon_guard;
    a.row_lo = hb.row_lo;
    a.row_hi = hb.row_hi == 0 ? X->dev.n_docs : std::min(hb.row_hi, X->dev.n_docs);
    a.flags = hb.flags;
    a.split = 1;
    a.nq_real = hb.n_queries;
    a.plan_tid = w->plan_tid;
    a.plan_mult = w->plan_mult;
    a.plan_len = w->plan_len;
    a.cost = w->cost;
    a.order = w->order;
    a.counters = w->counters;
    a.out_ids = out.ids;
    a.out_scores = out.scores;
    a.out_n = out.n;
    a.out_conf = out.conf;
    a.out_skip = out.skip;
    a.out_post = out.postings;
    return a;
}

// The wide path over queries d_qlist[0..n) of a planned batch: groups of G
// queries whose fp64 score rows fit a 1 GiB budget (kernels/wide.cu).
void run_wide(hm_index* X, Workspace* w, const hm::BatchArgs& a, const uint32_t* d_qlist, uint32_t n) {
    if (n == 0) return;
    cudaStream_t st = w->stream;
    const uint64_t span = a.row_hi > a.row_lo ? a.row_hi - a.row_lo : 0;
    const uint64_t k = std::max<uint32_t>(a.k, 1u);
    uint64_t G = 64;
    if (span) G = std::min<uint64_t>(G, std::max<uint64_t>(1, (1ull << 30) / (span * 8ull)));
    G = std::min<uint64_t>(G, std::max<uint64_t>(1, (256ull << 20) / (k * sizeof(hm::WideCand))));
    G = std::min<uint64_t>(G, n);
    const size_t sb = hm::wide_sort_bytes(G * k);
    if (G * span > w->wd_scores_cap || G > w->wd_g_cap || G * k > w->wd_cand_cap || sb > w->wd_sort_bytes) {
        ck(cudaStreamSynchronize(st), "sync");
        void* ps[] = {w->wd_scores, w->wd_hist, w->wd_st, w->wd_cand, w->wd_sort};
        for (void* p : ps)
            if (p) cudaFree(p);
        w->wd_scores = nullptr;
        w->wd_hist = nullptr;
        w->wd_st = nullptr;
        w->wd_cand = nullptr;
        w->wd_sort = nullptr;
        w->wd_scores_cap = std::max(G * span, w->wd_scores_cap);
        w->wd_g_cap = static_cast<uint32_t>(std::max<uint64_t>(G, w->wd_g_cap));
        w->wd_cand_cap = std::max(G * k, w->wd_cand_cap);
        w->wd_sort_bytes = std::max(sb, w->wd_sort_bytes);
        dalloc(w->wd_scores, w->wd_scores_cap);
        dalloc(w->wd_hist, w->wd_g_cap * 256ull);
        dalloc(w->wd_st, w->wd_g_cap);
        dalloc(w->wd_cand, w->wd_cand_cap);
        unsigned char* t = nullptr;
        dalloc(t, std::max<size_t>(w->wd_sort_bytes, 16));
        w->wd_sort = t;
    }
    for (uint64_t g0 = 0; g0 < n; g0 += G) {
        hm::WideArgs wa{};
        wa.G = static_cast<uint32_t>(std::min<uint64_t>(G, n - g0));
        wa.qlist = d_qlist + g0;
        wa.span = static_cast<uint32_t>(span);
        wa.scores = w->wd_scores;
        wa.hist = w->wd_hist;
        wa.st = w->wd_st;
        wa.cand = w->wd_cand;
        ck(hm::launch_wide_group(X->dev, a, wa, w->wd_sort, w->wd_sort_bytes, st), "wide path");
    }
    g_last_wide += n;
}

// A batch with k > kMaxK: plan, then every query on the wide path.
void run_wide_batch(hm_index* X, Workspace* w, const hm_query_batch& hb, const uint32_t* d_off, const uint32_t* d_tid,
                    const double* d_tau, const hm_results& out) {
    const uint32_t nq = hb.n_queries;
    cudaStream_t st = w->stream;
    if (nq > w->wd_iota_cap) {
        ck(cudaStreamSynchronize(st), "sync");
        if (w->wd_iota) cudaFree(w->wd_iota);
        w->wd_iota = nullptr;
        dalloc(w->wd_iota, nq);
        std::vector<uint32_t> io(nq);
        for (uint32_t i = 0; i < nq; ++i) io[i] = i;
        ck(cudaMemcpy(w->wd_iota, io.data(), nq * 4ull, cudaMemcpyHostToDevice), "iota");
        w->wd_iota_cap = nq;
    }
    hm::BatchArgs a = wide_args(X, w, hb, d_off, d_tid, d_tau, out);
    ck(cudaMemsetAsync(w->counters, 0, 16 * sizeof(uint32_t), st), "memset counters");
    ck(hm::launch_plan(X->dev, a, w->order_in, st), "plan kernel");
    g_last_launches = 1;
    g_last_graph = 0;
    g_last_seeded = false;
    g_last_split = 1;
    run_wide(X, w, a, w->wd_iota, nq);
}

// which queries of the last (synchronised) batch the seeded pass handed to
// the tile sweep: every query when the pass did not run
void save_handover(Workspace* w, uint32_t nq) {
    g_handover.assign(nq, 1u);
    if (g_last_seeded && g_last_split == 1)
        ck(cudaMemcpy(g_handover.data(), w->fb_list, nq * 4ull, cudaMemcpyDeviceToHost), "D2H hand-over");
}

void read_timing(Workspace* w) {
    ck(cudaEventSynchronize(w->ev[3]), "event sync");
    ck(cudaEventElapsedTime(&g_ms_plan, w->ev[0], w->ev[1]), "elapsed");
    ck(cudaEventElapsedTime(&g_ms_seed, w->ev[1], w->ev[4]), "elapsed");
    ck(cudaEventElapsedTime(&g_ms_search, w->ev[4], w->ev[2]), "elapsed");
    ck(cudaEventElapsedTime(&g_ms_exact, w->ev[2], w->ev[3]), "elapsed");
}

// Hold the baked postings for (k1, b) for the duration of a batch: shared
// lock while they match, exclusive re-bake (K0, ~1 ms at C2) when they do not.
// Returns false when these parameters cannot be baked (an impact outside the
// representable range): the batch then runs on the exact fp64 kernel.
bool ensure_baked(hm_index* X, double k1, double b, std::shared_lock<std::shared_mutex>& lk) {
    if (needs_exact(k1, b)) {
        lk = std::shared_lock<std::shared_mutex>(X->bake_mu);
        return false;
    }
    for (;;) {
        lk = std::shared_lock<std::shared_mutex>(X->bake_mu);
        if (X->bake_valid && X->bake_k1 == k1 && X->bake_b == b) return X->bake_ok;
        lk.unlock();
        std::unique_lock<std::shared_mutex> ul(X->bake_mu);
        if (X->bake_valid && X->bake_k1 == k1 && X->bake_b == b) continue;
        X->bake_valid = false;
        const uint32_t ks = hm::bake_ks(k1);
        cudaStream_t st = nullptr;
        ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "bake stream");
        uint32_t err = 0;
        try {
            ck(cudaMemsetAsync(X->d_bake_err, 0, 4, st), "bake memset");
            ck(cudaMemsetAsync(const_cast<float*>(X->dev.tmax), 0, std::max<uint64_t>(X->dev.n_terms, 1) * 4, st),
               "tmax memset");
            hm::DevIndex d = X->dev;
            ck(hm::launch_bake(d, X->d_long_terms, X->n_long, k1, b, ks, X->d_bk, X->d_bake_err, st),
               "bake kernel");
            ck(cudaMemcpyAsync(&err, X->d_bake_err, 4, cudaMemcpyDeviceToHost, st), "bake D2H");
            ck(cudaStreamSynchronize(st), "bake sync");
        } catch (...) {
            cudaStreamDestroy(st);
            throw;
        }
        cudaStreamDestroy(st);
        X->dev.bk_ks = ks;
        X->bake_k1 = k1;
        X->bake_b = b;
        X->bake_ok = err == 0;
        X->bake_valid = true;
    }
}

void validate(const hm_index* X, const hm_query_batch* b) {
    if (!b) throw std::invalid_argument("null batch");
    if (b->n_queries && (!b->q_off)) throw std::invalid_argument("q_off is required");
    (void)X;
}

// the batch's longest query (raw term count): plans longer than kMaxTerms
// distinct terms are only possible above it
uint32_t max_query_len(const uint32_t* q_off, uint32_t nq) {
    uint32_t m = 0;
    for (uint32_t i = 0; i < nq; ++i) m = std::max(m, q_off[i + 1] - q_off[i]);
    return m;
}

}  // namespace

namespace hm_host {
std::string& error_slot() {
    thread_local std::string s;
    return s;
}
}  // namespace hm_host

extern "C" {

const char* hm_last_error(void) { return hm_host::error_slot().c_str(); }

int hm_index_create(const hm_csr_view* view, int device, hm_index** out) {
    return guard([&] {
        if (!view || !out) throw std::invalid_argument("null argument");
        use_device(device);
        auto* X = new hm_index();
        X->device = device;
        try {
            build_index(view, X);
        } catch (...) {
            delete X;
            throw;
        }
        *out = X;
    });
}

int hm_index_destroy(hm_index* index) {
    return guard([&] { delete index; });
}

uint64_t hm_index_device_bytes(const hm_index* index) { return index ? index->bytes : 0; }

int hm_index_format(const hm_index* X, uint32_t* row_bits, uint32_t* code_bits, uint32_t* n_codes,
                    uint64_t* n_escaped) {
    return guard([&] {
        if (!X) throw std::invalid_argument("null index");
        if (row_bits) *row_bits = X->row_bits;
        if (code_bits) *code_bits = X->code_bits;
        if (n_codes) *n_codes = X->n_codes;
        if (n_escaped) *n_escaped = X->n_escaped;
    });
}

}  // extern "C"

namespace {

// The host-buffer batch (hm_search_batch), or with n_parts > 0 the batch
// searched inside each of the parts [part_row[p], part_row[p+1]) separately
// (hm_search_batch_parts): outputs [n_parts][n_queries][k], no conf / skip.
void search_host(hm_index* X, const hm_query_batch* b, hm_results* out, uint32_t n_parts,
                 const uint32_t* part_row) {
    {
        if (!X || !out) throw std::invalid_argument("null argument");
        validate(X, b);
        const uint32_t nq = b->n_queries;
        if (nq == 0) return;
        if (b->ext_bound || b->out_bound || (b->flags & HM_FLAG_BOUND_ONLY))
            throw std::invalid_argument("shard bounds (ext_bound / out_bound) are for hm_search_batch_device");
        if (!out->ids || !out->scores || !out->n) throw std::invalid_argument("null result buffer");
        const uint32_t ntid = b->q_off[nq];
        for (uint32_t i = 0; i < nq; ++i)
            if (b->q_off[i + 1] < b->q_off[i]) throw std::invalid_argument("q_off not monotone");
        if (ntid && !b->q_tid) throw std::invalid_argument("q_tid is required");
        for (uint32_t i = 0; i < ntid; ++i)
            if (b->q_tid[i] != hm::kNoTerm && b->q_tid[i] >= X->dev.n_terms)
                throw std::out_of_range("term id out of range");
        ck(cudaSetDevice(X->device), "cudaSetDevice");
        // k > 256: the wide path for the whole batch; queries longer than 256
        // terms: no row slabs, and the ones whose plans exceed 256 distinct
        // terms are served by the wide path after the batch
        const bool wide_all = b->k > static_cast<uint32_t>(hm::kMaxK);
        const bool long_any = max_query_len(b->q_off, nq) > static_cast<uint32_t>(hm::kMaxTerms);
        if (n_parts) {
            if (!part_row) throw std::invalid_argument("part_row is required");
            for (uint32_t p = 0; p < n_parts; ++p)
                if (part_row[p + 1] < part_row[p]) throw std::invalid_argument("part_row not ascending");
            if (part_row[n_parts] > X->dev.n_docs) throw std::out_of_range("part_row beyond the index's rows");
            const uint64_t kk = b->k;
            if (wide_all || long_any || part_row[n_parts] == part_row[0]) {  // part by part
                uint32_t wide = 0;
                for (uint32_t p = 0; p < n_parts; ++p) {
                    const uint64_t o = static_cast<uint64_t>(p) * nq;
                    hm_results r{out->ids + o * kk, out->scores + o * kk, out->n + o, nullptr, nullptr,
                                 out->postings ? out->postings + o : nullptr};
                    if (part_row[p] == part_row[p + 1]) {  // (row_hi = 0 would mean "every row")
                        std::fill(r.n, r.n + nq, 0u);
                        if (r.postings) std::fill(r.postings, r.postings + nq, 0ull);
                        continue;
                    }
                    hm_query_batch hb = *b;
                    hb.row_lo = part_row[p];
                    hb.row_hi = part_row[p + 1];
                    search_host(X, &hb, &r, 0, nullptr);
                    wide += g_last_wide;
                }
                g_last_wide = wide;
                return;
            }
        }
        const uint32_t nv = nq * std::max(n_parts, 1u);  // result rows
        g_last_wide = 0;
        std::shared_lock<std::shared_mutex> bake_lk;
        const bool baked = wide_all ? false : ensure_baked(X, b->k1, b->b, bake_lk);
        Workspace* w = acquire(X);
        try {
            const uint32_t k = std::max(b->k, 1u);
            hm_query_batch hb = *b;
            if (!baked) hb.flags |= HM_FLAG_FORCE_EXACT;
            if (long_any) hb.flags |= HM_FLAG_NO_SPLIT;
            if (n_parts) {
                hb.row_lo = part_row[0];
                hb.row_hi = part_row[n_parts];
            }
            ensure(w, n_parts ? nv : nq * (wide_all ? 1 : split_for(X, hb)), std::max(ntid, 1u), k, true);
            unsigned char* p = w->pin;
            auto take = [&](size_t bytes) {
                unsigned char* r = p;
                p += (bytes + 15) & ~size_t(15);
                return r;
            };
            float* pw = reinterpret_cast<float*>(take(hm::kMaxCodes * 4));
            uint32_t* poff = reinterpret_cast<uint32_t*>(take((nq + 1ull) * 4));
            uint32_t* ptid = reinterpret_cast<uint32_t*>(take(ntid * 4ull));
            double* ptau = reinterpret_cast<double*>(take(nq * 8ull));
            uint64_t* rids = reinterpret_cast<uint64_t*>(take(static_cast<size_t>(nv) * k * 8));
            double* rsc = reinterpret_cast<double*>(take(static_cast<size_t>(nv) * k * 8));
            uint32_t* rn = reinterpret_cast<uint32_t*>(take(nv * 4ull));
            double* rconf = reinterpret_cast<double*>(take(nq * 8ull));
            uint8_t* rskip = take(nq);
            uint64_t* rpost = reinterpret_cast<uint64_t*>(take(nv * 8ull));
            uint32_t* rcnt = reinterpret_cast<uint32_t*>(take(32));
            uint32_t* prow = reinterpret_cast<uint32_t*>(take((n_parts + 1ull) * 4));
            std::memcpy(poff, b->q_off, (nq + 1ull) * 4);
            if (ntid) std::memcpy(ptid, b->q_tid, ntid * 4ull);
            if (b->tau) std::memcpy(ptau, b->tau, nq * 8ull);
            cudaStream_t st = w->stream;
            ck(cudaMemcpyAsync(w->q_off, poff, (nq + 1ull) * 4, cudaMemcpyHostToDevice, st), "H2D");
            if (ntid) ck(cudaMemcpyAsync(w->q_tid, ptid, ntid * 4ull, cudaMemcpyHostToDevice, st), "H2D");
            if (b->tau) ck(cudaMemcpyAsync(w->tau, ptau, nq * 8ull, cudaMemcpyHostToDevice, st), "H2D");
            hm_results dout{w->out_ids, w->out_scores, w->out_n, w->out_conf, w->out_skip, w->out_post};
            // the k used on device must match the output stride
            if (n_parts) {  // every part a slab of each query, lists left in v_*
                if (n_parts + 1 > w->slab_cap) {
                    ck(cudaStreamSynchronize(st), "sync");
                    if (w->slab_row) cudaFree(w->slab_row);
                    w->slab_row = nullptr;
                    dalloc(w->slab_row, n_parts + 1ull);
                    w->slab_cap = n_parts + 1;
                }
                std::memcpy(prow, part_row, (n_parts + 1ull) * 4);
                ck(cudaMemcpyAsync(w->slab_row, prow, (n_parts + 1ull) * 4, cudaMemcpyHostToDevice, st), "H2D");
                run_batch(X, w, hb, w->q_off, w->q_tid, nullptr, dout, pw, n_parts, w->slab_row);
                dout = hm_results{w->v_ids, w->v_scores, w->v_n, nullptr, nullptr, w->v_post};
            } else if (wide_all) {
                run_wide_batch(X, w, hb, w->q_off, w->q_tid, b->tau ? w->tau : nullptr, dout);
            } else {
                run_batch(X, w, hb, w->q_off, w->q_tid, b->tau ? w->tau : nullptr, dout, pw);
                if (long_any) {  // plans beyond 256 distinct terms: the wide path
                    ck(cudaMemcpyAsync(rcnt, w->counters, 32, cudaMemcpyDeviceToHost, st), "D2H");
                    ck(cudaStreamSynchronize(st), "batch");
                    if (b->flags & HM_FLAG_TIMING) read_timing(w);
                    run_wide(X, w, wide_args(X, w, hb, w->q_off, w->q_tid, b->tau ? w->tau : nullptr, dout),
                             w->wide_list, rcnt[6]);
                }
            }
            const size_t kk = b->k;
            if (kk) {
                ck(cudaMemcpyAsync(rids, dout.ids, nv * kk * 8, cudaMemcpyDeviceToHost, st), "D2H");
                ck(cudaMemcpyAsync(rsc, dout.scores, nv * kk * 8, cudaMemcpyDeviceToHost, st), "D2H");
            }
            ck(cudaMemcpyAsync(rn, dout.n, nv * 4ull, cudaMemcpyDeviceToHost, st), "D2H");
            if (!n_parts) {
                ck(cudaMemcpyAsync(rconf, dout.conf, nq * 8ull, cudaMemcpyDeviceToHost, st), "D2H");
                ck(cudaMemcpyAsync(rskip, dout.skip, nq, cudaMemcpyDeviceToHost, st), "D2H");
            }
            ck(cudaMemcpyAsync(rpost, dout.postings, nv * 8ull, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaMemcpyAsync(rcnt, w->counters, 32, cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaStreamSynchronize(st), "batch");
            if ((b->flags & HM_FLAG_TIMING) && !wide_all && !long_any) read_timing(w);
            g_last_exact = rcnt[1];
            g_last_handed = rcnt[4];
            if ((b->flags & HM_FLAG_TIMING) && !n_parts) save_handover(w, nq);
            if (rcnt[3] & hm::kErrTooManyTerms)
                throw std::invalid_argument("a query has more than 256 distinct terms");
            if (rcnt[3] & 2u) throw std::runtime_error("exact kernel failed to converge");
            for (uint32_t i = 0; i < nv; ++i) {
                out->n[i] = rn[i];
                for (uint32_t j = 0; j < rn[i]; ++j) {
                    out->ids[i * kk + j] = rids[i * kk + j];
                    out->scores[i * kk + j] = rsc[i * kk + j];
                }
            }
            if (out->conf && !n_parts) std::memcpy(out->conf, rconf, nq * 8ull);
            if (out->skip && !n_parts) std::memcpy(out->skip, rskip, nq);
            if (out->postings) std::memcpy(out->postings, rpost, nv * 8ull);
        } catch (...) {
            cudaStreamSynchronize(w->stream);
            release(X, w);
            throw;
        }
        release(X, w);
    }
}

}  // namespace

extern "C" {

int hm_search_batch(hm_index* X, const hm_query_batch* b, hm_results* out) {
    return guard([&] { search_host(X, b, out, 0, nullptr); });
}

int hm_search_batch_parts(hm_index* X, const hm_query_batch* b, uint32_t n_parts, const uint32_t* part_row,
                          hm_results* out) {
    return guard([&] {
        if (n_parts == 0) throw std::invalid_argument("n_parts must be >= 1");
        search_host(X, b, out, n_parts, part_row);
    });
}

int hm_search_batch_device(hm_index* X, const hm_query_batch* b, hm_results* out, void* stream) {
    return guard([&] {
        if (!X || !out) throw std::invalid_argument("null argument");
        validate(X, b);
        const uint32_t nq = b->n_queries;
        if (nq == 0) return;
        ck(cudaSetDevice(X->device), "cudaSetDevice");
        // the batch's tid count is unknown on the host: plan scratch is sized
        // from q_off[nq] read back once (a 4-byte D2H on the caller's stream)
        cudaStream_t ust = static_cast<cudaStream_t>(stream);
        // (q_off is read back whole: a query longer than kMaxTerms terms
        // disables row slabs and may need the wide path)
        std::vector<uint32_t> hoff(nq + 1ull);
        ck(cudaMemcpyAsync(hoff.data(), b->q_off, (nq + 1ull) * 4, cudaMemcpyDeviceToHost, ust), "D2H q_off");
        ck(cudaStreamSynchronize(ust), "sync");
        const uint32_t ntid = hoff[nq];
        const bool wide_all = b->k > static_cast<uint32_t>(hm::kMaxK);
        const bool bonly = (b->flags & HM_FLAG_BOUND_ONLY) != 0;
        if (bonly && !b->out_bound) throw std::invalid_argument("HM_FLAG_BOUND_ONLY needs out_bound");
        if (bonly && wide_all) {  // the wide path has no bound: none reported
            ck(cudaMemsetAsync(b->out_bound, 0, static_cast<uint64_t>(nq) * b->k * sizeof(float), ust),
               "memset bounds");
            return;
        }
        const bool long_any = max_query_len(hoff.data(), nq) > static_cast<uint32_t>(hm::kMaxTerms);
        g_last_wide = 0;
        std::shared_lock<std::shared_mutex> bake_lk;
        const bool baked = wide_all ? false : ensure_baked(X, b->k1, b->b, bake_lk);
        Workspace* w = acquire(X);
        try {
            hm_query_batch hb = *b;
            if (!baked) hb.flags |= HM_FLAG_FORCE_EXACT;
            if (long_any) hb.flags |= HM_FLAG_NO_SPLIT;
            ensure(w, nq * (wide_all ? 1 : split_for(X, hb)), std::max(ntid, 1u), std::max(b->k, 1u), false);
            // order the workspace stream after the caller's stream and back
            cudaEvent_t ev;
            ck(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
            ck(cudaEventRecord(ev, ust), "event record");
            ck(cudaStreamWaitEvent(w->stream, ev, 0), "wait");
            if (wide_all) {
                run_wide_batch(X, w, hb, b->q_off, b->q_tid, b->tau, *out);
            } else {
                run_batch(X, w, hb, b->q_off, b->q_tid, b->tau, *out, reinterpret_cast<float*>(w->pin));
                if (long_any && !bonly) {
                    uint32_t* rc = reinterpret_cast<uint32_t*>(w->pin) + hm::kMaxCodes;
                    ck(cudaMemcpyAsync(rc, w->counters, 32, cudaMemcpyDeviceToHost, w->stream), "D2H counters");
                    ck(cudaStreamSynchronize(w->stream), "sync");
                    run_wide(X, w, wide_args(X, w, hb, b->q_off, b->q_tid, b->tau, *out), w->wide_list, rc[6]);
                }
            }
            ck(cudaEventRecord(ev, w->stream), "event record");
            ck(cudaStreamWaitEvent(ust, ev, 0), "wait");
            if (b->flags & HM_FLAG_TIMING) {  // plus the batch counters (32 B D2H)
                uint32_t* rc = reinterpret_cast<uint32_t*>(w->pin) + hm::kMaxCodes;
                ck(cudaMemcpyAsync(rc, w->counters, 32, cudaMemcpyDeviceToHost, w->stream), "D2H counters");
                ck(cudaStreamSynchronize(w->stream), "sync");
                g_last_exact = rc[1];
                g_last_handed = rc[4];
                save_handover(w, nq);
            }
            // pinned w32 staging is reused by the next call on this workspace:
            // make sure the async upload finished before handing it back
            ck(cudaStreamSynchronize(w->stream), "sync");
            if ((b->flags & HM_FLAG_TIMING) && !wide_all) read_timing(w);
            cudaEventDestroy(ev);
        } catch (...) {
            cudaStreamSynchronize(w->stream);
            release(X, w);
            throw;
        }
        release(X, w);
    });
}

int hm_last_batch_stats(uint32_t* n_exact, uint32_t* n_launches) {
    if (n_exact) *n_exact = g_last_exact;
    if (n_launches) *n_launches = g_last_launches;
    return HM_OK;
}

int hm_last_batch_handover(uint32_t* flags, uint32_t n) {
    const uint32_t m = std::min<uint32_t>(n, static_cast<uint32_t>(g_handover.size()));
    for (uint32_t i = 0; i < m; ++i) flags[i] = g_handover[i] ? 1u : 0u;
    return m == n ? HM_OK : HM_ERR_RANGE;
}

int hm_last_batch_wide(uint32_t* n_wide) {
    if (n_wide) *n_wide = g_last_wide;
    return HM_OK;
}

int hm_last_batch_graph(uint32_t* mode) {
    if (mode) *mode = g_last_graph;
    return HM_OK;
}

int hm_last_batch_seed(float* ms_seed, uint32_t* n_handed_over) {
    if (ms_seed) *ms_seed = g_ms_seed;
    if (n_handed_over) *n_handed_over = g_last_handed;
    return HM_OK;
}

int hm_last_batch_timing(float* ms_plan, float* ms_search, float* ms_exact) {
    if (ms_plan) *ms_plan = g_ms_plan;
    if (ms_search) *ms_search = g_ms_search;
    if (ms_exact) *ms_exact = g_ms_exact;
    return HM_OK;
}

int hm_merge_shards_device(uint32_t G, uint32_t nq, uint32_t k, const uint64_t* ids,
                           const double* scores, const uint32_t* n, const double* tau,
                           double tau_default, double eps, hm_results* out, void* stream) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null result");
        if (static_cast<uint64_t>(G) * k > 2048)
            throw std::invalid_argument("n_shards * k must be <= 2048");
        ck(hm::launch_merge(G, nq, k, ids, scores, n, tau, tau_default, eps, out->ids, out->scores,
                            out->n, out->conf, out->skip, static_cast<cudaStream_t>(stream)),
           "merge kernel");
    });
}

double hm_margin(const double* s, uint32_t n, double eps) {
    if (n == 0 || s[0] <= 0.0) return 0.0;  // src/cascade.cpp:14
    if (n < 2) return 0.0;
    return (s[0] - s[1]) / std::max(s[0], eps);
}

}  // extern "C"
