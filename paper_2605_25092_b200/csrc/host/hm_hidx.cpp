// HIDX v1 container reader (include/hm_b200.h: hm_hidx_*): the reference's
// on-disk index (proj/src/io.cpp:91-157 write/read_index_body, :223-232
// save/load_index) parsed straight into the flat arrays hm_index_create
// uploads -- no std::unordered_map vocabulary or per-element stream reads.
// Little-endian fixed-width fields; the same validation and messages as the
// reference reader (bad magic, version, idf convention, truncation), so a
// `hybridmem search --index file.hidx` index feeds the GPU without a rebuild.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <unordered_map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "hm_b200.h"

struct hm_hidx {
    uint8_t mode = 0, tok_mode = 0;
    double build_k1 = 0.0, build_b = 0.0, avgdl = 0.0;
    uint32_t n_terms = 0, n_docs = 0;
    uint64_t n_postings = 0;
    std::vector<char> term_chars;        // all term strings, back to back
    std::vector<uint64_t> term_start;    // [n_terms + 1] offsets into term_chars
    std::vector<uint64_t> term_offsets;  // [n_terms + 1]
    std::vector<uint32_t> posting_rows;
    std::vector<double> posting_weights;
    std::vector<double> term_idfs, term_maxscores, term_order_keys;
    std::vector<uint32_t> doc_lens;
    std::vector<uint64_t> doc_ids;
};

// HTIX v1 (io.cpp:234-318) assembled as ONE flat index whose rows are laid
// out partition by partition (oldest first) -- the layout the framework's
// temporal path scores with a row window -- over the shared statistics
// (the flat corpus's idf / order keys / avgdl, temporal_index.cpp:136-142).
struct hm_htix {
    hm_hidx flat;                        // the assembled index (terms = the shared vocabulary)
    std::vector<uint32_t> part_row;      // [K + 1] first row of every partition
    std::vector<int64_t> win_start, win_end;
    int64_t window_ms = 0;
    double epsilon = 0.0, lambda_hat = 0.0;
    uint32_t k_max = 0;
    uint64_t total_docs = 0;
};

namespace {

thread_local std::string g_hidx_err;

// little-endian field readers over a file or an in-memory blob (HTIX partitions)
template <typename Derived>
struct Reader {
    template <typename T>
    T get(const char* what) {  // little-endian host (x86-64 / aarch64)
        T v;
        static_cast<Derived*>(this)->raw(&v, sizeof(T), what);
        return v;
    }
    template <typename T>
    void vec(std::vector<T>& v, uint64_t n, const char* what) {
        v.resize(n);
        static_cast<Derived*>(this)->raw(v.data(), n * sizeof(T), what);
    }
    std::string str(const char* what) {
        const uint32_t n = get<uint32_t>(what);
        std::string s(n, '\0');
        static_cast<Derived*>(this)->raw(&s[0], n, what);
        return s;
    }
};

[[noreturn]] void truncated(const char* what) {
    throw std::runtime_error(std::string("index file truncated reading ") + what);
}

struct File : Reader<File> {
    std::FILE* f;
    explicit File(const char* path) : f(std::fopen(path, "rb")) {
        if (!f) throw std::runtime_error(std::string("cannot open ") + path);
    }
    ~File() { std::fclose(f); }
    void raw(void* dst, size_t n, const char* what) {
        if (n && std::fread(dst, 1, n, f) != n) truncated(what);
    }
    int peek4(char* m) { return static_cast<int>(std::fread(m, 1, 4, f)); }
};

struct Mem : Reader<Mem> {
    const char* p;
    size_t n, off = 0;
    Mem(const char* p_, size_t n_) : p(p_), n(n_) {}
    void raw(void* dst, size_t k, const char* what) {
        if (k > n - off) truncated(what);
        std::memcpy(dst, p + off, k);
        off += k;
    }
    int peek4(char* m) {
        const size_t k = std::min<size_t>(4, n - off);
        std::memcpy(m, p + off, k);
        off += k;
        return static_cast<int>(k);
    }
};

// HIDX v1 body (io.cpp:114-157)
template <typename R>
void read_body(R& in, hm_hidx& h_) {
    hm_hidx* h = &h_;
    char magic[4] = {0, 0, 0, 0};
    if (in.peek4(magic) != 4 || std::memcmp(magic, "HIDX", 4) != 0)
        throw std::runtime_error("not an index file (bad magic)");
    const uint32_t version = in.template get<uint32_t>("version");
    if (version != 1) throw std::runtime_error("unsupported index version " + std::to_string(version));
    h->mode = in.template get<uint8_t>("mode");
    h->tok_mode = in.template get<uint8_t>("tokenizer mode");
    h->build_k1 = in.template get<double>("k1");
    h->build_b = in.template get<double>("b");
    const std::string conv = in.str("idf convention");
    if (conv != "lucene_ln1p") throw std::runtime_error("unsupported idf convention: " + conv);
    h->avgdl = in.template get<double>("avgdl");
    h->n_terms = in.template get<uint32_t>("term count");
    h->n_docs = in.template get<uint32_t>("doc count");
    h->n_postings = in.template get<uint64_t>("posting count");
    h->term_start.resize(static_cast<size_t>(h->n_terms) + 1);
    h->term_start[0] = 0;
    for (uint32_t i = 0; i < h->n_terms; ++i) {
        const uint32_t n = in.template get<uint32_t>("term");
        const size_t at = h->term_chars.size();
        h->term_chars.resize(at + n);
        in.raw(h->term_chars.data() + at, n, "term");
        h->term_start[i + 1] = at + n;
    }
    in.vec(h->term_offsets, static_cast<uint64_t>(h->n_terms) + 1, "term offsets");
    in.vec(h->posting_rows, h->n_postings, "posting rows");
    in.vec(h->posting_weights, h->n_postings, "posting weights");
    in.vec(h->term_idfs, h->n_terms, "idfs");
    in.vec(h->term_maxscores, h->n_terms, "maxscores");
    in.vec(h->term_order_keys, h->n_terms, "order keys");
    in.vec(h->doc_lens, h->n_docs, "doc lens");
    in.vec(h->doc_ids, h->n_docs, "doc ids");
    if (h->term_offsets.back() != h->n_postings)
        throw std::runtime_error("index file inconsistent: term offsets do not end at the posting count");
}

}  // namespace

extern "C" {

int hm_hidx_load(const char* path, hm_hidx** out) {
    try {
        if (!path || !out) throw std::invalid_argument("null argument");
        File in(path);
        auto h = std::make_unique<hm_hidx>();
        read_body(in, *h);
        *out = h.release();
        return HM_OK;
    } catch (const std::invalid_argument& e) {
        g_hidx_err = e.what();
        return HM_ERR_INVALID;
    } catch (const std::exception& e) {
        g_hidx_err = e.what();
        return HM_ERR_RUNTIME;
    }
}

int hm_htix_load(const char* path, hm_htix** out) {
    try {
        if (!path || !out) throw std::invalid_argument("null argument");
        File in(path);
        char magic[4] = {0, 0, 0, 0};
        if (in.peek4(magic) != 4 || std::memcmp(magic, "HTIX", 4) != 0)
            throw std::runtime_error("not a temporal index file (bad magic)");
        const uint32_t version = in.get<uint32_t>("version");
        if (version != 1) throw std::runtime_error("unsupported temporal index version " + std::to_string(version));
        auto t = std::make_unique<hm_htix>();
        t->window_ms = in.get<int64_t>("window");
        t->epsilon = in.get<double>("epsilon");
        t->lambda_hat = in.get<double>("lambda");
        t->k_max = in.get<uint32_t>("k_max");
        t->total_docs = in.get<uint64_t>("total docs");
        hm_hidx& f = t->flat;
        f.avgdl = in.get<double>("avgdl");
        // the shared vocabulary: the idf map's keys (written in sorted order)
        std::unordered_map<std::string, uint32_t> tid;
        const uint64_t n_idf = in.get<uint64_t>("idf count");
        f.term_start.assign(1, 0);
        for (uint64_t i = 0; i < n_idf; ++i) {
            const std::string term = in.str("idf term");
            const double v = in.get<double>("idf value");
            auto it = tid.emplace(term, static_cast<uint32_t>(f.term_idfs.size()));
            if (!it.second) {  // a repeated key overwrites, as std::map assignment does
                f.term_idfs[it.first->second] = v;
                continue;
            }
            f.term_chars.insert(f.term_chars.end(), term.begin(), term.end());
            f.term_start.push_back(f.term_chars.size());
            f.term_idfs.push_back(v);
        }
        f.n_terms = static_cast<uint32_t>(f.term_idfs.size());
        f.term_order_keys.assign(f.n_terms, 0.0);
        f.term_maxscores.assign(f.n_terms, 0.0);
        const uint64_t n_ord = in.get<uint64_t>("order-key count");
        for (uint64_t i = 0; i < n_ord; ++i) {
            const std::string term = in.str("order-key term");
            const double v = in.get<double>("order-key value");
            auto it = tid.find(term);
            if (it != tid.end()) f.term_order_keys[it->second] = v;
        }
        const uint32_t K = in.get<uint32_t>("partition count");
        std::vector<uint64_t> size(K);
        t->win_start.resize(K);
        t->win_end.resize(K);
        for (uint32_t p = 0; p < K; ++p) {
            t->win_start[p] = in.get<int64_t>("window start");
            t->win_end[p] = in.get<int64_t>("window end");
            size[p] = in.get<uint64_t>("partition size");
        }
        // partitions in order; postings of every shared term concatenated
        std::vector<hm_hidx> parts(K);
        std::vector<char> blob;
        for (uint32_t p = 0; p < K; ++p) {
            blob.resize(size[p]);
            if (size[p] && std::fread(blob.data(), 1, size[p], in.f) != size[p]) truncated("partition blob");
            Mem m(blob.data(), blob.size());
            read_body(m, parts[p]);
        }
        t->part_row.assign(1, 0);
        std::vector<uint64_t> cnt(static_cast<size_t>(f.n_terms) + 1, 0);
        std::vector<std::vector<uint32_t>> local_to_global(K);
        for (uint32_t p = 0; p < K; ++p) {
            const hm_hidx& q = parts[p];
            t->part_row.push_back(t->part_row.back() + q.n_docs);
            local_to_global[p].resize(q.n_terms);
            for (uint32_t lt = 0; lt < q.n_terms; ++lt) {
                const std::string term(q.term_chars.data() + q.term_start[lt], q.term_start[lt + 1] - q.term_start[lt]);
                auto it = tid.find(term);
                if (it == tid.end())
                    throw std::runtime_error("temporal index inconsistent: partition term missing from the shared statistics");
                local_to_global[p][lt] = it->second;
                cnt[it->second + 1] += q.term_offsets[lt + 1] - q.term_offsets[lt];
            }
        }
        f.term_offsets.resize(static_cast<size_t>(f.n_terms) + 1);
        for (uint32_t g = 0; g < f.n_terms; ++g) cnt[g + 1] += cnt[g];
        f.term_offsets.assign(cnt.begin(), cnt.end());
        f.n_postings = f.term_offsets.back();
        f.posting_rows.resize(f.n_postings);
        f.posting_weights.resize(f.n_postings);
        std::vector<uint64_t> fill(f.term_offsets.begin(), f.term_offsets.end() - 1);
        for (uint32_t p = 0; p < K; ++p) {
            const hm_hidx& q = parts[p];
            const uint32_t base = t->part_row[p];
            for (uint32_t lt = 0; lt < q.n_terms; ++lt) {
                const uint32_t g = local_to_global[p][lt];
                for (uint64_t i = q.term_offsets[lt]; i < q.term_offsets[lt + 1]; ++i) {
                    f.posting_rows[fill[g]] = base + q.posting_rows[i];
                    f.posting_weights[fill[g]] = q.posting_weights[i];
                    ++fill[g];
                }
            }
            f.doc_lens.insert(f.doc_lens.end(), q.doc_lens.begin(), q.doc_lens.end());
            f.doc_ids.insert(f.doc_ids.end(), q.doc_ids.begin(), q.doc_ids.end());
            if (p == 0) {
                f.mode = q.mode;
                f.tok_mode = q.tok_mode;
                f.build_k1 = q.build_k1;
                f.build_b = q.build_b;
            }
        }
        f.n_docs = t->part_row.back();
        *out = t.release();
        return HM_OK;
    } catch (const std::invalid_argument& e) {
        g_hidx_err = e.what();
        return HM_ERR_INVALID;
    } catch (const std::exception& e) {
        g_hidx_err = e.what();
        return HM_ERR_RUNTIME;
    }
}

const hm_hidx* hm_htix_flat(const hm_htix* t) { return t ? &t->flat : nullptr; }

int hm_htix_partitions(const hm_htix* t, uint32_t* n_partitions, const uint32_t** part_row,
                       const int64_t** window_start, const int64_t** window_end) {
    if (!t) return HM_ERR_INVALID;
    if (n_partitions) *n_partitions = static_cast<uint32_t>(t->win_start.size());
    if (part_row) *part_row = t->part_row.data();
    if (window_start) *window_start = t->win_start.data();
    if (window_end) *window_end = t->win_end.data();
    return HM_OK;
}

int hm_htix_params(const hm_htix* t, int64_t* window_ms, double* epsilon, double* lambda_hat,
                   uint32_t* k_max, uint64_t* total_docs) {
    if (!t) return HM_ERR_INVALID;
    if (window_ms) *window_ms = t->window_ms;
    if (epsilon) *epsilon = t->epsilon;
    if (lambda_hat) *lambda_hat = t->lambda_hat;
    if (k_max) *k_max = t->k_max;
    if (total_docs) *total_docs = t->total_docs;
    return HM_OK;
}

void hm_htix_free(hm_htix* t) { delete t; }

const char* hm_hidx_last_error(void) { return g_hidx_err.c_str(); }

int hm_hidx_view(const hm_hidx* h, hm_csr_view* v, uint32_t* mode, double* build_k1, double* build_b) {
    if (!h || !v) return HM_ERR_INVALID;
    v->n_terms = h->n_terms;
    v->term_offsets = h->term_offsets.data();
    v->posting_rows = h->posting_rows.data();
    v->posting_weights = h->posting_weights.data();
    v->posting_tf = nullptr;
    v->term_idfs = h->term_idfs.data();
    v->term_order_keys = h->term_order_keys.data();
    v->n_docs = h->n_docs;
    v->doc_lens = h->doc_lens.data();
    v->doc_ids = h->doc_ids.data();
    v->avgdl = h->avgdl;
    if (mode) *mode = h->mode;
    if (build_k1) *build_k1 = h->build_k1;
    if (build_b) *build_b = h->build_b;
    return HM_OK;
}

uint32_t hm_hidx_term(const hm_hidx* h, uint32_t tid, const char** s) {
    if (!h || tid >= h->n_terms) {
        if (s) *s = nullptr;
        return 0;
    }
    if (s) *s = h->term_chars.data() + h->term_start[tid];
    return static_cast<uint32_t>(h->term_start[tid + 1] - h->term_start[tid]);
}

const double* hm_hidx_maxscores(const hm_hidx* h) { return h ? h->term_maxscores.data() : nullptr; }

void hm_hidx_free(hm_hidx* h) { delete h; }

}  // extern "C"
