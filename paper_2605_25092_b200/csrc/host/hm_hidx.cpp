// HIDX v1 container reader (include/hm_b200.h: hm_hidx_*): the reference's
// on-disk index (proj/src/io.cpp:91-157 write/read_index_body, :223-232
// save/load_index) parsed straight into the flat arrays hm_index_create
// uploads -- no std::unordered_map vocabulary or per-element stream reads.
// Little-endian fixed-width fields; the same validation and messages as the
// reference reader (bad magic, version, idf convention, truncation), so a
// `hybridmem search --index file.hidx` index feeds the GPU without a rebuild.
#include <cstdio>
#include <cstring>
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

namespace {

thread_local std::string g_hidx_err;

struct File {
    std::FILE* f;
    explicit File(const char* path) : f(std::fopen(path, "rb")) {
        if (!f) throw std::runtime_error(std::string("cannot open ") + path);
    }
    ~File() { std::fclose(f); }
    void raw(void* dst, size_t n, const char* what) {
        if (n && std::fread(dst, 1, n, f) != n)
            throw std::runtime_error(std::string("index file truncated reading ") + what);
    }
    template <typename T>
    T get(const char* what) {  // little-endian host (x86-64 / aarch64)
        T v;
        raw(&v, sizeof(T), what);
        return v;
    }
    template <typename T>
    void vec(std::vector<T>& v, uint64_t n, const char* what) {
        v.resize(n);
        raw(v.data(), n * sizeof(T), what);
    }
    std::string str(const char* what) {
        const uint32_t n = get<uint32_t>(what);
        std::string s(n, '\0');
        raw(&s[0], n, what);
        return s;
    }
};

}  // namespace

extern "C" {

int hm_hidx_load(const char* path, hm_hidx** out) {
    try {
        if (!path || !out) throw std::invalid_argument("null argument");
        File in(path);
        char magic[4] = {0, 0, 0, 0};
        if (std::fread(magic, 1, 4, in.f) != 4 || std::memcmp(magic, "HIDX", 4) != 0)
            throw std::runtime_error("not an index file (bad magic)");
        const uint32_t version = in.get<uint32_t>("version");
        if (version != 1) throw std::runtime_error("unsupported index version " + std::to_string(version));
        auto h = std::make_unique<hm_hidx>();
        h->mode = in.get<uint8_t>("mode");
        h->tok_mode = in.get<uint8_t>("tokenizer mode");
        h->build_k1 = in.get<double>("k1");
        h->build_b = in.get<double>("b");
        const std::string conv = in.str("idf convention");
        if (conv != "lucene_ln1p") throw std::runtime_error("unsupported idf convention: " + conv);
        h->avgdl = in.get<double>("avgdl");
        h->n_terms = in.get<uint32_t>("term count");
        h->n_docs = in.get<uint32_t>("doc count");
        h->n_postings = in.get<uint64_t>("posting count");
        h->term_start.resize(static_cast<size_t>(h->n_terms) + 1);
        h->term_start[0] = 0;
        for (uint32_t i = 0; i < h->n_terms; ++i) {
            const uint32_t n = in.get<uint32_t>("term");
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
