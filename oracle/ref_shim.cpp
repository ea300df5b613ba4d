// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A thin extern "C" shim over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled from where the sources lie by
// oracle/Makefile into oracle/_ref/libhybridref.so).  Only tests/, smoke() and
// bench.py's cpu_baseline / --impl reference leg load it.  It exposes:
//   * the reference generators   gen_corpus / gen_queries   (workload.cpp:47-135)
//   * the reference index build  build_index                (csr_index.cpp:232-324)
//   * the reference searches     CsrIndex::bm25_topk        (csr_index.cpp:77-104)
//                                CsrIndex::bm25_topk_maxscore (csr_index.cpp:106-207)
//                                TemporalIndex::topk        (temporal_index.cpp:72-123)
//   * the reference HIDX container  save_index / load_index   (io.cpp:91-157, 223-232)
//   * the learned-sparse bridge  bridge_ingest / bridge_export / bridge_topk /
//                                bridge_topk_maxscore / SparseVector::validate
//                                (bridge.cpp:10-204)
//   * the dense channel          hash_embed / dense_topk / save+load_embeddings
//                                (dense.cpp:44-192) and agent_rrf (fusion.cpp:22-50)
//   * confidence / k_star / ndcg_at_k / TwoPhaseSelector known-answer hooks
//   * a CPU batch driver shaped like hybridmem's cmd_search parallel_for
//     (tools/hybridmem.cpp:58-71, 305-313) for the CPU baseline timing.
// Nothing here re-implements reference logic; it only marshals arrays.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <optional>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "hybrid/bridge.hpp"
#include "hybrid/cascade.hpp"
#include "hybrid/csr_index.hpp"
#include "hybrid/dense.hpp"
#include "hybrid/fusion.hpp"
#include "hybrid/eval.hpp"
#include "hybrid/io.hpp"
#include "hybrid/temporal_index.hpp"
#include "hybrid/twophase.hpp"
#include "hybrid/workload.hpp"

using namespace hybrid;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    } catch (...) {
        g_err = "unknown error";
        return 1;
    }
}

struct Corpus {
    std::vector<MemoryRecord> recs;
    WorkloadSpec spec;
};
struct Queries {
    std::vector<GeneratedQuery> qs;
};
struct Index {
    CsrIndex idx;
};
struct Temporal {
    TemporalIndex t;
};

TokenizerMode tmode(int m) { return static_cast<TokenizerMode>(m); }

std::vector<std::string> terms_of(const char* const* terms, std::uint32_t n) {
    std::vector<std::string> v;
    v.reserve(n);
    for (std::uint32_t i = 0; i < n; ++i) v.emplace_back(terms[i]);
    return v;
}

void emit(const RankedList& r, std::uint64_t* ids, double* scores,
          std::uint32_t* n) {
    *n = static_cast<std::uint32_t>(r.entries.size());
    for (std::size_t i = 0; i < r.entries.size(); ++i) {
        ids[i] = r.entries[i].first;
        scores[i] = r.entries[i].second;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- workload
int ref_gen_corpus(std::uint64_t n_records, std::uint64_t seed,
                   std::uint32_t vocab_size, double zipf_s,
                   std::uint32_t min_tok, std::uint32_t max_tok,
                   std::int64_t time_span_ms, void** out) {
    return guard([&] {
        auto c = std::make_unique<Corpus>();
        c->spec.n_records = n_records;
        c->spec.seed = seed;
        c->spec.vocab_size = vocab_size;
        c->spec.zipf_s = zipf_s;
        c->spec.min_doc_tokens = min_tok;
        c->spec.max_doc_tokens = max_tok;
        if (time_span_ms > 0) c->spec.time_span_ms = time_span_ms;
        c->recs = gen_corpus(c->spec);
        *out = c.release();
    });
}

void ref_corpus_free(void* h) { delete static_cast<Corpus*>(h); }
std::uint64_t ref_corpus_size(void* h) {
    return static_cast<Corpus*>(h)->recs.size();
}
std::uint64_t ref_corpus_text_bytes(void* h) {
    std::uint64_t n = 0;
    for (auto& r : static_cast<Corpus*>(h)->recs) n += r.text.size() + 1;
    return n;
}
// ids[n], ts[n]; texts concatenated NUL-separated into buf (size from
// ref_corpus_text_bytes).
void ref_corpus_export(void* h, std::uint64_t* ids, std::int64_t* ts,
                       char* buf) {
    auto* c = static_cast<Corpus*>(h);
    std::size_t o = 0;
    for (std::size_t i = 0; i < c->recs.size(); ++i) {
        ids[i] = c->recs[i].id;
        ts[i] = c->recs[i].ts_ms;
        std::memcpy(buf + o, c->recs[i].text.c_str(), c->recs[i].text.size() + 1);
        o += c->recs[i].text.size() + 1;
    }
}

int ref_gen_queries(void* corpus, std::uint64_t n_queries,
                    std::uint32_t min_terms, std::uint32_t max_terms,
                    std::uint64_t seed, void** out) {
    return guard([&] {
        auto* c = static_cast<Corpus*>(corpus);
        QuerySpec qs;
        qs.n_queries = n_queries;
        qs.min_terms = min_terms;
        qs.max_terms = max_terms;
        qs.seed = seed;
        auto q = std::make_unique<Queries>();
        q->qs = gen_queries(c->recs, qs, c->spec);
        *out = q.release();
    });
}
void ref_queries_free(void* h) { delete static_cast<Queries*>(h); }
std::uint64_t ref_queries_size(void* h) {
    return static_cast<Queries*>(h)->qs.size();
}
std::uint64_t ref_queries_text_bytes(void* h) {
    std::uint64_t n = 0;
    for (auto& q : static_cast<Queries*>(h)->qs)
        for (auto& t : q.terms) n += t.size() + 1;
    return n;
}
// n_terms[nq], gold[nq] (first gold id), ts[nq]; terms NUL-separated.
void ref_queries_export(void* h, std::uint32_t* n_terms, std::uint64_t* gold,
                        std::int64_t* ts, char* buf) {
    auto* q = static_cast<Queries*>(h);
    std::size_t o = 0;
    for (std::size_t i = 0; i < q->qs.size(); ++i) {
        n_terms[i] = static_cast<std::uint32_t>(q->qs[i].terms.size());
        gold[i] = q->qs[i].gold.empty() ? ~0ull : *q->qs[i].gold.begin();
        ts[i] = q->qs[i].ts_ms;
        for (auto& t : q->qs[i].terms) {
            std::memcpy(buf + o, t.c_str(), t.size() + 1);
            o += t.size() + 1;
        }
    }
}

// ---------------------------------------------------------------- index
int ref_build_index_texts(std::uint64_t n, const std::uint64_t* ids,
                          const char* const* texts, int tok_mode, double k1,
                          double b, void** out) {
    return guard([&] {
        std::vector<std::pair<DocId, std::string>> docs;
        docs.reserve(n);
        for (std::uint64_t i = 0; i < n; ++i) docs.emplace_back(ids[i], texts[i]);
        auto ix = std::make_unique<Index>();
        ix->idx = build_index(docs, tmode(tok_mode), 50000, Bm25Params{k1, b});
        *out = ix.release();
    });
}

int ref_build_index_corpus(void* corpus, int tok_mode, double k1, double b,
                           void** out) {
    return guard([&] {
        auto* c = static_cast<Corpus*>(corpus);
        std::vector<std::pair<DocId, std::string>> docs;
        docs.reserve(c->recs.size());
        for (auto& r : c->recs) docs.emplace_back(r.id, r.text);
        auto ix = std::make_unique<Index>();
        ix->idx = build_index(docs, tmode(tok_mode), 50000, Bm25Params{k1, b});
        *out = ix.release();
    });
}

// Adopt raw CSR arrays (e.g. from the framework's own native builder) into a
// reference CsrIndex so the reference search code runs on the same index.
int ref_index_from_arrays(std::uint32_t n_terms, const char* const* terms,
                          const std::uint64_t* term_offsets,
                          const std::uint32_t* posting_rows,
                          const double* posting_weights, const double* idfs,
                          const double* maxscores, const double* order_keys,
                          std::uint32_t n_docs, const std::uint32_t* doc_lens,
                          const std::uint64_t* doc_ids, double avgdl,
                          double build_k1, double build_b, void** out) {
    return guard([&] {
        auto ix = std::make_unique<Index>();
        CsrIndex& x = ix->idx;
        x.build_params = Bm25Params{build_k1, build_b};
        x.terms.reserve(n_terms);
        for (std::uint32_t t = 0; t < n_terms; ++t) {
            x.terms.emplace_back(terms[t]);
            x.vocab.emplace(x.terms.back(), t);
        }
        std::uint64_t P = term_offsets[n_terms];
        x.term_offsets.assign(term_offsets, term_offsets + n_terms + 1);
        x.posting_rows.assign(posting_rows, posting_rows + P);
        x.posting_weights.assign(posting_weights, posting_weights + P);
        x.term_idfs.assign(idfs, idfs + n_terms);
        x.term_maxscores.assign(maxscores, maxscores + n_terms);
        x.term_order_keys.assign(order_keys, order_keys + n_terms);
        x.doc_lens.assign(doc_lens, doc_lens + n_docs);
        x.doc_ids.assign(doc_ids, doc_ids + n_docs);
        x.avgdl = avgdl;
        *out = ix.release();
    });
}

void ref_index_free(void* h) { delete static_cast<Index*>(h); }

// HIDX v1 files written / read by the reference's own io.cpp
int ref_save_index(void* h, const char* path) {
    return guard([&] { save_index(static_cast<Index*>(h)->idx, path); });
}
int ref_load_index(const char* path, void** out) {
    return guard([&] {
        auto ix = std::make_unique<Index>();
        ix->idx = load_index(path);
        *out = ix.release();
    });
}

// sizes[0]=n_terms sizes[1]=n_postings sizes[2]=n_docs sizes[3]=term_bytes
void ref_index_sizes(void* h, std::uint64_t* sizes) {
    auto& x = static_cast<Index*>(h)->idx;
    sizes[0] = x.terms.size();
    sizes[1] = x.posting_rows.size();
    sizes[2] = x.doc_ids.size();
    std::uint64_t tb = 0;
    for (auto& t : x.terms) tb += t.size() + 1;
    sizes[3] = tb;
}

void ref_index_export(void* h, char* term_buf, std::uint64_t* term_offsets,
                      std::uint32_t* posting_rows, double* posting_weights,
                      double* idfs, double* maxscores, double* order_keys,
                      std::uint32_t* doc_lens, std::uint64_t* doc_ids,
                      double* avgdl) {
    auto& x = static_cast<Index*>(h)->idx;
    std::size_t o = 0;
    for (auto& t : x.terms) {
        std::memcpy(term_buf + o, t.c_str(), t.size() + 1);
        o += t.size() + 1;
    }
    std::memcpy(term_offsets, x.term_offsets.data(),
                x.term_offsets.size() * sizeof(std::uint64_t));
    std::memcpy(posting_rows, x.posting_rows.data(),
                x.posting_rows.size() * sizeof(std::uint32_t));
    std::memcpy(posting_weights, x.posting_weights.data(),
                x.posting_weights.size() * sizeof(double));
    std::memcpy(idfs, x.term_idfs.data(), x.term_idfs.size() * sizeof(double));
    std::memcpy(maxscores, x.term_maxscores.data(),
                x.term_maxscores.size() * sizeof(double));
    std::memcpy(order_keys, x.term_order_keys.data(),
                x.term_order_keys.size() * sizeof(double));
    std::memcpy(doc_lens, x.doc_lens.data(), x.doc_lens.size() * sizeof(std::uint32_t));
    std::memcpy(doc_ids, x.doc_ids.data(), x.doc_ids.size() * sizeof(std::uint64_t));
    *avgdl = x.avgdl;
}

// mode 0 = bm25_topk (exhaustive), 1 = bm25_topk_maxscore
int ref_search(void* h, const char* const* terms, std::uint32_t n_terms,
               std::uint64_t k, double k1, double b, int mode,
               std::uint64_t* out_ids, double* out_scores, std::uint32_t* out_n,
               std::uint64_t* postings) {
    return guard([&] {
        auto& x = static_cast<Index*>(h)->idx;
        SearchStats st;
        auto q = terms_of(terms, n_terms);
        RankedList r = mode == 1 ? x.bm25_topk_maxscore(q, k, Bm25Params{k1, b}, &st)
                                 : x.bm25_topk(q, k, Bm25Params{k1, b}, &st);
        emit(r, out_ids, out_scores, out_n);
        if (postings) *postings = st.postings_touched;
    });
}

// Batch driver with the CLI's structure: optional warm-up, then an
// index-order atomic work queue over `workers` std::threads
// (tools/hybridmem.cpp:58-71, 305-313).  Outputs are [nq*k]; lat_ms[nq] is
// each query's wall time; *wall_ms the whole measured pass.
int ref_search_batch(void* h, std::uint32_t nq, const std::uint32_t* q_off,
                     const char* const* terms, std::uint64_t k, double k1,
                     double b, int mode, unsigned workers, unsigned warmup,
                     std::uint64_t* out_ids, double* out_scores,
                     std::uint32_t* out_n, std::uint64_t* postings,
                     double* lat_ms, double* wall_ms) {
    return guard([&] {
        auto& x = static_cast<Index*>(h)->idx;
        Bm25Params p{k1, b};
        auto run_one = [&](std::size_t i, bool record) {
            std::vector<std::string> q;
            for (std::uint32_t j = q_off[i]; j < q_off[i + 1]; ++j) q.emplace_back(terms[j]);
            SearchStats st;
            RankedList r = mode == 1 ? x.bm25_topk_maxscore(q, k, p, &st)
                                     : x.bm25_topk(q, k, p, &st);
            if (record) {
                emit(r, out_ids + i * k, out_scores + i * k, out_n + i);
                if (postings) postings[i] = st.postings_touched;
            }
        };
        for (std::size_t i = 0; i < std::min<std::size_t>(nq, warmup); ++i) run_one(i, false);
        using clk = std::chrono::steady_clock;
        auto t0 = clk::now();
        std::atomic<std::size_t> next{0};
        auto body = [&] {
            for (std::size_t i; (i = next.fetch_add(1)) < nq;) {
                auto a = clk::now();
                run_one(i, true);
                if (lat_ms)
                    lat_ms[i] = std::chrono::duration<double, std::milli>(clk::now() - a).count();
            }
        };
        if (workers <= 1) {
            body();
        } else {
            std::vector<std::thread> pool;
            for (unsigned w = 0; w < workers; ++w) pool.emplace_back(body);
            for (auto& t : pool) t.join();
        }
        *wall_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
    });
}

// ---------------------------------------------------------------- temporal
int ref_build_temporal(std::uint64_t n, const std::uint64_t* ids,
                       const std::int64_t* ts, const char* const* texts,
                       std::int64_t window_ms, double epsilon, double lambda_hat,
                       std::uint32_t k_max, int tok_mode, double k1, double b,
                       void** out) {
    return guard([&] {
        std::vector<MemoryRecord> recs(n);
        for (std::uint64_t i = 0; i < n; ++i) {
            recs[i].id = ids[i];
            recs[i].ts_ms = ts[i];
            recs[i].text = texts[i];
        }
        TemporalParams tp;
        tp.window_ms = window_ms;
        tp.epsilon = epsilon;
        tp.lambda_hat = lambda_hat;
        tp.k_max_partitions = k_max;
        auto t = std::make_unique<Temporal>();
        t->t = build_temporal_index(recs, tp, tmode(tok_mode), Bm25Params{k1, b});
        *out = t.release();
    });
}
// A reference TemporalIndex over a partition-ordered flat index (rows of
// partition j are [part_row[j], part_row[j+1])): each partition a CsrIndex of
// its rows with the flat (shared) idf / order keys / avgdl and its own
// maxscores from the reference's compute_term_maxscores -- the object
// build_temporal_index produces (temporal_index.cpp:125-169), without
// re-tokenising the corpus.  Marshalling only (bench CPU baseline, tests).
int ref_temporal_from_flat(std::uint32_t n_terms, const char* const* terms,
                           const std::uint64_t* term_offsets, const std::uint32_t* posting_rows,
                           const double* posting_weights, const double* idfs, const double* order_keys,
                           const std::uint32_t* doc_lens, const std::uint64_t* doc_ids, double avgdl,
                           std::uint32_t n_parts, const std::uint32_t* part_row, std::int64_t t0,
                           std::int64_t window_ms, double epsilon, double lambda_hat, std::uint32_t k_max,
                           double build_k1, double build_b, void** out) {
    return guard([&] {
        auto t = std::make_unique<Temporal>();
        TemporalIndex& T = t->t;
        T.params.window_ms = window_ms;
        T.params.epsilon = epsilon;
        T.params.lambda_hat = lambda_hat;
        T.params.k_max_partitions = k_max;
        T.total_docs = part_row[n_parts];
        T.shared.avgdl = avgdl;
        for (std::uint32_t g = 0; g < n_terms; ++g) {
            T.shared.idf.emplace(terms[g], idfs[g]);
            T.shared.order_key.emplace(terms[g], order_keys[g]);
        }
        std::vector<std::uint64_t> cur(term_offsets, term_offsets + n_terms);  // per-term cursor
        T.partitions.resize(n_parts);
        for (std::uint32_t j = 0; j < n_parts; ++j) {
            auto& part = T.partitions[j];
            part.window_start = t0 + static_cast<std::int64_t>(j) * window_ms;
            part.window_end = part.window_start + window_ms;
            CsrIndex& x = part.index;
            x.build_params = Bm25Params{build_k1, build_b};
            x.avgdl = avgdl;
            const std::uint32_t lo = part_row[j], hi = part_row[j + 1];
            x.term_offsets.push_back(0);
            for (std::uint32_t g = 0; g < n_terms; ++g) {
                std::uint64_t i = cur[g];
                const std::uint64_t e = term_offsets[g + 1];
                if (i == e || posting_rows[i] >= hi) continue;
                for (; i < e && posting_rows[i] < hi; ++i) {
                    x.posting_rows.push_back(posting_rows[i] - lo);
                    x.posting_weights.push_back(posting_weights[i]);
                }
                cur[g] = i;
                x.vocab.emplace(terms[g], static_cast<std::uint32_t>(x.terms.size()));
                x.terms.emplace_back(terms[g]);
                x.term_idfs.push_back(idfs[g]);
                x.term_order_keys.push_back(order_keys[g]);
                x.term_offsets.push_back(x.posting_rows.size());
            }
            x.doc_lens.assign(doc_lens + lo, doc_lens + hi);
            x.doc_ids.assign(doc_ids + lo, doc_ids + hi);
            x.term_maxscores = x.compute_term_maxscores(x.build_params);
        }
        *out = t.release();
    });
}

int ref_build_temporal_corpus(void* corpus, std::int64_t window_ms,
                              double epsilon, double lambda_hat,
                              std::uint32_t k_max, int tok_mode, double k1,
                              double b, void** out) {
    return guard([&] {
        auto* c = static_cast<Corpus*>(corpus);
        TemporalParams tp;
        tp.window_ms = window_ms;
        tp.epsilon = epsilon;
        tp.lambda_hat = lambda_hat;
        tp.k_max_partitions = k_max;
        auto t = std::make_unique<Temporal>();
        t->t = build_temporal_index(c->recs, tp, tmode(tok_mode), Bm25Params{k1, b});
        *out = t.release();
    });
}
void ref_temporal_free(void* h) { delete static_cast<Temporal*>(h); }

// HTIX v1 files written / read by the reference's own io.cpp (:234-318)
int ref_save_temporal(void* h, const char* path) {
    return guard([&] { save_temporal_index(static_cast<Temporal*>(h)->t, path); });
}
int ref_load_temporal(const char* path, void** out) {
    return guard([&] {
        auto t = std::make_unique<Temporal>();
        t->t = load_temporal_index(path);
        *out = t.release();
    });
}
std::uint32_t ref_temporal_num_partitions(void* h) {
    return static_cast<Temporal*>(h)->t.num_partitions();
}
// window_start[K], window_end[K], n_docs[K]
void ref_temporal_partitions(void* h, std::int64_t* ws, std::int64_t* we,
                             std::uint32_t* nd) {
    auto& t = static_cast<Temporal*>(h)->t;
    for (std::uint32_t i = 0; i < t.num_partitions(); ++i) {
        ws[i] = t.partitions[i].window_start;
        we[i] = t.partitions[i].window_end;
        nd[i] = t.partitions[i].index.num_docs();
    }
}
int ref_temporal_topk(void* h, const char* const* terms, std::uint32_t n_terms,
                      std::uint64_t k, double k1, double b, int use_ub_stop,
                      std::uint64_t* out_ids, double* out_scores,
                      std::uint32_t* out_n, std::uint32_t* searched,
                      std::uint64_t* postings) {
    return guard([&] {
        auto& t = static_cast<Temporal*>(h)->t;
        TemporalStats st;
        auto r = t.topk(terms_of(terms, n_terms), k, Bm25Params{k1, b}, &st,
                        use_ub_stop != 0);
        emit(r, out_ids, out_scores, out_n);
        if (searched) *searched = st.partitions_searched;
        if (postings) *postings = st.postings_touched;
    });
}
int ref_temporal_batch(void* h, std::uint32_t nq, const std::uint32_t* q_off,
                       const char* const* terms, std::uint64_t k, double k1,
                       double b, unsigned workers, std::uint64_t* out_ids,
                       double* out_scores, std::uint32_t* out_n,
                       double* wall_ms) {
    return guard([&] {
        auto& t = static_cast<Temporal*>(h)->t;
        Bm25Params p{k1, b};
        using clk = std::chrono::steady_clock;
        auto t0 = clk::now();
        std::atomic<std::size_t> next{0};
        auto body = [&] {
            for (std::size_t i; (i = next.fetch_add(1)) < nq;) {
                std::vector<std::string> q;
                for (std::uint32_t j = q_off[i]; j < q_off[i + 1]; ++j) q.emplace_back(terms[j]);
                auto r = t.topk(q, k, p);
                emit(r, out_ids + i * k, out_scores + i * k, out_n + i);
            }
        };
        std::vector<std::thread> pool;
        for (unsigned w = 0; w < std::max(1u, workers); ++w) pool.emplace_back(body);
        for (auto& th : pool) th.join();
        *wall_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
    });
}

// ---------------------------------------------------------------- scalars
double ref_bm25_score(double tf, double idf, double len, double avgdl,
                      double k1, double b) {
    return bm25_score(tf, idf, len, avgdl, Bm25Params{k1, b});
}
int ref_confidence(const double* s, std::uint32_t n, int proxy, double eps,
                   double* out) {
    return guard([&] {
        *out = confidence(std::vector<double>(s, s + n),
                          static_cast<ConfidenceProxy>(proxy), eps);
    });
}
int ref_k_star(double eps, double lambda, std::uint32_t* out) {
    return guard([&] { *out = k_star(eps, lambda); });
}
// rels: parallel arrays (doc, grade)
int ref_ndcg(const std::uint64_t* ids, const double* scores, std::uint32_t n,
             const std::uint64_t* rel_docs, const std::uint32_t* rel_grades,
             std::uint32_t n_rel, std::uint64_t k, int linear, double* out) {
    return guard([&] {
        RankedList r;
        for (std::uint32_t i = 0; i < n; ++i) r.entries.emplace_back(ids[i], scores[i]);
        std::map<DocId, std::uint32_t> rels;
        for (std::uint32_t i = 0; i < n_rel; ++i) rels[rel_docs[i]] = rel_grades[i];
        *out = linear ? linear_gain_ndcg_at_k(r, rels, k) : ndcg_at_k(r, rels, k);
    });
}
// Two-phase selector over a batch of score rows (row-major [rows x n]).
int ref_twophase_batch(std::uint64_t capacity, int reset_sentinel,
                       std::uint32_t rows, std::uint32_t n, const double* scores,
                       std::uint64_t k, std::uint64_t* out_ids,
                       double* out_scores, std::uint32_t* out_n) {
    return guard([&] {
        TwoPhaseSelector sel(capacity, reset_sentinel != 0);
        for (std::uint32_t r = 0; r < rows; ++r) {
            std::vector<double> row(scores + std::size_t(r) * n, scores + std::size_t(r + 1) * n);
            emit(sel.select(row, k), out_ids + r * k, out_scores + r * k, out_n + r);
        }
    });
}

// ---------------------------------------------------------------- bridge
// Documents as concatenated sparse vectors: doc d owns idx/val[vec_off[d] ..
// vec_off[d+1]).  The result is a Bridge-mode CsrIndex (an Index handle).
int ref_bridge_ingest(std::uint32_t n_docs, const std::uint64_t* ids,
                      const std::uint64_t* vec_off, const std::uint32_t* idx,
                      const double* val, void** out) {
    return guard([&] {
        std::vector<std::pair<DocId, SparseVector>> docs(n_docs);
        for (std::uint32_t d = 0; d < n_docs; ++d) {
            docs[d].first = ids[d];
            docs[d].second.indices.assign(idx + vec_off[d], idx + vec_off[d + 1]);
            docs[d].second.values.assign(val + vec_off[d], val + vec_off[d + 1]);
        }
        auto x = std::make_unique<Index>();
        x->idx = bridge_ingest(docs);
        *out = x.release();
    });
}

// bridge_export (the exact inverse): ids[n_docs], vec_off[n_docs+1], idx/val[P]
int ref_bridge_export(void* h, std::uint64_t* ids, std::uint64_t* vec_off,
                      std::uint32_t* idx, double* val) {
    return guard([&] {
        auto v = bridge_export(static_cast<Index*>(h)->idx);
        std::uint64_t o = 0;
        for (std::size_t d = 0; d < v.size(); ++d) {
            ids[d] = v[d].first;
            vec_off[d] = o;
            for (std::size_t i = 0; i < v[d].second.nnz(); ++i, ++o) {
                idx[o] = v[d].second.indices[i];
                val[o] = v[d].second.values[i];
            }
        }
        vec_off[v.size()] = o;
    });
}

int ref_sparse_validate(const std::uint32_t* idx, std::uint32_t n_idx, const double* val,
                        std::uint32_t n_val) {
    return guard([&] { SparseVector{std::vector<std::uint32_t>(idx, idx + n_idx),
                                    std::vector<double>(val, val + n_val)}.validate(); });
}

// mode 0 = bridge_topk, 1 = bridge_topk_maxscore; queries as concatenated
// sparse vectors q_off[nq+1]; outputs stride k; workers as ref_search_batch.
int ref_bridge_batch(void* h, std::uint32_t nq, const std::uint64_t* q_off,
                     const std::uint32_t* q_idx, const double* q_val, std::uint64_t k,
                     int mode, unsigned workers, std::uint64_t* out_ids,
                     double* out_scores, std::uint32_t* out_n, std::uint64_t* postings,
                     double* wall_ms) {
    return guard([&] {
        auto& x = static_cast<Index*>(h)->idx;
        std::vector<SparseVector> qs(nq);
        for (std::uint32_t i = 0; i < nq; ++i) {
            qs[i].indices.assign(q_idx + q_off[i], q_idx + q_off[i + 1]);
            qs[i].values.assign(q_val + q_off[i], q_val + q_off[i + 1]);
        }
        std::vector<std::string> errs(nq);
        using clk = std::chrono::steady_clock;
        auto t0 = clk::now();
        std::atomic<std::size_t> next{0};
        auto body = [&] {
            for (std::size_t i; (i = next.fetch_add(1)) < nq;) {
                try {
                    SearchStats st;
                    RankedList r = mode == 1 ? bridge_topk_maxscore(x, qs[i], k, &st)
                                             : bridge_topk(x, qs[i], k, &st);
                    emit(r, out_ids + i * k, out_scores + i * k, out_n + i);
                    if (postings) postings[i] = st.postings_touched;
                } catch (const std::exception& e) {
                    errs[i] = e.what();
                }
            }
        };
        if (workers <= 1) {
            body();
        } else {
            std::vector<std::thread> pool;
            for (unsigned w = 0; w < workers; ++w) pool.emplace_back(body);
            for (auto& t : pool) t.join();
        }
        if (wall_ms) *wall_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
        for (auto& e : errs)
            if (!e.empty()) throw std::runtime_error(e);
    });
}

// A Bridge-mode CsrIndex adopted from CSR arrays (the layout bridge_ingest
// produces, bridge.cpp:38-72), for large timing workloads where building
// per-doc vectors first would dominate.  Marshalling only: fields are filled
// as bridge_ingest fills them.
int ref_bridge_from_arrays(std::uint32_t n_terms, const std::uint64_t* term_offsets,
                           const std::uint32_t* rows, const double* weights,
                           std::uint32_t n_docs, const std::uint64_t* doc_ids,
                           const std::uint32_t* doc_lens, double avgdl, void** out) {
    return guard([&] {
        auto x = std::make_unique<Index>();
        CsrIndex& idx = x->idx;
        idx.mode = IndexMode::Bridge;
        const std::uint64_t P = term_offsets[n_terms];
        idx.term_offsets.assign(term_offsets, term_offsets + n_terms + 1);
        idx.posting_rows.assign(rows, rows + P);
        idx.posting_weights.assign(weights, weights + P);
        idx.doc_ids.assign(doc_ids, doc_ids + n_docs);
        idx.doc_lens.assign(doc_lens, doc_lens + n_docs);
        idx.avgdl = avgdl;
        for (std::uint32_t t = 0; t < n_terms; ++t) {
            idx.terms.push_back(std::to_string(t));
            idx.vocab.emplace(idx.terms.back(), t);
            double maxw = 0.0;
            for (std::uint64_t i = term_offsets[t]; i < term_offsets[t + 1]; ++i) maxw = std::max(maxw, weights[i]);
            idx.term_idfs.push_back(0.0);
            idx.term_maxscores.push_back(maxw);
        }
        idx.term_order_keys = idx.term_maxscores;
        *out = x.release();
    });
}

// ---------------------------------------------------------------- dense
int ref_hash_embed(const char* text, std::uint32_t dim, std::uint64_t seed, float* out) {
    return guard([&] {
        auto v = hash_embed(text, dim, seed);
        std::memcpy(out, v.data(), v.size() * sizeof(float));
    });
}

// dense_topk per query over a matrix adopted from arrays (EmbeddingMatrix is
// a plain struct, dense.hpp:13-22); queries [nq x qdim]; outputs stride k.
int ref_dense_batch(std::uint32_t dim, std::uint64_t count, const float* data,
                    const std::uint64_t* ids, std::uint32_t nq, std::uint32_t qdim,
                    const float* queries, std::uint64_t k, unsigned workers,
                    std::uint64_t* out_ids, double* out_scores, std::uint32_t* out_n,
                    double* wall_ms) {
    return guard([&] {
        EmbeddingMatrix m;
        m.dim = dim;
        m.doc_ids.assign(ids, ids + count);
        m.data.assign(data, data + count * dim);
        std::vector<std::string> errs(nq);
        using clk = std::chrono::steady_clock;
        auto t0 = clk::now();
        std::atomic<std::size_t> next{0};
        auto body = [&] {
            for (std::size_t i; (i = next.fetch_add(1)) < nq;) {
                try {
                    std::vector<float> q(queries + i * qdim, queries + (i + 1) * qdim);
                    emit(dense_topk(m, q, k), out_ids + i * k, out_scores + i * k, out_n + i);
                } catch (const std::exception& e) {
                    errs[i] = e.what();
                }
            }
        };
        if (workers <= 1) {
            body();
        } else {
            std::vector<std::thread> pool;
            for (unsigned w = 0; w < workers; ++w) pool.emplace_back(body);
            for (auto& t : pool) t.join();
        }
        if (wall_ms) *wall_ms = std::chrono::duration<double, std::milli>(clk::now() - t0).count();
        for (auto& e : errs)
            if (!e.empty()) throw std::runtime_error(e);
    });
}

int ref_save_embeddings(std::uint32_t dim, std::uint64_t count, const float* data,
                        const std::uint64_t* ids, const char* path) {
    return guard([&] {
        EmbeddingMatrix m;
        m.dim = dim;
        m.doc_ids.assign(ids, ids + count);
        m.data.assign(data, data + count * dim);
        save_embeddings(m, path);
    });
}

// agent_rrf (fusion.cpp:22-50) over two ranked lists; records given as
// parallel arrays (id, ts_ms, weight); qtype NULL = nullopt
int ref_agent_rrf(const std::uint64_t* s_ids, const double* s_sc, std::uint32_t ns,
                  const std::uint64_t* d_ids, const double* d_sc, std::uint32_t nd,
                  const std::uint64_t* rec_ids, const std::int64_t* rec_ts, const double* rec_w,
                  std::uint32_t n_rec, std::int64_t query_ts, const char* qtype, double k_rrf,
                  double alpha, std::int64_t tau_ms, double beta, std::uint64_t cap,
                  std::uint64_t* out_ids, double* out_scores, std::uint32_t* out_n) {
    return guard([&] {
        RankedList a, b;
        for (std::uint32_t i = 0; i < ns; ++i) a.entries.emplace_back(s_ids[i], s_sc[i]);
        for (std::uint32_t i = 0; i < nd; ++i) b.entries.emplace_back(d_ids[i], d_sc[i]);
        std::vector<MemoryRecord> recs(n_rec);
        std::unordered_map<DocId, const MemoryRecord*> by_id;
        for (std::uint32_t i = 0; i < n_rec; ++i) {
            recs[i].id = rec_ids[i];
            recs[i].ts_ms = rec_ts[i];
            recs[i].weight = rec_w[i];
        }
        for (auto& r : recs) by_id[r.id] = &r;
        RecordLookup lookup = [&](DocId d) -> const MemoryRecord* {
            auto it = by_id.find(d);
            return it == by_id.end() ? nullptr : it->second;
        };
        FusionParams p;
        p.k_rrf = k_rrf;
        p.alpha = alpha;
        p.tau_ms = tau_ms;
        p.beta = beta;
        std::optional<std::string> qt;
        if (qtype) qt = std::string(qtype);
        RankedList r = agent_rrf(a, b, lookup, query_ts, qt, p);
        if (r.entries.size() > cap) r.entries.resize(cap);
        emit(r, out_ids, out_scores, out_n);
    });
}

// BM25 scoring on a bridge-mode index (the reference's refusal message)
int ref_bm25_on(void* h, const char* term) {
    return guard([&] { static_cast<Index*>(h)->idx.bm25_topk({term}, 5, Bm25Params{}); });
}

}  // extern "C"
