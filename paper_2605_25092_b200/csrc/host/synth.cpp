// Native synthetic workload generator + CSR builder (see include/hm_synth.h).
//
// Bit-parity contract with the reference (paths under /root/reference/proj):
//   * draws come from std::mt19937_64 exactly as src/workload.cpp:47-135 and
//     include/hybrid/rng.hpp:13-39 consume them (next_double = (x>>11)*2^-53,
//     uniform_u64 = x % n with no draw when n == 0);
//   * the Zipf inverse CDF is built with the same pow/sum/normalise sequence as
//     ZipfSampler (workload.cpp:15-33); sampling returns lower_bound(cdf, u)
//     but narrows the search with a 2^20-bucket guide table whose bucket edges
//     b/2^20 are exact doubles, so the answer is the same index;
//   * the CSR follows build_index (csr_index.cpp:232-324): alphabetical term
//     ids, rows strictly increasing per term, raw tf, idf = ln(1+(N-df+.5)/
//     (df+.5)), avgdl = sequential double sum / N, maxscore = max bm25_score
//     under the build params, order key = maxscore.
// Parallelism: generation runs one sequential pass that only advances the
// engine and snapshots it every kChunk records, then regenerates chunks in
// parallel; the build counts per-thread document-frequencies and fills
// postings in parallel at precomputed cursors.  Output is independent of the
// thread count.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "hm_synth.h"

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

inline double next_double(std::mt19937_64& g) {
    return static_cast<double>(g() >> 11) * 0x1.0p-53;
}
inline std::uint64_t uniform_u64(std::mt19937_64& g, std::uint64_t n) {
    return n == 0 ? 0 : g() % n;
}

int n_threads(int t) {
    if (t > 0) return t;
    unsigned h = std::thread::hardware_concurrency();
    return h ? static_cast<int>(h) : 1;
}

template <typename F>
void parallel_ranges(std::size_t n, int threads, F&& f) {
    threads = std::max(1, std::min<int>(threads, static_cast<int>(std::max<std::size_t>(n, 1))));
    if (threads == 1) {
        f(0, std::size_t{0}, n);
        return;
    }
    std::vector<std::thread> pool;
    std::exception_ptr err;
    std::atomic<bool> failed{false};
    for (int t = 0; t < threads; ++t) {
        std::size_t a = n * t / threads, b = n * (t + 1) / threads;
        pool.emplace_back([&, t, a, b] {
            try {
                f(t, a, b);
            } catch (...) {
                if (!failed.exchange(true)) err = std::current_exception();
            }
        });
    }
    for (auto& th : pool) th.join();
    if (err) std::rethrow_exception(err);
}

// ZipfSampler of workload.cpp:15-33 with an exact guide table.
class Zipf {
public:
    Zipf(std::uint32_t n, double s) : cdf_(n) {
        double sum = 0.0;
        for (std::uint32_t k = 1; k <= n; ++k) {
            sum += 1.0 / std::pow(static_cast<double>(k), s);
            cdf_[k - 1] = sum;
        }
        for (double& v : cdf_) v /= sum;
        guide_.resize(kBuckets + 1);
        for (std::uint32_t bkt = 0; bkt <= kBuckets; ++bkt) {
            double edge = static_cast<double>(bkt) * (1.0 / kBuckets);  // exact
            guide_[bkt] = static_cast<std::uint32_t>(
                std::lower_bound(cdf_.begin(), cdf_.end(), edge) - cdf_.begin());
        }
    }
    std::uint32_t sample(std::mt19937_64& g) const {
        double u = next_double(g);
        std::uint32_t bkt = static_cast<std::uint32_t>(u * kBuckets);  // floor, exact
        // lower_bound(u) lies in [lower_bound(b/B), lower_bound((b+1)/B)]
        std::uint32_t lo = guide_[bkt];
        std::uint32_t hi = std::min<std::uint32_t>(guide_[bkt + 1] + 1,
                                                   static_cast<std::uint32_t>(cdf_.size()));
        return static_cast<std::uint32_t>(
            std::lower_bound(cdf_.begin() + lo, cdf_.begin() + hi, u) - cdf_.begin());
    }

private:
    static constexpr std::uint32_t kBuckets = 1u << 20;
    std::vector<double> cdf_;
    std::vector<std::uint32_t> guide_;
};

// role draw of workload.cpp:36-44; returns true for ToolCall/ToolOutput
inline bool role_is_tool(double u) { return u >= 0.60 && u < 0.90; }

// One record's draws after the tokens (workload.cpp:67-76).
inline void skip_record_tail(std::mt19937_64& g, const hm_wspec& s) {
    bool tool = role_is_tool(next_double(g));
    uniform_u64(g, s.n_sessions);
    uniform_u64(g, s.n_agents);
    if (tool) uniform_u64(g, 3);
}

}  // namespace

struct hm_synth_corpus {
    hm_wspec spec;
    std::vector<std::uint32_t> tokens;
    std::vector<std::uint64_t> offsets;
    std::vector<std::int64_t> ts;
};

struct hm_synth_queries {
    std::vector<std::uint32_t> terms;
    std::vector<std::uint64_t> offsets;
    std::vector<std::uint64_t> gold;
    std::vector<std::int64_t> ts;
    std::vector<std::uint8_t> para;
};

struct hm_synth_index {
    std::vector<std::uint32_t> term_rank, rank_to_tid, posting_rows, posting_tf,
        doc_lens;
    std::vector<std::uint64_t> term_offsets, doc_ids;
    std::vector<double> idf, maxscore, order_key;
    double avgdl = 0.0;
};

extern "C" {

const char* hm_synth_last_error(void) { return g_err.c_str(); }

void hm_wspec_default(hm_wspec* w) {
    w->n_records = 4052;
    w->seed = 42;
    w->recency_mass = 0.8;
    w->recency_window = 0.2;
    w->vocab_size = 5000;
    w->zipf_s = 1.1;
    w->min_doc_tokens = 5;
    w->max_doc_tokens = 30;
    w->n_sessions = 50;
    w->n_agents = 4;
    w->time_span_ms = 28LL * 24 * 3600 * 1000;
    w->t0_ms = 1700000000000LL;
}

void hm_qspec_default(hm_qspec* q) {
    q->n_queries = 1000;
    q->min_terms = 3;
    q->max_terms = 6;
    q->paraphrase_noise = 0.0;
    q->seed = 42;
}

int hm_synth_corpus_create(const hm_wspec* spec, int threads, hm_synth_corpus** out) {
    return guard([&] {
        if (spec->n_records == 0) throw std::invalid_argument("n_records must be >= 1");
        if (spec->max_doc_tokens < spec->min_doc_tokens)
            throw std::invalid_argument("max_doc_tokens < min_doc_tokens");
        auto c = std::make_unique<hm_synth_corpus>();
        c->spec = *spec;
        const hm_wspec& s = *spec;
        const std::uint64_t n = s.n_records;
        const std::uint64_t span_n = static_cast<std::uint64_t>(s.time_span_ms);
        constexpr std::uint64_t kChunk = 1u << 16;
        // pass 1: advance the engine, record lengths, timestamps and snapshots
        std::mt19937_64 g(s.seed);
        std::vector<std::mt19937_64> snaps;
        c->offsets.resize(n + 1);
        c->ts.resize(n);
        c->offsets[0] = 0;
        for (std::uint64_t i = 0; i < n; ++i) {
            if (i % kChunk == 0) snaps.push_back(g);
            std::uint32_t len = s.min_doc_tokens + static_cast<std::uint32_t>(uniform_u64(
                                    g, s.max_doc_tokens - s.min_doc_tokens + 1));
            g.discard(len);
            skip_record_tail(g, s);
            c->ts[i] = s.t0_ms + static_cast<std::int64_t>(uniform_u64(g, span_n));
            next_double(g);  // weight
            c->offsets[i + 1] = c->offsets[i] + len;
        }
        c->tokens.resize(c->offsets[n]);
        Zipf zipf(s.vocab_size, s.zipf_s);
        std::size_t n_chunks = snaps.size();
        std::atomic<std::size_t> next{0};
        parallel_ranges(n_threads(threads), n_threads(threads), [&](int, std::size_t, std::size_t) {
            for (std::size_t ch; (ch = next.fetch_add(1)) < n_chunks;) {
                std::mt19937_64 gg = snaps[ch];
                std::uint64_t a = ch * kChunk, b = std::min<std::uint64_t>(n, a + kChunk);
                for (std::uint64_t i = a; i < b; ++i) {
                    std::uint32_t len = s.min_doc_tokens + static_cast<std::uint32_t>(uniform_u64(
                                            gg, s.max_doc_tokens - s.min_doc_tokens + 1));
                    std::uint32_t* dst = c->tokens.data() + c->offsets[i];
                    for (std::uint32_t t = 0; t < len; ++t) dst[t] = zipf.sample(gg);
                    skip_record_tail(gg, s);
                    uniform_u64(gg, span_n);
                    next_double(gg);
                }
            }
        });
        *out = c.release();
    });
}

void hm_synth_corpus_destroy(hm_synth_corpus* c) { delete c; }
uint64_t hm_synth_corpus_n(const hm_synth_corpus* c) { return c->ts.size(); }
uint64_t hm_synth_corpus_n_tokens(const hm_synth_corpus* c) { return c->tokens.size(); }
const uint32_t* hm_synth_corpus_tokens(const hm_synth_corpus* c) { return c->tokens.data(); }
const uint64_t* hm_synth_corpus_offsets(const hm_synth_corpus* c) { return c->offsets.data(); }
const int64_t* hm_synth_corpus_ts(const hm_synth_corpus* c) { return c->ts.data(); }

// gen_queries, workload.cpp:84-135.  Query terms are the gold record's
// distinct tokens in STRING order (tokenize+sort+unique, :111-113), sampled
// without replacement.
int hm_synth_queries_create(const hm_synth_corpus* c, const hm_qspec* q,
                            hm_synth_queries** out) {
    return guard([&] {
        const hm_wspec& w = c->spec;
        const std::uint64_t n = c->ts.size();
        if (n == 0) throw std::invalid_argument("empty corpus");
        std::mt19937_64 g(q->seed ^ 0x9E3779B97F4A7C15ULL);
        std::int64_t window_start =
            w.t0_ms + static_cast<std::int64_t>(static_cast<double>(w.time_span_ms) *
                                                (1.0 - w.recency_window));
        std::vector<std::uint64_t> recent, older;
        for (std::uint64_t i = 0; i < n; ++i)
            (c->ts[i] >= window_start ? recent : older).push_back(i);
        if (recent.empty()) recent = older;
        if (older.empty()) older = recent;
        auto r = std::make_unique<hm_synth_queries>();
        r->offsets.push_back(0);
        std::vector<std::pair<std::string, std::uint32_t>> toks;
        for (std::uint64_t qi = 0; qi < q->n_queries; ++qi) {
            bool pick_recent = next_double(g) < w.recency_mass;
            const auto& pool = pick_recent ? recent : older;
            std::uint64_t gold = pool[uniform_u64(g, pool.size())];
            toks.clear();
            for (std::uint64_t j = c->offsets[gold]; j < c->offsets[gold + 1]; ++j)
                toks.emplace_back("w" + std::to_string(c->tokens[j]), c->tokens[j]);
            std::sort(toks.begin(), toks.end());
            toks.erase(std::unique(toks.begin(), toks.end()), toks.end());
            std::uint32_t want = q->min_terms + static_cast<std::uint32_t>(
                                     uniform_u64(g, q->max_terms - q->min_terms + 1));
            for (std::uint32_t t = 0; t < want && !toks.empty(); ++t) {
                std::size_t j = uniform_u64(g, toks.size());
                r->terms.push_back(toks[j].second);
                toks.erase(toks.begin() + static_cast<std::ptrdiff_t>(j));
            }
            bool para = next_double(g) < q->paraphrase_noise;
            r->para.push_back(para ? 1 : 0);
            r->gold.push_back(gold);
            std::int64_t after = static_cast<std::int64_t>(
                uniform_u64(g, static_cast<std::uint64_t>(w.time_span_ms / 10 + 1)));
            r->ts.push_back(c->ts[gold] + after);
            r->offsets.push_back(r->terms.size());
        }
        *out = r.release();
    });
}

void hm_synth_queries_destroy(hm_synth_queries* q) { delete q; }
uint64_t hm_synth_queries_n(const hm_synth_queries* q) { return q->gold.size(); }
const uint32_t* hm_synth_queries_terms(const hm_synth_queries* q) { return q->terms.data(); }
const uint64_t* hm_synth_queries_offsets(const hm_synth_queries* q) { return q->offsets.data(); }
const uint64_t* hm_synth_queries_gold(const hm_synth_queries* q) { return q->gold.data(); }
const int64_t* hm_synth_queries_ts(const hm_synth_queries* q) { return q->ts.data(); }
const uint8_t* hm_synth_queries_paraphrased(const hm_synth_queries* q) { return q->para.data(); }

}  // extern "C"

namespace {

// Distinct token ranks of record rec, sorted (the tf runs of its postings).
inline void distinct_tokens(const hm_synth_corpus* c, std::uint64_t rec, std::vector<std::uint32_t>& buf) {
    buf.assign(c->tokens.begin() + static_cast<std::ptrdiff_t>(c->offsets[rec]),
               c->tokens.begin() + static_cast<std::ptrdiff_t>(c->offsets[rec + 1]));
    std::sort(buf.begin(), buf.end());
}

// Document frequency per rank over rows [lo, hi) of the row order, per thread.
std::vector<std::vector<std::uint32_t>> count_df(const hm_synth_corpus* c, const std::vector<std::uint64_t>& recs,
                                                 int T) {
    const std::uint32_t V = c->spec.vocab_size;
    std::vector<std::vector<std::uint32_t>> dfl(T);
    parallel_ranges(recs.size(), T, [&](int t, std::size_t a, std::size_t e) {
        dfl[t].assign(V, 0);
        std::vector<std::uint32_t> buf;
        for (std::size_t row = a; row < e; ++row) {
            distinct_tokens(c, recs[row], buf);
            for (std::size_t i = 0; i < buf.size(); ++i)
                if (i == 0 || buf[i] != buf[i - 1]) {
                    if (buf[i] >= V) throw std::runtime_error("token rank >= vocab_size");
                    ++dfl[t][buf[i]];
                }
        }
    });
    return dfl;
}

// The CSR of the records recs[0..n) (row r = recs[r]); the statistics come
// from global_df / n_global / avgdl_global when given (a doc-range shard of a
// larger corpus: SharedStats, csr_index.hpp:28-35), else from these records.
hm_synth_index* build_rows(const hm_synth_corpus* c, double k1, double b, const std::vector<std::uint64_t>& recs,
                           const std::uint64_t* global_df, std::uint64_t n_global, double avgdl_global, int T) {
    const std::uint64_t n = recs.size();
    if (n >= (1ull << 32)) throw std::invalid_argument("too many records for u32 rows");
    const std::uint32_t V = c->spec.vocab_size;
    auto x = std::make_unique<hm_synth_index>();
    x->doc_lens.resize(n);
    x->doc_ids.resize(n);
    for (std::uint64_t r = 0; r < n; ++r) {
        x->doc_ids[r] = recs[r];
        x->doc_lens[r] = static_cast<std::uint32_t>(c->offsets[recs[r] + 1] - c->offsets[recs[r]]);
    }
    std::vector<std::vector<std::uint32_t>> dfl = count_df(c, recs, T);
    std::vector<std::uint64_t> df(V, 0);  // postings per rank in these rows
    for (int t = 0; t < T; ++t)
        if (!dfl[t].empty())
            for (std::uint32_t r = 0; r < V; ++r) df[r] += dfl[t][r];
    // alphabetical term ids over present ranks (csr_index.cpp:272-274); a
    // shard keeps every term of the corpus, so term ids agree across shards
    const std::uint64_t* present = global_df ? global_df : df.data();
    std::vector<std::pair<std::string, std::uint32_t>> names;
    for (std::uint32_t r = 0; r < V; ++r)
        if (present[r]) names.emplace_back("w" + std::to_string(r), r);
    std::sort(names.begin(), names.end());
    const std::uint32_t NT = static_cast<std::uint32_t>(names.size());
    x->term_rank.resize(NT);
    x->rank_to_tid.assign(V, ~0u);
    x->term_offsets.resize(NT + 1);
    std::uint64_t off = 0;
    for (std::uint32_t t = 0; t < NT; ++t) {
        std::uint32_t r = names[t].second;
        x->term_rank[t] = r;
        x->rank_to_tid[r] = t;
        x->term_offsets[t] = off;
        off += df[r];
    }
    x->term_offsets[NT] = off;
    names.clear();
    names.shrink_to_fit();
    x->posting_rows.resize(off);
    x->posting_tf.resize(off);
    // per-thread cursors: tid start + rows owned by earlier threads
    std::vector<std::uint64_t> base(V, 0);
    for (std::uint32_t t = 0; t < NT; ++t) base[x->term_rank[t]] = x->term_offsets[t];
    std::vector<std::vector<std::uint64_t>> cur(T);
    for (int t = 0; t < T; ++t) {
        if (dfl[t].empty()) continue;
        cur[t].resize(V);
        for (std::uint32_t r = 0; r < V; ++r) {
            cur[t][r] = base[r];
            base[r] += dfl[t][r];
        }
        std::vector<std::uint32_t>().swap(dfl[t]);
    }
    parallel_ranges(n, T, [&](int t, std::size_t a, std::size_t e) {
        std::vector<std::uint32_t> buf;
        auto& cu = cur[t];
        for (std::size_t row = a; row < e; ++row) {
            distinct_tokens(c, recs[row], buf);
            for (std::size_t i = 0; i < buf.size();) {
                std::size_t j = i;
                while (j < buf.size() && buf[j] == buf[i]) ++j;
                std::uint64_t p = cu[buf[i]]++;
                x->posting_rows[p] = static_cast<std::uint32_t>(row);
                x->posting_tf[p] = static_cast<std::uint32_t>(j - i);
                i = j;
            }
        }
    });
    // statistics (csr_index.cpp:283-322)
    double len_sum = 0.0;
    for (auto l : x->doc_lens) len_sum += l;
    x->avgdl = global_df ? avgdl_global : n ? len_sum / static_cast<double>(n) : 0.0;
    x->idf.resize(NT);
    x->maxscore.assign(NT, 0.0);
    const std::uint32_t N32 = static_cast<std::uint32_t>(global_df ? n_global : n);
    const double avgdl = x->avgdl;
    parallel_ranges(NT, T, [&](int, std::size_t a, std::size_t e) {
        for (std::size_t t = a; t < e; ++t) {
            std::uint64_t lo = x->term_offsets[t], hi = x->term_offsets[t + 1];
            std::uint32_t dfv = static_cast<std::uint32_t>(global_df ? global_df[x->term_rank[t]] : hi - lo);
            double idf = std::log(1.0 + (static_cast<double>(N32) - dfv + 0.5) / (dfv + 0.5));
            x->idf[t] = idf;
            double ms = 0.0;
            for (std::uint64_t i = lo; i < hi; ++i) {
                double tf = static_cast<double>(x->posting_tf[i]);
                double dl = static_cast<double>(x->doc_lens[x->posting_rows[i]]);
                double norm = avgdl > 0.0 ? dl / avgdl : 1.0;
                double denom = tf + k1 * (1.0 - b + b * norm);
                double s = idf * tf * (k1 + 1.0) / denom;
                if (s > ms) ms = s;
            }
            x->maxscore[t] = ms;
        }
    });
    x->order_key = x->maxscore;  // a shard's caller replaces them by the global maxima
    return x.release();
}

}  // namespace

extern "C" {

int hm_synth_build(const hm_synth_corpus* c, double k1, double b,
                   const uint32_t* row_order, int threads, hm_synth_index** out) {
    return guard([&] {
        const std::uint64_t n = c->ts.size();
        std::vector<std::uint64_t> recs(n);
        for (std::uint64_t r = 0; r < n; ++r) {
            recs[r] = row_order ? row_order[r] : r;
            if (recs[r] >= n) throw std::invalid_argument("row_order out of range");
        }
        *out = build_rows(c, k1, b, recs, nullptr, 0, 0.0, n_threads(threads));
    });
}

int hm_synth_shard_counts(const hm_synth_corpus* c, uint64_t row_lo, uint64_t row_hi, int threads,
                          uint64_t* df, uint64_t* len_sum) {
    return guard([&] {
        const std::uint64_t n = c->ts.size();
        if (row_lo > row_hi || row_hi > n) throw std::invalid_argument("shard rows out of range");
        std::vector<std::uint64_t> recs(row_hi - row_lo);
        for (std::uint64_t r = row_lo; r < row_hi; ++r) recs[r - row_lo] = r;
        const auto dfl = count_df(c, recs, n_threads(threads));
        const std::uint32_t V = c->spec.vocab_size;
        std::fill(df, df + V, 0ull);
        for (const auto& d : dfl)
            if (!d.empty())
                for (std::uint32_t r = 0; r < V; ++r) df[r] += d[r];
        std::uint64_t s = 0;
        for (std::uint64_t r = row_lo; r < row_hi; ++r) s += c->offsets[r + 1] - c->offsets[r];
        *len_sum = s;
    });
}

int hm_synth_build_shard(const hm_synth_corpus* c, double k1, double b, uint64_t row_lo, uint64_t row_hi,
                         const uint64_t* global_df, uint64_t n_global, uint64_t len_sum_global, int threads,
                         hm_synth_index** out) {
    return guard([&] {
        const std::uint64_t n = c->ts.size();
        if (row_lo > row_hi || row_hi > n) throw std::invalid_argument("shard rows out of range");
        if (!global_df) throw std::invalid_argument("global_df is required");
        std::vector<std::uint64_t> recs(row_hi - row_lo);
        for (std::uint64_t r = row_lo; r < row_hi; ++r) recs[r - row_lo] = r;
        // the reference's avgdl: a double sum of the integral lengths (exact
        // below 2^53) over the flat corpus, divided by N
        const double avgdl = n_global ? static_cast<double>(len_sum_global) / static_cast<double>(n_global) : 0.0;
        *out = build_rows(c, k1, b, recs, global_df, n_global, avgdl, n_threads(threads));
    });
}

void hm_synth_index_destroy(hm_synth_index* x) { delete x; }
uint32_t hm_synth_index_n_terms(const hm_synth_index* x) {
    return static_cast<uint32_t>(x->term_rank.size());
}
uint64_t hm_synth_index_n_postings(const hm_synth_index* x) { return x->posting_rows.size(); }
uint32_t hm_synth_index_n_docs(const hm_synth_index* x) {
    return static_cast<uint32_t>(x->doc_ids.size());
}
double hm_synth_index_avgdl(const hm_synth_index* x) { return x->avgdl; }
const uint32_t* hm_synth_index_term_rank(const hm_synth_index* x) { return x->term_rank.data(); }
const uint32_t* hm_synth_index_rank_to_tid(const hm_synth_index* x) { return x->rank_to_tid.data(); }
const uint64_t* hm_synth_index_term_offsets(const hm_synth_index* x) { return x->term_offsets.data(); }
const uint32_t* hm_synth_index_posting_rows(const hm_synth_index* x) { return x->posting_rows.data(); }
const uint32_t* hm_synth_index_posting_tf(const hm_synth_index* x) { return x->posting_tf.data(); }
const double* hm_synth_index_idf(const hm_synth_index* x) { return x->idf.data(); }
const double* hm_synth_index_maxscore(const hm_synth_index* x) { return x->maxscore.data(); }
const double* hm_synth_index_order_key(const hm_synth_index* x) { return x->order_key.data(); }
const uint32_t* hm_synth_index_doc_lens(const hm_synth_index* x) { return x->doc_lens.data(); }
const uint64_t* hm_synth_index_doc_ids(const hm_synth_index* x) { return x->doc_ids.data(); }

// build_temporal_index bucketing, temporal_index.cpp:144-157
int hm_synth_partition(const hm_synth_corpus* c, int64_t window_ms, uint32_t* out_K,
                       uint32_t* row_order, uint32_t* part_row, int64_t* t0_out) {
    return guard([&] {
        if (window_ms <= 0) throw std::invalid_argument("window must be > 0");
        const std::uint64_t n = c->ts.size();
        if (n == 0) {
            *out_K = 0;
            return;
        }
        std::int64_t t0 = c->ts[0], t1 = t0;
        for (auto t : c->ts) {
            t0 = std::min(t0, t);
            t1 = std::max(t1, t);
        }
        std::uint32_t K = static_cast<std::uint32_t>((t1 - t0) / window_ms + 1);
        *out_K = K;
        if (t0_out) *t0_out = t0;
        if (!part_row) return;
        std::vector<std::uint64_t> cnt(K + 1, 0);
        for (auto t : c->ts) ++cnt[static_cast<std::size_t>((t - t0) / window_ms) + 1];
        for (std::uint32_t j = 0; j < K; ++j) cnt[j + 1] += cnt[j];
        for (std::uint32_t j = 0; j <= K; ++j) part_row[j] = static_cast<std::uint32_t>(cnt[j]);
        for (std::uint64_t i = 0; i < n; ++i) {
            std::size_t j = static_cast<std::size_t>((c->ts[i] - t0) / window_ms);
            row_order[cnt[j]++] = static_cast<std::uint32_t>(i);
        }
    });
}

}  // extern "C"
