// Test driver for the C++ drop-in (paper_2605_25092_b200/csrc/dropin/hybrid_b200.cpp).
// Linked with the reference's remaining objects (tokenizer, porter, ... but NOT
// csr_index.o / temporal_index.o) exactly as a maintainer would link the
// drop-in, it executes a line protocol on stdin and prints results; the pytest
// side (tests/test_dropin.py) computes the same calls on the unmodified
// reference library and compares bit patterns.
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "hybrid/bridge.hpp"
#include "hybrid/cascade.hpp"
#include "hybrid/csr_index.hpp"
#include "hybrid/dense.hpp"
#include "hybrid/temporal_index.hpp"
#include "hybrid_b200.hpp"

using namespace hybrid;

static std::string hexd(double v) {
    char buf[64];
    std::snprintf(buf, sizeof buf, "%a", v);
    return buf;
}

// "nnz i:v i:v ..." with hex-float values (exact)
static SparseVector read_vec(std::istream& in) {
    SparseVector v;
    std::size_t n = 0;
    in >> n;
    for (std::size_t i = 0; i < n; ++i) {
        std::string tok;
        in >> tok;
        const auto c = tok.find(':');
        v.indices.push_back(static_cast<std::uint32_t>(std::stoul(tok.substr(0, c))));
        v.values.push_back(std::strtod(tok.c_str() + c + 1, nullptr));
    }
    return v;
}

static void print_list(const RankedList& r, const std::string& extra) {
    std::cout << "R " << r.entries.size() << extra;
    for (const auto& [id, s] : r.entries) std::cout << ' ' << id << ':' << hexd(s);
    std::cout << '\n';
}

int main() {
    std::ios::sync_with_stdio(false);
    std::vector<std::pair<DocId, std::string>> docs;
    std::vector<MemoryRecord> recs;
    CsrIndex idx, bidx;
    TemporalIndex tidx;
    std::vector<std::pair<DocId, SparseVector>> bdocs;
    EmbeddingMatrix emb;
    std::uint32_t emb_dim = 0;
    std::uint64_t emb_seed = 0;
    std::vector<MemoryRecord> drecs;
    std::string line;
    while (std::getline(std::cin, line)) {
        std::istringstream in(line);
        std::string cmd;
        in >> cmd;
        try {
            if (cmd == "DOCS") {
                std::size_t n;
                in >> n;
                docs.clear();
                for (std::size_t i = 0; i < n; ++i) {
                    std::getline(std::cin, line);
                    auto tab = line.find('\t');
                    docs.emplace_back(std::stoull(line.substr(0, tab)), line.substr(tab + 1));
                }
            } else if (cmd == "INDEX") {
                int mode;
                double k1, b;
                in >> mode >> k1 >> b;
                idx = build_index(docs, static_cast<TokenizerMode>(mode), 50000, Bm25Params{k1, b});
                std::cout << "OK " << idx.num_docs() << ' ' << idx.num_postings() << '\n';
            } else if (cmd == "QUERY") {
                std::size_t k;
                double k1, b;
                int ms;
                in >> k >> k1 >> b >> ms;
                std::vector<std::string> q;
                for (std::string t; in >> t;) q.push_back(t);
                SearchStats st;
                st.postings_touched = 7;  // stats accumulate (csr_index.cpp:102)
                RankedList r = ms ? idx.bm25_topk_maxscore(q, k, Bm25Params{k1, b}, &st)
                                  : idx.bm25_topk(q, k, Bm25Params{k1, b}, &st);
                print_list(r, " " + std::to_string(st.postings_touched - 7));
            } else if (cmd == "TERMSCORE") {
                std::uint32_t t;
                std::uint64_t i;
                in >> t >> i;
                const double v = idx.bm25_term_score(t, i, Bm25Params{});  // may throw: print nothing first
                std::cout << "V " << hexd(v) << '\n';
            } else if (cmd == "UB") {
                std::vector<std::string> q;
                for (std::string t; in >> t;) q.push_back(t);
                const double v = idx.query_upper_bound(q);
                std::cout << "V " << hexd(v) << '\n';
            } else if (cmd == "RECORDS") {
                std::size_t n;
                in >> n;
                recs.clear();
                for (std::size_t i = 0; i < n; ++i) {
                    std::getline(std::cin, line);
                    std::istringstream r(line);
                    MemoryRecord m;
                    std::string rest;
                    r >> m.id >> m.ts_ms;
                    std::getline(r, rest);
                    m.text = rest.empty() ? rest : rest.substr(1);
                    recs.push_back(std::move(m));
                }
            } else if (cmd == "TEMPORAL") {
                TemporalParams tp;
                int mode;
                in >> tp.window_ms >> tp.epsilon >> tp.lambda_hat >> tp.k_max_partitions >> mode;
                tidx = build_temporal_index(recs, tp, static_cast<TokenizerMode>(mode));
                std::cout << "OK " << tidx.num_partitions() << '\n';
            } else if (cmd == "TQUERY") {
                std::size_t k;
                int ub;
                in >> k >> ub;
                std::vector<std::string> q;
                for (std::string t; in >> t;) q.push_back(t);
                TemporalStats st;
                RankedList r = tidx.topk(q, k, Bm25Params{}, &st, ub != 0);
                print_list(r, " " + std::to_string(st.partitions_searched));
            } else if (cmd == "QBATCH" || cmd == "TBATCH") {  // k ub n, then n query lines: one GPU batch
                std::size_t k, n;
                int ub;
                in >> k >> ub >> n;
                std::vector<std::vector<std::string>> qs(n);
                for (auto& q : qs) {
                    std::getline(std::cin, line);
                    std::istringstream ql(line);
                    for (std::string t; ql >> t;) q.push_back(t);
                }
                if (cmd == "QBATCH") {
                    std::vector<SearchStats> st;
                    std::vector<hybrid_b200::Decision> dec;
                    auto r = hybrid_b200::bm25_topk_batch(idx, qs, k, Bm25Params{}, &st, &dec, 0.10);
                    for (std::size_t i = 0; i < n; ++i)
                        print_list(r[i], " " + std::to_string(st[i].postings_touched) + " " + hexd(dec[i].conf) +
                                             " " + std::to_string(dec[i].skip ? 1 : 0));
                } else {
                    std::vector<TemporalStats> st;
                    auto r = hybrid_b200::temporal_topk_batch(tidx, qs, k, Bm25Params{}, &st, ub != 0);
                    for (std::size_t i = 0; i < n; ++i)
                        print_list(r[i], " " + std::to_string(st[i].partitions_searched) + " " +
                                             std::to_string(st[i].early_stopped ? 1 : 0));
                }
            } else if (cmd == "NCACHED") {
                std::cout << "V " << hybrid_b200::cached_device_indexes() << '\n';
            } else if (cmd == "BDOCS") {  // n lines of "id nnz i:v ..."
                std::size_t n;
                in >> n;
                bdocs.clear();
                for (std::size_t i = 0; i < n; ++i) {
                    std::getline(std::cin, line);
                    std::istringstream r(line);
                    DocId id;
                    r >> id;
                    bdocs.emplace_back(id, read_vec(r));
                }
            } else if (cmd == "BINGEST") {
                bidx = bridge_ingest(bdocs);
                std::cout << "OK " << bidx.num_docs() << ' ' << bidx.num_postings() << ' ' << hexd(bidx.avgdl)
                          << '\n';
            } else if (cmd == "BQUERY") {  // k ms nnz i:v ...
                std::size_t k;
                int ms;
                in >> k >> ms;
                const SparseVector q = read_vec(in);
                SearchStats st;
                st.postings_touched = 5;
                RankedList r = ms ? bridge_topk_maxscore(bidx, q, k, &st) : bridge_topk(bidx, q, k, &st);
                print_list(r, " " + std::to_string(st.postings_touched - 5));
            } else if (cmd == "BEXPORT") {  // one line: per doc "id:nnz" then the checksum of values
                auto v = bridge_export(bidx);
                std::cout << "E " << v.size();
                for (const auto& [id, sv] : v) {
                    std::cout << ' ' << id << ':' << sv.nnz();
                    for (std::size_t i = 0; i < sv.nnz(); ++i) std::cout << ',' << sv.indices[i] << '=' << hexd(sv.values[i]);
                }
                std::cout << '\n';
            } else if (cmd == "BVALIDATE") {
                read_vec(in).validate();
                std::cout << "OK\n";
            } else if (cmd == "BM25ONBRIDGE") {
                bidx.bm25_topk({"0"}, 5, Bm25Params{});
                std::cout << "OK\n";
            } else if (cmd == "BONBM25") {
                bridge_topk(idx, SparseVector{{0}, {1.0}}, 5);
                std::cout << "OK\n";
            } else if (cmd == "EMBDOCS") {  // dim seed: hash_embed every DOCS text
                in >> emb_dim >> emb_seed;
                emb = EmbeddingMatrix{};
                emb.dim = emb_dim;
                drecs.clear();
                for (const auto& [id, text] : docs) {
                    emb.add(id, hash_embed(text, emb_dim, emb_seed));
                    MemoryRecord r;
                    r.id = id;
                    r.ts_ms = static_cast<std::int64_t>(id) * 1000;
                    drecs.push_back(r);
                }
                std::cout << "OK " << emb.count() << '\n';
            } else if (cmd == "DQUERY") {  // k text...
                std::size_t k;
                in >> k;
                std::string text, t;
                while (in >> t) text += (text.empty() ? "" : " ") + t;
                print_list(dense_topk(emb, hash_embed(text, emb_dim, emb_seed), k), " 0");
            } else if (cmd == "DBADDIM") {
                dense_topk(emb, std::vector<float>(emb_dim + 1, 0.0f), 3);
                std::cout << "OK\n";
            } else if (cmd == "CASCADE") {  // k tau query_ts terms...
                std::size_t k;
                double tau;
                std::int64_t qts;
                in >> k >> tau >> qts;
                std::vector<std::string> q;
                for (std::string t; in >> t;) q.push_back(t);
                std::string text;
                for (const auto& t : q) text += (text.empty() ? "" : " ") + t;
                CascadeConfig cfg;
                cfg.conf_threshold = tau;
                RetrieveFn bm25_fn = [&](std::size_t kk) { return idx.bm25_topk_maxscore(q, kk, Bm25Params{}); };
                RetrieveFn dense_fn = [&](std::size_t kk) {
                    return dense_topk(emb, hash_embed(text, emb_dim, emb_seed), kk);
                };
                RecordLookup lookup = [&](DocId d) -> const MemoryRecord* {
                    for (const auto& r : drecs)
                        if (r.id == d) return &r;
                    return nullptr;
                };
                auto d = cascade_retrieve(k, cfg, bm25_fn, dense_fn, lookup, qts, FusionParams{});
                print_list(d.results, std::string(" ") + (d.escalated ? "1" : "0"));
            } else if (cmd == "KSTAR") {
                double e, l;
                in >> e >> l;
                const auto v = k_star(e, l);
                std::cout << "V " << v << '\n';
            } else {
                std::cout << "ERR unknown " << cmd << '\n';
            }
        } catch (const std::invalid_argument& e) {
            std::cout << "THROW invalid_argument " << e.what() << '\n';
        } catch (const std::out_of_range& e) {
            std::cout << "THROW out_of_range " << e.what() << '\n';
        } catch (const std::runtime_error& e) {
            std::cout << "THROW runtime_error " << e.what() << '\n';
        }
        std::cout.flush();
    }
    return 0;
}
