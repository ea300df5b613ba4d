// hm_dropin_bench -- the reference's own C++ search API on the B200 path at
// BASELINE scale, the way hybridmem drives it (measurement tool).
//
// The corpus and queries come from the reference's gen_corpus / gen_queries
// and the index from its build_index (workload.o, csr_index.o: the
// reference's objects, search symbols weakened).  Two ways a C++ caller
// searches it through the drop-in (csrc/dropin/hybrid_b200.cpp):
//   1. per query: CsrIndex::bm25_topk called from `workers` threads, each
//      thread taking the next query -- hybridmem's parallel_for loop
//      (tools/hybridmem.cpp:58-71, 305-313); every call is one single-query
//      GPU batch (row slabs: one query spread over the SMs);
//   2. batch: hybrid_b200::bm25_topk_batch over all queries (one GPU batch).
// Both are checked against each other query by query (ids and score bits);
// the reference CPU answers on the same inputs are bench.py's parity block
// (tests/golden/fullsize_c2).
// Prints one JSON line: qps and per-query latency p50/p95/p99 (report_latency's
// ceil(p n) - 1 rule, hybridmem.cpp:82-93) of both.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "hybrid/csr_index.hpp"
#include "hybrid/workload.hpp"
#include "hybrid_b200.hpp"

namespace {

double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

double pctl(std::vector<double> v, double p) {  // report_latency: v[ceil(p n) - 1]
    if (v.empty()) return 0.0;
    std::sort(v.begin(), v.end());
    std::size_t i = static_cast<std::size_t>(std::ceil(p * static_cast<double>(v.size())));
    return v[std::min(v.size() - 1, i ? i - 1 : 0)];
}

}  // namespace

int main(int argc, char** argv) {
    std::uint64_t n_records = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 8841823ull;
    std::uint64_t n_queries = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 10000ull;
    unsigned workers = argc > 3 ? static_cast<unsigned>(std::atoi(argv[3])) : std::thread::hardware_concurrency();
    std::uint32_t vocab = argc > 4 ? static_cast<std::uint32_t>(std::atoi(argv[4])) : 1000000u;
    if (workers == 0) workers = 1;
    const std::size_t k = 10;
    const hybrid::Bm25Params p{};

    double t0 = now_ms();
    hybrid::WorkloadSpec ws;
    ws.n_records = n_records;
    ws.vocab_size = vocab;
    ws.min_doc_tokens = vocab >= 1000000u ? 20 : 5;
    ws.max_doc_tokens = vocab >= 1000000u ? 60 : 30;
    const auto corpus = hybrid::gen_corpus(ws);
    hybrid::QuerySpec qs;
    qs.n_queries = n_queries;
    const auto queries = hybrid::gen_queries(corpus, qs, ws);
    std::vector<std::pair<hybrid::DocId, std::string>> docs;
    docs.reserve(corpus.size());
    for (const auto& r : corpus) docs.emplace_back(r.id, r.text);
    const hybrid::CsrIndex idx = hybrid::build_index(docs, hybrid::TokenizerMode::Stopword);
    docs.clear();
    docs.shrink_to_fit();
    const double build_s = (now_ms() - t0) / 1e3;
    std::vector<std::vector<std::string>> qterms;
    for (const auto& q : queries) qterms.push_back(q.terms);

    // warm-up: device upload, bake, workspaces (hybridmem's 32 warm-up queries)
    for (std::size_t i = 0; i < std::min<std::size_t>(32, qterms.size()); ++i) (void)idx.bm25_topk(qterms[i], k, p);
    (void)hybrid_b200::bm25_topk_batch(idx, qterms, k, p);

    // 1. per query under parallel_for(workers)
    std::vector<hybrid::RankedList> per(qterms.size());
    std::vector<double> lat(qterms.size());
    std::atomic<std::size_t> next{0};
    const double w0 = now_ms();
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < workers; ++t)
        pool.emplace_back([&] {
            for (;;) {
                const std::size_t i = next.fetch_add(1);
                if (i >= qterms.size()) return;
                const double s = now_ms();
                per[i] = idx.bm25_topk(qterms[i], k, p);
                lat[i] = now_ms() - s;
            }
        });
    for (auto& th : pool) th.join();
    const double per_ms = now_ms() - w0;

    // 2. one batch (three repetitions, the median)
    std::vector<double> bt;
    std::vector<hybrid::RankedList> bat;
    for (int r = 0; r < 3; ++r) {
        const double s = now_ms();
        bat = hybrid_b200::bm25_topk_batch(idx, qterms, k, p);
        bt.push_back(now_ms() - s);
    }
    std::sort(bt.begin(), bt.end());
    const double batch_ms = bt[1];

    std::size_t mismatch = 0;
    for (std::size_t i = 0; i < qterms.size(); ++i) {
        bool same = per[i].size() == bat[i].size();
        for (std::size_t j = 0; same && j < per[i].size(); ++j)
            same = per[i].entries[j].first == bat[i].entries[j].first &&
                   std::memcmp(&per[i].entries[j].second, &bat[i].entries[j].second, sizeof(double)) == 0;
        mismatch += same ? 0 : 1;
    }
    std::printf(
        "{\"tool\": \"hm_dropin_bench\", \"n_docs\": %zu, \"n_queries\": %zu, \"k\": %zu, \"build_s\": %.1f, "
        "\"per_query\": {\"api\": \"hybrid::CsrIndex::bm25_topk (drop-in) under parallel_for\", \"workers\": %u, "
        "\"qps\": %.1f, \"p50_ms\": %.4f, \"p95_ms\": %.4f, \"p99_ms\": %.4f}, "
        "\"batch\": {\"api\": \"hybrid_b200::bm25_topk_batch\", \"qps\": %.1f, \"batch_ms\": %.3f}, "
        "\"per_query_equals_batch\": %s, \"mismatches\": %zu}\n",
        static_cast<std::size_t>(idx.num_docs()), qterms.size(), k, build_s, workers, 1e3 * static_cast<double>(qterms.size()) / per_ms,
        pctl(lat, 0.50), pctl(lat, 0.95), pctl(lat, 0.99), 1e3 * static_cast<double>(qterms.size()) / batch_ms,
        batch_ms, mismatch ? "false" : "true", mismatch);
    return mismatch ? 1 : 0;
}
