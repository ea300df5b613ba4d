// hm_search -- the `hybridmem search` batch loop (tools/hybridmem.cpp:169-331)
// on the B200 path, for the BM25 modes bm25 | maxscore | temporal.
//
// Same inputs, outputs and conventions as cmd_search:
//   * --config / HYBRID_* environment overrides (load_config,
//     apply_env_overrides), HIDX / HTIX magic check with the same
//     "mode/index mismatch" message, load_index / load_temporal_index,
//     load_queries_tsv -- the reference's own io.o / config.o, linked;
//   * a discarded warm-up over the first 32 queries, then the measured pass;
//   * report_latency's "latency ms (warm): p50=.. p95=.. p99=.." line (the
//     ceil(p * n) - 1 percentile rule, :82-93) -- a query's latency is the
//     wall time of the GPU batch that served it;
//   * save_run_trec (TREC 6-column, %.17g scores, tag = --tag or the mode);
//   * --stats: "# config_hash=<hash>" then qid,postings_touched,
//     partitions_searched,escalated (:321-329).
// What differs is the loop: instead of one bm25_topk per query under
// parallel_for(--workers), queries go to the GPU in batches of --batch
// (default: all of them) through hybrid_b200::bm25_topk_batch /
// temporal_topk_batch (include/hybrid_b200.hpp).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "hybrid/config.hpp"
#include "hybrid/csr_index.hpp"
#include "hybrid/io.hpp"
#include "hybrid/temporal_index.hpp"
#include "hybrid_b200.hpp"

namespace {

double now_ms() {
    using namespace std::chrono;
    return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

[[noreturn]] void usage(const char* msg) {
    std::fprintf(stderr,
                 "%s\nusage: hm_search [--config PATH] --index PATH --queries PATH [--mode bm25|maxscore|temporal]\n"
                 "                 [--k K] [--batch N] [--tag TAG] [--stats CSV] --out RUN\n",
                 msg);
    std::exit(2);
}

}  // namespace

int main(int argc, char** argv) {
    std::string config_path, index_path, queries_path, mode = "bm25", tag, stats_out, out;
    std::size_t k = 10, batch = 0;
    for (int i = 1; i < argc; ++i) {
        const std::string a = argv[i];
        auto val = [&]() -> std::string {
            if (i + 1 >= argc) usage(("missing value for " + a).c_str());
            return argv[++i];
        };
        if (a == "--config") config_path = val();
        else if (a == "--index") index_path = val();
        else if (a == "--queries") queries_path = val();
        else if (a == "--mode") mode = val();
        else if (a == "--k") k = std::stoull(val());
        else if (a == "--batch") batch = std::stoull(val());
        else if (a == "--tag") tag = val();
        else if (a == "--stats") stats_out = val();
        else if (a == "--out") out = val();
        else if (a == "--workers") val();  // accepted for command-line parity; the GPU batch replaces the pool
        else usage(("unknown option " + a).c_str());
    }
    if (index_path.empty() || queries_path.empty() || out.empty()) usage("--index, --queries and --out are required");
    try {
        hybrid::RunConfig cfg = hybrid::load_config(config_path);
        hybrid::apply_env_overrides(cfg);
        if (mode != "bm25" && mode != "maxscore" && mode != "temporal")
            throw std::runtime_error("unknown search mode: " + mode + " (hm_search serves bm25|maxscore|temporal)");
        const bool want_temporal = mode == "temporal";
        {
            std::ifstream probe(index_path, std::ios::binary);
            char magic[4] = {0};
            probe.read(magic, 4);
            const bool is_temporal = std::string(magic, 4) == "HTIX";
            if (want_temporal != is_temporal)
                throw std::runtime_error("mode/index mismatch: mode '" + mode + "' needs a " +
                                         (want_temporal ? "temporal (HTIX)" : "flat (HIDX)") + " index, got " +
                                         index_path);
        }
        hybrid::CsrIndex flat;
        hybrid::TemporalIndex temporal;
        if (want_temporal) temporal = hybrid::load_temporal_index(index_path);
        else flat = hybrid::load_index(index_path);
        const auto queries = hybrid::load_queries_tsv(queries_path);
        const std::size_t n = queries.size();
        std::vector<hybrid::RankedList> results(n);
        std::vector<std::uint64_t> postings(n, 0);
        std::vector<std::uint32_t> partitions(n, 0);

        // one GPU batch over queries [a, b)
        auto run = [&](std::size_t a, std::size_t b, bool record) {
            std::vector<std::vector<std::string>> terms;
            terms.reserve(b - a);
            for (std::size_t i = a; i < b; ++i) terms.push_back(queries[i].terms);
            if (want_temporal) {
                std::vector<hybrid::TemporalStats> st;
                auto r = hybrid_b200::temporal_topk_batch(temporal, terms, k, cfg.bm25, &st);
                if (!record) return;
                for (std::size_t i = a; i < b; ++i) {
                    results[i] = std::move(r[i - a]);
                    postings[i] = st[i - a].postings_touched;
                    partitions[i] = st[i - a].partitions_searched;
                }
            } else {
                std::vector<hybrid::SearchStats> st;
                auto r = hybrid_b200::bm25_topk_batch(flat, terms, k, cfg.bm25, &st);
                if (!record) return;
                for (std::size_t i = a; i < b; ++i) {
                    results[i] = std::move(r[i - a]);
                    postings[i] = st[i - a].postings_touched;
                }
            }
        };

        run(0, std::min<std::size_t>(n, 32), false);  // warm-up (discarded): uploads the index
        const std::size_t B = batch ? batch : std::max<std::size_t>(n, 1);
        std::vector<double> lat(n);
        const double t_all = now_ms();
        for (std::size_t a = 0; a < n; a += B) {
            const std::size_t b = std::min(n, a + B);
            const double t0 = now_ms();
            run(a, b, true);
            const double dt = now_ms() - t0;
            for (std::size_t i = a; i < b; ++i) lat[i] = dt;
        }
        const double wall = now_ms() - t_all;
        if (n) {
            std::vector<double> v = lat;
            std::sort(v.begin(), v.end());
            auto pct = [&](double p) {
                const auto i = static_cast<std::size_t>(std::ceil(p * static_cast<double>(v.size())));
                return v[i ? i - 1 : 0];
            };
            std::fprintf(stderr, "latency ms (warm): p50=%.4f p95=%.4f p99=%.4f\n", pct(0.50), pct(0.95), pct(0.99));
            std::fprintf(stderr, "throughput: %zu queries in %.3f ms (%.0f queries/s), %zu GPU batch(es) of <= %zu\n", n,
                         wall, wall > 0 ? 1000.0 * static_cast<double>(n) / wall : 0.0, (n + B - 1) / B, B);
        }
        std::vector<std::pair<std::string, hybrid::RankedList>> runfile;
        runfile.reserve(n);
        for (std::size_t i = 0; i < n; ++i) runfile.emplace_back("q" + std::to_string(i + 1), std::move(results[i]));
        hybrid::save_run_trec(runfile, tag.empty() ? mode : tag, out);
        if (!stats_out.empty()) {
            std::ofstream csv(stats_out, std::ios::trunc);
            if (!csv) throw std::runtime_error("cannot write " + stats_out);
            csv << "# config_hash=" << hybrid::config_hash(cfg) << '\n'
                << "qid,postings_touched,partitions_searched,escalated\n";
            for (std::size_t i = 0; i < n; ++i)
                csv << 'q' << i + 1 << ',' << postings[i] << ',' << partitions[i] << ",0\n";
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
    return 0;
}
