/* oracle/bm25_oracle.h -- TEST INFRASTRUCTURE ONLY (the checker).
 *
 * Plain-C restatement of the reference hot path over raw CSR arrays, used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg to check the
 * CUDA path.  It is never linked into, or called by, the product.
 * Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj).
 *
 * Parity pinning: tests/test_oracle_*.py check this restatement against the
 * reference library itself (oracle/_ref/libhybridref.so, built from the
 * reference sources by oracle/Makefile) and against the committed golden
 * vectors in tests/golden/ generated from it.
 */
#ifndef BM25_ORACLE_H
#define BM25_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* src/csr_index.cpp:10-15 */
double or_bm25_score(double tf, double idf, double doc_len, double avgdl,
                     double k1, double b);

/* src/csr_index.cpp:19-22 */
double or_idf_from_df(uint32_t df, uint32_t n_docs);

/* src/csr_index.cpp:31-48.  tids[n] are vocab-resolved term ids; entries
 * equal to 0xFFFFFFFF are unknown terms and are dropped (csr_index.cpp:35-36).
 * Writes the plan (unique tids with multiplicity, canonical order) and
 * returns its length. */
uint32_t or_make_plan(const double* order_keys, const uint32_t* tids,
                      uint32_t n, uint32_t* plan_tid, uint32_t* plan_mult);

/* Exhaustive TAAT top-k, src/csr_index.cpp:77-104 + collect_topk :50-59 +
 * RankedList::sort_and_truncate include/hybrid/types.hpp:21-30, restricted to
 * rows in [row_lo, row_hi) (the full index when row_lo=0,row_hi=n_docs).
 * postings_touched counts every posting of every plan term (csr_index.cpp:100). */
int or_topk(const uint64_t* term_offsets, const uint32_t* posting_rows,
            const double* posting_weights, const double* idfs,
            uint32_t n_docs, const uint32_t* doc_lens, const uint64_t* doc_ids,
            double avgdl, const uint32_t* plan_tid, const uint32_t* plan_mult,
            uint32_t plan_len, uint64_t k, double k1, double b,
            uint32_t row_lo, uint32_t row_hi, uint64_t* out_ids,
            double* out_scores, uint32_t* out_n, uint64_t* postings_touched);

/* Batch of queries (plans concatenated, plan_off[nq+1]); output stride k. */
int or_topk_batch(const uint64_t* term_offsets, const uint32_t* posting_rows,
                  const double* posting_weights, const double* idfs,
                  uint32_t n_docs, const uint32_t* doc_lens,
                  const uint64_t* doc_ids, double avgdl,
                  const uint32_t* plan_off, const uint32_t* plan_tid,
                  const uint32_t* plan_mult, uint32_t nq, uint64_t k, double k1,
                  double b, uint32_t row_lo, uint32_t row_hi,
                  uint64_t* out_ids, double* out_scores, uint32_t* out_n,
                  uint64_t* postings_touched);

/* Learned-sparse bridge top-k, src/bridge.cpp:112-137 + collect :100-108.
 * Queries are concatenated sparse vectors q_off[nq+1]; output stride k. */
int or_bridge_topk_batch(const uint64_t* term_offsets, const uint32_t* posting_rows,
                         const double* posting_weights, uint32_t n_terms,
                         uint32_t n_docs, const uint64_t* doc_ids,
                         const uint64_t* q_off, const uint32_t* q_idx,
                         const double* q_val, uint32_t nq, uint64_t k,
                         uint32_t row_lo, uint32_t row_hi, uint64_t* out_ids,
                         double* out_scores, uint32_t* out_n,
                         uint64_t* postings_touched);

/* Dense channel: exact inner-product top-k, src/dense.cpp:86-101.
 * queries [nq x dim]; output stride k. */
int or_dense_topk_batch(const float* data, const uint64_t* ids, uint64_t count,
                        uint32_t dim, const float* queries, uint32_t nq,
                        uint64_t k, uint64_t* out_ids, double* out_scores,
                        uint32_t* out_n);

/* src/cascade.cpp:10-21 (Margin proxy) */
double or_margin(const double* scores, uint32_t n, double eps);
/* src/cascade.cpp:10-42 (proxy 0 Margin, 1 Top1Fraction, 2 EntropyComplement) */
double or_confidence(const double* scores, uint32_t n, int proxy, double eps);
/* src/cascade.cpp:79-84 */
int or_skip(double conf, double tau);

/* src/temporal_index.cpp:9-17; returns 0 on a domain error */
uint32_t or_k_star(double epsilon, double lambda);
/* src/temporal_index.cpp:78-80: min(k*, k_max, K) */
uint32_t or_temporal_budget(double epsilon, double lambda, uint32_t k_max,
                            uint32_t n_partitions);

/* src/eval.cpp:14-61, exponential gain (linear=0) or linear gain (linear=1) */
double or_ndcg_at_k(const uint64_t* ids, uint32_t n, const uint64_t* rel_docs,
                    const uint32_t* rel_grades, uint32_t n_rel, uint64_t k,
                    int linear);

/* src/twophase.cpp:18-64: the reference's CPU spec of the GPU two-phase top-k.
 * `slots` is caller-owned state of `capacity` (score,doc,valid) triples that
 * persists across calls exactly like TwoPhaseSelector::buffer_. */
typedef struct {
    double score;
    uint64_t doc;
    int valid;
} or_slot;
void or_twophase_init(or_slot* slots, uint64_t capacity);
int or_twophase_select(or_slot* slots, uint64_t capacity, int reset_sentinel,
                       const double* scores, uint64_t n, uint64_t k,
                       uint64_t* out_ids, double* out_scores, uint32_t* out_n);

#ifdef __cplusplus
}
#endif
#endif
