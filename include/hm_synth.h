/* include/hm_synth.h -- native synthetic workload generator and CSR builder.
 *
 * B200-side host tooling for the benchmark inputs.  These functions produce
 * BIT-IDENTICAL inputs to the reference generator and index builder, but
 * multithreaded and without materialising token strings, so the 8.84M-doc
 * corpora of BASELINE.json configs 2/4/5 can be built on the GPU box in
 * seconds:
 *
 *   hm_synth_corpus   replaces  hybrid::gen_corpus      src/workload.cpp:47-82
 *   hm_synth_queries  replaces  hybrid::gen_queries     src/workload.cpp:84-135
 *   hm_synth_build    replaces  hybrid::build_index     src/csr_index.cpp:232-324
 *                     for corpora whose tokens are the generator's "w<rank>"
 *                     words (never stopwords, so every tokenizer mode except
 *                     Porter/Full keeps them verbatim).
 *   hm_synth_build_temporal   the flat build + partition row order of
 *                     hybrid::build_temporal_index  src/temporal_index.cpp:125-169
 *
 * Term ids follow the reference: terms sorted alphabetically by their string
 * ("w0" < "w1" < "w10" < ...), tid = position.  Tokens are exchanged as Zipf
 * rank indices r (the token string is "w" + decimal(r)).
 * All functions return 0 on success, nonzero on error (hm_synth_last_error()).
 */
#ifndef HM_SYNTH_H
#define HM_SYNTH_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hm_synth_corpus hm_synth_corpus;
typedef struct hm_synth_queries hm_synth_queries;
typedef struct hm_synth_index hm_synth_index;

/* fields of hybrid::WorkloadSpec (include/hybrid/workload.hpp:12-25) */
typedef struct {
    uint64_t n_records;
    uint64_t seed;
    double recency_mass;
    double recency_window;
    uint32_t vocab_size;
    double zipf_s;
    uint32_t min_doc_tokens;
    uint32_t max_doc_tokens;
    uint32_t n_sessions;
    uint32_t n_agents;
    int64_t time_span_ms;
    int64_t t0_ms;
} hm_wspec;

/* fields of hybrid::QuerySpec (include/hybrid/workload.hpp:27-33) */
typedef struct {
    uint64_t n_queries;
    uint32_t min_terms;
    uint32_t max_terms;
    double paraphrase_noise;
    uint64_t seed;
} hm_qspec;

/* reference defaults */
void hm_wspec_default(hm_wspec* w);
void hm_qspec_default(hm_qspec* q);

const char* hm_synth_last_error(void);

int hm_synth_corpus_create(const hm_wspec* spec, int threads, hm_synth_corpus** out);
void hm_synth_corpus_destroy(hm_synth_corpus* c);
uint64_t hm_synth_corpus_n(const hm_synth_corpus* c);
uint64_t hm_synth_corpus_n_tokens(const hm_synth_corpus* c);
/* borrowed pointers valid until destroy: token ranks [n_tokens], token
 * offsets [n+1], timestamps [n]; doc id of record i is i (workload.cpp:57) */
const uint32_t* hm_synth_corpus_tokens(const hm_synth_corpus* c);
const uint64_t* hm_synth_corpus_offsets(const hm_synth_corpus* c);
const int64_t* hm_synth_corpus_ts(const hm_synth_corpus* c);

int hm_synth_queries_create(const hm_synth_corpus* c, const hm_qspec* q,
                            hm_synth_queries** out);
void hm_synth_queries_destroy(hm_synth_queries* q);
uint64_t hm_synth_queries_n(const hm_synth_queries* q);
/* query terms as ranks in generation order; term offsets [n+1]; one gold doc
 * per query; query timestamps; paraphrased flag ("syn_" terms never match) */
const uint32_t* hm_synth_queries_terms(const hm_synth_queries* q);
const uint64_t* hm_synth_queries_offsets(const hm_synth_queries* q);
const uint64_t* hm_synth_queries_gold(const hm_synth_queries* q);
const int64_t* hm_synth_queries_ts(const hm_synth_queries* q);
const uint8_t* hm_synth_queries_paraphrased(const hm_synth_queries* q);

/* Build the flat CSR index (build params k1,b define maxscores/order keys).
 * row_order may be NULL (insertion order, the flat index) or a permutation
 * of records (row r holds record row_order[r]); order keys/idf/avgdl are
 * always the flat corpus statistics. */
int hm_synth_build(const hm_synth_corpus* c, double k1, double b,
                   const uint32_t* row_order, int threads, hm_synth_index** out);
void hm_synth_index_destroy(hm_synth_index* x);
uint32_t hm_synth_index_n_terms(const hm_synth_index* x);
uint64_t hm_synth_index_n_postings(const hm_synth_index* x);
uint32_t hm_synth_index_n_docs(const hm_synth_index* x);
double hm_synth_index_avgdl(const hm_synth_index* x);
const uint32_t* hm_synth_index_term_rank(const hm_synth_index* x);   /* [V'] */
const uint32_t* hm_synth_index_rank_to_tid(const hm_synth_index* x); /* [vocab_size], ~0u absent */
const uint64_t* hm_synth_index_term_offsets(const hm_synth_index* x);/* [V'+1] */
const uint32_t* hm_synth_index_posting_rows(const hm_synth_index* x);/* [P] */
const uint32_t* hm_synth_index_posting_tf(const hm_synth_index* x);  /* [P] */
const double* hm_synth_index_idf(const hm_synth_index* x);           /* [V'] */
const double* hm_synth_index_maxscore(const hm_synth_index* x);      /* [V'] */
const double* hm_synth_index_order_key(const hm_synth_index* x);     /* [V'] */
const uint32_t* hm_synth_index_doc_lens(const hm_synth_index* x);    /* [N] */
const uint64_t* hm_synth_index_doc_ids(const hm_synth_index* x);     /* [N] */

/* Doc-range shard [row_lo, row_hi) of the flat index, built by the rank that
 * serves it: phase 1 counts the shard's document frequencies
 * (df[vocab_size], by Zipf rank) and length sum; the caller sums them over the
 * ranks (an all-reduce); phase 2 builds the shard's postings (rows
 * renumbered from 0, doc ids global) with the GLOBAL idf and avgdl -- the
 * reference's SharedStats (csr_index.hpp:28-35), so shard scores are the flat
 * scores bit for bit.  Term ids are the flat index's (every term with a
 * global df).  The shard's maxscore is its LOCAL maximum: order keys are the
 * max over the ranks (a MAX all-reduce), set by the caller. */
int hm_synth_shard_counts(const hm_synth_corpus* c, uint64_t row_lo, uint64_t row_hi, int threads,
                          uint64_t* df, uint64_t* len_sum);
int hm_synth_build_shard(const hm_synth_corpus* c, double k1, double b, uint64_t row_lo, uint64_t row_hi,
                         const uint64_t* global_df, uint64_t n_global, uint64_t len_sum_global, int threads,
                         hm_synth_index** out);

/* Temporal partitioning of a corpus (temporal_index.cpp:144-167):
 * window index of each record, partition count K, and the row order that lays
 * records out partition by partition (stable insertion order inside a
 * partition) plus the first row of every partition part_row[K+1]. */
int hm_synth_partition(const hm_synth_corpus* c, int64_t window_ms,
                       uint32_t* out_K, uint32_t* row_order /*[n]*/,
                       uint32_t* part_row /*[K+1], may be NULL to size*/,
                       int64_t* t0_out);

#ifdef __cplusplus
}
#endif
#endif
