/* include/hm_b200.h -- C ABI of the B200-native BM25 search path.
 *
 * This is the drop-in boundary under the reference's C++ search API.  The
 * reference has no FFI of its own: its boundary is the C++
 * API in proj/include/hybrid/.  Each entry point below names the reference
 * interface it replaces.  The C++ drop-in (paper_2605_25092_b200/csrc/dropin/)
 * is compiled against the reference's own, unmodified headers -- used in
 * place, never copied into this repo -- and defines the reference's search
 * entry points on top of this ABI; include/hybrid_b200.hpp adds the batch
 * extension.  INTEGRATION.md shows the bindings (C++, ctypes) a maintainer
 * would add.
 *
 * Conventions: plain pointers and sizes only; every function returns
 * HM_OK (0) or a nonzero hm_status, with a thread-local message in
 * hm_last_error().  Host buffers are borrowed for the duration of the call.
 * An index is immutable after creation and hm_search_batch is re-entrant:
 * concurrent calls from many threads on one index are allowed (the
 * reference's concurrent const readers, tools/hybridmem.cpp:309)
 * and results do not depend on concurrency or batch composition.
 */
#ifndef HM_B200_H
#define HM_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    HM_OK = 0,
    HM_ERR_INVALID = 1,    /* std::invalid_argument in the reference */
    HM_ERR_RUNTIME = 2,    /* std::runtime_error (CUDA/NCCL failures map here) */
    HM_ERR_RANGE = 3,      /* std::out_of_range */
    HM_ERR_NO_DEVICE = 4   /* no usable sm_100 device: there is no CPU fallback */
} hm_status;

typedef struct hm_index hm_index;

/* Borrowed view of a hybrid::CsrIndex (proj/include/hybrid/csr_index.hpp:44-60).
 * Exactly one of posting_weights (the reference's raw-tf doubles) or
 * posting_tf must be non-NULL.  Rows must be strictly increasing per term. */
typedef struct {
    uint32_t n_terms;
    const uint64_t* term_offsets;     /* [n_terms + 1] */
    const uint32_t* posting_rows;     /* [P] */
    const double* posting_weights;    /* [P] raw tf as double, or NULL */
    const uint32_t* posting_tf;       /* [P] raw tf, or NULL */
    const double* term_idfs;          /* [n_terms] */
    const double* term_order_keys;    /* [n_terms] canonical accumulation order */
    uint32_t n_docs;
    const uint32_t* doc_lens;         /* [n_docs] */
    const uint64_t* doc_ids;          /* [n_docs] external DocId of each row */
    double avgdl;
} hm_csr_view;

/* Upload an index to `device` (HBM-resident until destroy).
 * Replaces: the in-memory CsrIndex produced by hybrid::build_index /
 * hybrid::load_index (src/csr_index.cpp:232-324, src/io.cpp:229-232). */
int hm_index_create(const hm_csr_view* view, int device, hm_index** out);
int hm_index_destroy(hm_index* index);

/* Device bytes held by the index (postings, tf, tables, per-doc arrays). */
uint64_t hm_index_device_bytes(const hm_index* index);
/* Packed posting format: bits of the row field and of the impact code. */
int hm_index_format(const hm_index* index, uint32_t* row_bits, uint32_t* code_bits,
                    uint32_t* n_codes, uint64_t* n_escaped);

/* One batch of queries.  Query i owns q_tid[q_off[i] .. q_off[i+1]):
 * vocabulary-resolved term ids in query order, duplicates allowed (they
 * become the plan multiplicity), 0xFFFFFFFF for an unknown term (dropped, as
 * in make_plan, src/csr_index.cpp:31-48).  Scoring is restricted to rows in
 * [row_lo, row_hi) (row_hi = 0 means n_docs): the temporal index's recency
 * window and doc-range shards use this. */
typedef struct {
    uint32_t n_queries;
    const uint32_t* q_off;     /* [n_queries + 1] */
    const uint32_t* q_tid;     /* [q_off[n_queries]] */
    uint32_t k;                /* top-k, any value; 0 gives empty results */
    double k1, b;              /* hybrid::Bm25Params */
    const double* tau;         /* [n_queries] per-query skip threshold, or NULL */
    double tau_default;        /* CascadeConfig::conf_threshold (0.10) */
    double epsilon_guard;      /* CascadeConfig::epsilon_guard (1e-9) */
    uint32_t row_lo, row_hi;
    uint32_t flags;            /* HM_FLAG_* */
    /* Doc-sharded search (optional; DEVICE pointers, hm_search_batch_device
     * only -- NULL for the other entry points), selection domain (score *
     * 2^-61, fp32).  With HM_FLAG_BOUND_ONLY only out_bound[n_queries * k] is
     * written: per query the k best complete scores of the seeded pass's seed
     * documents on this index (zeros where there are fewer).  ext_bound[i]:
     * a lower bound on the k-th score of the UNION of the shards -- the k-th
     * largest of all shards' out_bound values of query i: the search then
     * returns only documents that can be in the union's top-k (possibly fewer
     * than k) and the k-way merge of the shards' lists is the exact answer.
     * Both disable row slabs; k <= 256. */
    const float* ext_bound;
    float* out_bound;
} hm_query_batch;

#define HM_FLAG_FORCE_EXACT 1u   /* run every query on the exact fp64 kernel */
#define HM_FLAG_DEBUG_NO_RESET 2u /* test-only: skip the per-query sentinel reset
                                    of the candidate state (pitfall-3 witness,
                                    src/twophase.cpp:24-27) */
#define HM_FLAG_EXHAUSTIVE 16u    /* skip the seeded MaxScore pre-pass: every query on the
                                    exhaustive tile-sweep kernel (same results; the roofline
                                    measurement of bench.py) */
#define HM_FLAG_SEED_ALL 32u      /* test-only: the seeded pre-pass tries every query that
                                    has a short term, whatever its cost estimate or window */
#define HM_FLAG_NO_SPLIT 64u     /* keep one CTA per query in small batches (no intra-query row
                                    slabs; same results -- a test / measurement switch) */
#define HM_FLAG_NO_NESKIP 128u   /* test / measurement switch: no essential-term sweep -- the
                                    tile sweep streams every term of every query (same results) */
#define HM_FLAG_NE_ALL 256u      /* test / measurement switch: every query the tile sweep serves
                                    goes through its essential-term variant, whatever its plan
                                    length (same results) */
#define HM_FLAG_BOUND_ONLY 512u  /* compute only out_bound (the seeded pass's bound), see
                                    hm_query_batch.out_bound */
#define HM_FLAG_TIMING 4u         /* time each kernel with CUDA events on the
                                    launching stream (the call then synchronises);
                                    read back with hm_last_batch_timing */

/* Results, caller-allocated.  Row i of ids/scores has stride k; out_n[i] <= k
 * entries ranked by (score desc, DocId asc), zero scores never emitted
 * (RankedList::better / sort_and_truncate, include/hybrid/types.hpp:21-30;
 * collect_topk, src/csr_index.cpp:50-59).  conf = Margin confidence
 * (src/cascade.cpp:15-21); skip = conf >= tau (src/cascade.cpp:79-84);
 * postings = SearchStats::postings_touched of the exhaustive path
 * (src/csr_index.cpp:100-102; postings inside the row window). */
typedef struct {
    uint64_t* ids;       /* [n_queries * k] */
    double* scores;      /* [n_queries * k] */
    uint32_t* n;         /* [n_queries] */
    double* conf;        /* [n_queries], may be NULL */
    uint8_t* skip;       /* [n_queries], may be NULL */
    uint64_t* postings;  /* [n_queries], may be NULL */
} hm_results;

/* Batch search with HOST buffers (synchronous).
 * Replaces: per-query CsrIndex::bm25_topk / bm25_topk_maxscore
 * (include/hybrid/csr_index.hpp:72-79, src/csr_index.cpp:77-207) driven by
 * hybridmem's parallel_for batch loop (tools/hybridmem.cpp:227-313), plus
 * cascade::confidence + the skip decision (src/cascade.cpp:10-21, 67-92). */
int hm_search_batch(hm_index* index, const hm_query_batch* batch, hm_results* out);

/* The batch searched inside each of n_parts contiguous row ranges
 * [part_row[p], part_row[p+1]) separately (part_row ascending, <= n_docs; the
 * batch's row_lo/row_hi are ignored): one launch sequence whose (query, part)
 * pairs are scheduled together.  Results are per part, row-major
 * [n_parts][n_queries][k] (ids, scores), [n_parts][n_queries] (n, postings);
 * conf and skip are not written.  Replaces: the per-partition loop of
 * TemporalIndex::topk (src/temporal_index.cpp:72-123) -- every partition of
 * the budget at once over a partition-ordered flat index, the caller merging
 * the per-partition lists in the reference's order (its upper-bound stop
 * only decides which of them it keeps). */
int hm_search_batch_parts(hm_index* index, const hm_query_batch* batch, uint32_t n_parts,
                          const uint32_t* part_row, hm_results* out_parts);

/* Same with DEVICE buffers (batch arrays and results on the index's device),
 * ordered on `stream` (a cudaStream_t, NULL = legacy default): the launches
 * run on a pooled workspace stream that waits for `stream`, and `stream`
 * waits for them.  `n_queries` etc. are read from the host struct.  The call
 * is NOT fully asynchronous: it reads q_off back (a (n_queries + 1) x 4-byte
 * D2H on `stream`, synchronised) to size the plan scratch, and synchronises
 * the workspace stream before returning (the pinned staging of the impact
 * table is reused by the next call); results are complete on return. */
int hm_search_batch_device(hm_index* index, const hm_query_batch* batch_dev,
                           hm_results* out_dev, void* stream);

/* Per query of the last HM_FLAG_TIMING batch on this thread (one without
 * row slabs): 1 if it was served by the exhaustive tile sweep (handed over
 * by the seeded MaxScore pass, or the pass did not run), 0 if the seeded pass
 * served it.  HM_ERR_RANGE when n exceeds the batch. */
int hm_last_batch_handover(uint32_t* flags, uint32_t n);

/* Queries of the last batch on this thread that ran on the wide path
 * (kernels/wide.cu): every query when k > 256, else those whose plan has more
 * than 256 distinct terms.  The wide path scores exhaustively in fp64 in plan
 * order and ranks by an exact radix select + sort: any k, any query length,
 * the reference's bits (csr_index.hpp:72-79 has no cap on either). */
int hm_last_batch_wide(uint32_t* n_wide);

/* Statistics of the last batch on this thread: queries that fell back to the
 * exact fp64 kernel (candidate overflow or non-positive impacts), kernel
 * launches issued. */
int hm_last_batch_stats(uint32_t* n_exact_fallback, uint32_t* n_launches);

/* Device time (ms) of the last HM_FLAG_TIMING batch on this thread: planner +
 * LPT sort, the fused selection kernel, the exact fallback kernel. */
int hm_last_batch_timing(float* ms_plan, float* ms_search, float* ms_exact);

/* How the last batch on this thread was launched: 0 stream operations
 * (first sighting of these arguments, or HM_FLAG_TIMING), 1 captured into a
 * CUDA graph (second identical batch on the workspace), 2 replayed from it. */
int hm_last_batch_graph(uint32_t* mode);

/* The seeded MaxScore pre-pass of the last batch on this thread: its device
 * time (HM_FLAG_TIMING batches) and how many queries it handed to the
 * exhaustive kernel (0 with HM_FLAG_EXHAUSTIVE). */
int hm_last_batch_seed(float* ms_seed, uint32_t* n_handed_over);

/* Doc-sharded multi-GPU merge (the step after the all-gather of k candidates
 * per query): shard_ids/shard_scores/shard_n hold G blocks of per-shard exact
 * top-k results ([G][n_queries][k], [G][n_queries]).  Produces the global
 * top-k, Margin confidence and skip per query.  DEVICE pointers, on `stream`.
 * New in this framework (the reference has no sharded path; precedent:
 * SharedStats, csr_index.hpp:28-35). */
int hm_merge_shards_device(uint32_t n_shards, uint32_t n_queries, uint32_t k,
                           const uint64_t* shard_ids, const double* shard_scores,
                           const uint32_t* shard_n, const double* tau, double tau_default,
                           double epsilon_guard, hm_results* out_dev, void* stream);

/* Doc-sharded search over several devices of one process (north_star's
 * multi-GPU path for C++ callers; the torch.distributed one-rank-per-GPU
 * path is paper_2605_25092_b200/shard.py).  hm_sharded_create splits the
 * view's rows into n_shards contiguous ranges [n_docs*g/G, n_docs*(g+1)/G)
 * and uploads shard g -- its sub-CSR with the flat index's idf, order keys
 * and avgdl (SharedStats, csr_index.hpp:28-35), so every local score is the
 * flat score bit for bit -- to devices[g] (a device may be listed more than
 * once).  n_shards <= 16 and <= n_docs.  Peer access devices[0] -> devices[g]
 * is enabled where the hardware allows it (NVLink / NVSwitch).
 * hm_sharded_search_batch takes the hm_search_batch arguments (HOST buffers,
 * row window in flat rows, any k): every shard searches its part of the
 * window on its own device concurrently, then ONE kernel on devices[0] reads
 * the shards' top-k lists over peer memory and merges them (all-gather +
 * k-way merge fused; shards the root cannot address are copied first) and
 * writes Margin confidence, skip and postings_touched summed over shards.
 * Results equal hm_search_batch on the unsharded index.  Calls on one
 * hm_sharded are serialised.  hm_sharded_info: shard count, first flat row of
 * each shard ([n_shards + 1]), devices, and a bit per shard read by the
 * merge over peer memory. */
typedef struct hm_sharded hm_sharded;
int hm_sharded_create(const hm_csr_view* view, const int* devices, uint32_t n_shards, hm_sharded** out);
int hm_sharded_destroy(hm_sharded* sharded);
int hm_sharded_info(const hm_sharded* sharded, uint32_t* n_shards, uint32_t* shard_row, int* devices,
                    uint32_t* p2p_mask);
int hm_sharded_search_batch(hm_sharded* sharded, const hm_query_batch* batch, hm_results* out);

/* The reference's on-disk index, HIDX v1 (proj/src/io.cpp:91-157, 223-232):
 * parsed straight into host arrays, validated with the reference's messages
 * ("not an index file (bad magic)", "unsupported index version N",
 * "unsupported idf convention: X", "index file truncated reading <field>").
 * hm_hidx_view fills an hm_csr_view for hm_index_create (a BM25-mode index:
 * mode 0; a Bridge-mode file is rejected there with the reference's
 * "BM25 scoring requires a BM25-mode index"); hm_hidx_term returns the
 * length of term `tid` and points *s at its bytes (not NUL-terminated).
 * Replaces: hybrid::load_index (src/io.cpp:229-232) on the search path. */
typedef struct hm_hidx hm_hidx;
int hm_hidx_load(const char* path, hm_hidx** out);
const char* hm_hidx_last_error(void);
int hm_hidx_view(const hm_hidx* h, hm_csr_view* view, uint32_t* mode, double* build_k1,
                 double* build_b);
uint32_t hm_hidx_term(const hm_hidx* h, uint32_t tid, const char** s);
const double* hm_hidx_maxscores(const hm_hidx* h);
void hm_hidx_free(hm_hidx* h);

/* The reference's temporal container, HTIX v1 (proj/src/io.cpp:234-318),
 * assembled as ONE flat index whose rows are laid out partition by partition
 * (oldest first) over the shared statistics -- the layout hm_search_batch
 * scores the newest min(k*, k_max, K) partitions of with a row window
 * (TemporalIndex::topk, src/temporal_index.cpp:72-123).  hm_htix_flat is an
 * hm_hidx (view / terms / free it through hm_htix_free only); part_row has
 * n_partitions + 1 entries.  Errors as the reference reader ("not a temporal
 * index file (bad magic)", "unsupported temporal index version N", partition
 * bodies as HIDX).  Replaces: hybrid::load_temporal_index. */
typedef struct hm_htix hm_htix;
int hm_htix_load(const char* path, hm_htix** out);
const hm_hidx* hm_htix_flat(const hm_htix* t);
int hm_htix_partitions(const hm_htix* t, uint32_t* n_partitions, const uint32_t** part_row,
                       const int64_t** window_start, const int64_t** window_end);
int hm_htix_params(const hm_htix* t, int64_t* window_ms, double* epsilon, double* lambda_hat,
                   uint32_t* k_max, uint64_t* total_docs);
void hm_htix_free(hm_htix* t);

/* ---------------------------------------------------------------- bridge
 * Learned-sparse ("bridge") scoring: a Bridge-mode CsrIndex
 * (bridge_ingest, src/bridge.cpp:22-73: per-term postings of per-doc sparse
 * weight vectors; or a Bridge-mode HIDX file through hm_hidx_view, mode 1)
 * HBM-resident in the reference's layout, and top-k by
 * S[doc] = sum over query terms, in ascending term-id order, of w_q * W_t in
 * fp64 without contraction -- bit-identical to bridge_topk and
 * bridge_topk_maxscore (src/bridge.cpp:112-204, whose outputs are identical).
 * Replaces: hybrid::bridge_topk / bridge_topk_maxscore
 * (include/hybrid/bridge.hpp:29-40) per query. */
typedef struct hm_bridge hm_bridge;

typedef struct {
    uint32_t n_terms;
    const uint64_t* term_offsets;     /* [n_terms + 1] */
    const uint32_t* posting_rows;     /* [P], strictly increasing per term */
    const double* posting_weights;    /* [P] learned weights */
    uint32_t n_docs;
    const uint64_t* doc_ids;          /* [n_docs], distinct */
} hm_bridge_view;

int hm_bridge_create(const hm_bridge_view* view, int device, hm_bridge** out);
int hm_bridge_destroy(hm_bridge* bridge);

/* Queries are SparseVectors (bridge.hpp:12-19): query i owns
 * q_idx/q_val[q_off[i] .. q_off[i+1]).  The host entry point validates each
 * like SparseVector::validate (bridge.cpp:10-20; HM_ERR_INVALID with its
 * messages); term ids >= n_terms are skipped (bridge.cpp:122).  k <= 512
 * (HM_ERR_INVALID beyond; the reference's TwoPhaseSelector has the same kind
 * of capacity rule, twophase.cpp:12-22).  Rows are restricted to
 * [row_lo, row_hi) (row_hi = 0: n_docs).  max_nnz: an upper bound on every
 * query's nnz (0 = computed by the host entry point; required by the device
 * one).  Results as hm_results (conf and skip unused); postings =
 * SearchStats::postings_touched (bridge.cpp:133) within the row window. */
typedef struct {
    uint32_t n_queries;
    const uint64_t* q_off;     /* [n_queries + 1] */
    const uint32_t* q_idx;
    const double* q_val;
    uint32_t k;
    uint32_t row_lo, row_hi;
    uint32_t max_nnz;
    uint32_t flags;            /* HM_FLAG_TIMING */
} hm_bridge_batch;

int hm_bridge_search_batch(hm_bridge* bridge, const hm_bridge_batch* batch, hm_results* out);
int hm_bridge_search_batch_device(hm_bridge* bridge, const hm_bridge_batch* batch_dev,
                                  hm_results* out_dev, void* stream);
/* Device time (ms) of the last HM_FLAG_TIMING bridge batch on this thread. */
int hm_bridge_last_timing(float* ms_kernel);

/* ---------------------------------------------------------------- dense
 * The cascade's escalate channel: brute-force inner-product
 * top-k over a hybrid::EmbeddingMatrix (include/hybrid/dense.hpp:13-22: unit
 * vectors, row-major fp32, one DocId per row) held in HBM.  Scores are
 * sum_j double(r_j) * q_j in fp64, j ascending, every row ranked by
 * (score desc, DocId asc) -- bit-identical to hybrid::dense_topk
 * (src/dense.cpp:86-101).  When dim % 32 == 0 and k <= 32 the tensor cores
 * (tcgen05, TF32) select candidates within a proven error bound and fp64
 * rescoring ranks them; otherwise k <= 256 runs the fp64 list kernel and
 * larger k scores every row and sorts on the device.  A query whose
 * dim differs from the matrix's fails with the reference's
 * "query dimension mismatch" (HM_ERR_INVALID).  Results as hm_results
 * (conf, skip, postings unused).  Replaces: hybrid::dense_topk per query. */
typedef struct hm_dense hm_dense;

typedef struct {
    uint32_t dim;
    uint32_t count;
    const float* data;         /* [count * dim] row-major */
    const uint64_t* doc_ids;   /* [count] */
} hm_dense_view;

int hm_dense_create(const hm_dense_view* view, int device, hm_dense** out);
int hm_dense_destroy(hm_dense* dense);

typedef struct {
    uint32_t n_queries;
    uint32_t dim;
    const float* queries;      /* [n_queries * dim] */
    uint32_t k;
    uint32_t flags;            /* HM_FLAG_TIMING */
} hm_dense_batch;

int hm_dense_search_batch(hm_dense* dense, const hm_dense_batch* batch, hm_results* out);
int hm_dense_search_batch_device(hm_dense* dense, const hm_dense_batch* batch_dev,
                                 hm_results* out_dev, void* stream);
/* Device time (ms) of the last HM_FLAG_TIMING dense batch on this thread. */
int hm_dense_last_timing(float* ms_kernels);
/* Last dense batch on this thread: path (1 = tensor-core TF32 candidates +
 * fp64 rescoring, the default when dim % 32 == 0 and k <= 32; 2 = fp64
 * shared-memory lists, also forced by HM_FLAG_FORCE_EXACT; 3 = fp64 + device
 * sort for k > 256) and, for HM_FLAG_TIMING tensor-core batches, queries
 * whose candidate list overflowed (rescored over every row) and the total
 * number of candidates. */
int hm_dense_last_stats(uint32_t* path, uint32_t* n_overflow, uint64_t* n_candidates);

/* ---------------------------------------------------------------- strings
 * Query strings -> term ids (the vocabulary lookup of make_plan,
 * src/csr_index.cpp:31-48, and the whitespace split of load_queries_tsv,
 * src/io.cpp:389-391).  hm_vocab_create copies terms[tid] (the CsrIndex's
 * alphabetical `terms`; lens NULL = NUL-terminated).  hm_vocab_resolve splits
 * query i = text[text_off[i] .. text_off[i+1]) on C-locale whitespace and
 * writes q_off[n_queries + 1] and q_tid (0xFFFFFFFF for an unknown term) --
 * exactly hm_query_batch's q_off / q_tid; HM_ERR_RANGE when the tokens exceed
 * tid_cap (*n_tids holds the count).  n_threads 0 = hardware concurrency
 * (batches under 4,096 queries resolve on the calling thread). */
typedef struct hm_vocab hm_vocab;
int hm_vocab_create(const char* const* terms, const uint32_t* lens, uint32_t n_terms, hm_vocab** out);
void hm_vocab_destroy(hm_vocab* vocab);
uint32_t hm_vocab_size(const hm_vocab* vocab);
int hm_vocab_resolve(const hm_vocab* vocab, uint32_t n_queries, const char* text, const uint64_t* text_off,
                     uint32_t* q_off, uint32_t* q_tid, uint64_t tid_cap, uint64_t* n_tids, uint32_t n_threads);

/* Margin confidence over a ranked score list (src/cascade.cpp:10-21). */
double hm_margin(const double* scores, uint32_t n, double epsilon_guard);

const char* hm_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
