/* oracle/bm25_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker).
 *
 * Plain-C restatement of the reference's BM25 hot path.  See bm25_oracle.h for
 * the contract; every function cites the reference file:line it restates
 * (relative to /root/reference/proj).  Built by oracle/Makefile with
 * -ffp-contract=off so no FMA contraction changes score bits (the reference is
 * built without -march and therefore without FMA, SURVEY.md finding 2).
 *
 * Parity: pinned against the reference library (oracle/_ref) and the golden
 * vectors in tests/golden/ by tests/test_oracle.py.
 */
#include "bm25_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* src/csr_index.cpp:10-15.  Operation order matters for bit parity:
 *   norm  = avgdl > 0 ? doc_len / avgdl : 1
 *   denom = tf + k1 * ((1 - b) + b * norm)
 *   score = ((idf * tf) * (k1 + 1)) / denom                                 */
double or_bm25_score(double tf, double idf, double doc_len, double avgdl,
                     double k1, double b) {
    double norm = avgdl > 0.0 ? doc_len / avgdl : 1.0;
    double denom = tf + k1 * (1.0 - b + b * norm);
    return idf * tf * (k1 + 1.0) / denom;
}

/* src/csr_index.cpp:19-22 */
double or_idf_from_df(uint32_t df, uint32_t n_docs) {
    return log(1.0 + ((double)n_docs - (double)df + 0.5) / ((double)df + 0.5));
}

/* ---- plan: src/csr_index.cpp:31-48 ------------------------------------ */
static const double* g_keys; /* qsort context (single-threaded oracle) */

static int plan_cmp(const void* a, const void* b) {
    uint32_t ta = ((const uint32_t*)a)[0], tb = ((const uint32_t*)b)[0];
    double ka = g_keys[ta], kb = g_keys[tb];
    if (ka != kb) return ka > kb ? -1 : 1; /* descending order key */
    return ta < tb ? -1 : (ta > tb ? 1 : 0); /* ties: ascending tid */
}

uint32_t or_make_plan(const double* order_keys, const uint32_t* tids,
                      uint32_t n, uint32_t* plan_tid, uint32_t* plan_mult) {
    /* unique tids with multiplicity (unknown terms dropped, :35-36) */
    uint32_t* pairs = (uint32_t*)malloc(sizeof(uint32_t) * 2 * (n ? n : 1));
    uint32_t m = 0;
    for (uint32_t i = 0; i < n; ++i) {
        if (tids[i] == 0xFFFFFFFFu) continue;
        uint32_t j = 0;
        while (j < m && pairs[2 * j] != tids[i]) ++j;
        if (j == m) {
            pairs[2 * m] = tids[i];
            pairs[2 * m + 1] = 0;
            ++m;
        }
        pairs[2 * j + 1]++;
    }
    g_keys = order_keys;
    qsort(pairs, m, 2 * sizeof(uint32_t), plan_cmp);
    for (uint32_t j = 0; j < m; ++j) {
        plan_tid[j] = pairs[2 * j];
        plan_mult[j] = pairs[2 * j + 1];
    }
    free(pairs);
    return m;
}

/* ---- canonical ranking: include/hybrid/types.hpp:21-25 ----------------- */
typedef struct {
    uint64_t id;
    double score;
} entry;

/* returns 1 if a ranks strictly before b (score desc, id asc) */
static int better(const entry* a, const entry* b) {
    if (a->score != b->score) return a->score > b->score;
    return a->id < b->id;
}
static int entry_cmp(const void* a, const void* b) {
    const entry* x = (const entry*)a;
    const entry* y = (const entry*)b;
    if (better(x, y)) return -1;
    if (better(y, x)) return 1;
    return 0;
}

/* bounded selection: heap whose root is the WORST kept entry.  The output of
 * "sort everything, truncate to k" (types.hpp:27-30) is identical because
 * `better` is a strict total order over distinct doc ids. */
static void sift_down(entry* h, uint64_t n, uint64_t i) {
    for (;;) {
        uint64_t l = 2 * i + 1, r = l + 1, w = i;
        if (l < n && better(&h[w], &h[l])) w = l;
        if (r < n && better(&h[w], &h[r])) w = r;
        if (w == i) return;
        entry t = h[i];
        h[i] = h[w];
        h[w] = t;
        i = w;
    }
}
static void sift_up(entry* h, uint64_t i) {
    while (i) {
        uint64_t p = (i - 1) / 2;
        if (!better(&h[p], &h[i])) return;
        entry t = h[i];
        h[i] = h[p];
        h[p] = t;
        i = p;
    }
}

/* collect (src/csr_index.cpp:50-59; bridge.cpp:100-108): rows with acc > 0,
 * best k by (score desc, id asc); resets acc/seen of the visited rows */
static void collect_best(double* acc, unsigned char* seen, const uint32_t* rows,
                         uint32_t n_rows, const uint64_t* doc_ids, uint64_t k,
                         uint64_t* out_ids, double* out_scores, uint32_t* out_n) {
    uint64_t cap = k < n_rows ? k : n_rows;
    entry* heap = (entry*)malloc(sizeof(entry) * (cap ? cap : 1));
    uint64_t hn = 0;
    for (uint32_t i = 0; i < n_rows; ++i) {
        uint32_t row = rows[i];
        double sc = acc[row];
        acc[row] = 0.0;
        seen[row] = 0;
        if (!(sc > 0.0) || cap == 0) continue;
        entry e = {doc_ids[row], sc};
        if (hn < cap) {
            heap[hn] = e;
            sift_up(heap, hn++);
        } else if (better(&e, &heap[0])) {
            heap[0] = e;
            sift_down(heap, hn, 0);
        }
    }
    qsort(heap, hn, sizeof(entry), entry_cmp);
    for (uint64_t i = 0; i < hn; ++i) {
        out_ids[i] = heap[i].id;
        out_scores[i] = heap[i].score;
    }
    *out_n = (uint32_t)hn;
    free(heap);
}

/* ---- exhaustive top-k: src/csr_index.cpp:77-104, collect_topk :50-59 --- */
static int topk_one(const uint64_t* term_offsets, const uint32_t* posting_rows,
                    const double* posting_weights, const double* idfs,
                    uint32_t n_docs, const uint32_t* doc_lens,
                    const uint64_t* doc_ids, double avgdl,
                    const uint32_t* plan_tid, const uint32_t* plan_mult,
                    uint32_t plan_len, uint64_t k, double k1, double b,
                    uint32_t row_lo, uint32_t row_hi, double* acc,
                    unsigned char* seen, uint32_t* rows, uint64_t* out_ids,
                    double* out_scores, uint32_t* out_n, uint64_t* touched_out) {
    (void)n_docs;
    uint64_t touched = 0;
    uint32_t n_rows = 0;
    for (uint32_t i = 0; i < plan_len; ++i) {
        uint32_t tid = plan_tid[i], mult = plan_mult[i];
        double idf = idfs[tid];
        uint64_t begin = term_offsets[tid], end = term_offsets[tid + 1];
        for (uint64_t j = begin; j < end; ++j) {
            uint32_t row = posting_rows[j];
            if (row < row_lo || row >= row_hi) continue;
            double s = or_bm25_score(posting_weights[j], idf,
                                     (double)doc_lens[row], avgdl, k1, b);
            for (uint32_t m = 0; m < mult; ++m) acc[row] += s; /* :94 */
            if (!seen[row]) {
                seen[row] = 1;
                rows[n_rows++] = row;
            }
            ++touched;
        }
    }
    if (touched_out) *touched_out = touched;
    collect_best(acc, seen, rows, n_rows, doc_ids, k, out_ids, out_scores, out_n);
    return 0;
}

int or_topk(const uint64_t* term_offsets, const uint32_t* posting_rows,
            const double* posting_weights, const double* idfs,
            uint32_t n_docs, const uint32_t* doc_lens, const uint64_t* doc_ids,
            double avgdl, const uint32_t* plan_tid, const uint32_t* plan_mult,
            uint32_t plan_len, uint64_t k, double k1, double b,
            uint32_t row_lo, uint32_t row_hi, uint64_t* out_ids,
            double* out_scores, uint32_t* out_n, uint64_t* postings_touched) {
    uint32_t plan_off[2] = {0, plan_len};
    return or_topk_batch(term_offsets, posting_rows, posting_weights, idfs,
                         n_docs, doc_lens, doc_ids, avgdl, plan_off, plan_tid,
                         plan_mult, 1, k, k1, b, row_lo, row_hi, out_ids,
                         out_scores, out_n, postings_touched);
}

int or_topk_batch(const uint64_t* term_offsets, const uint32_t* posting_rows,
                  const double* posting_weights, const double* idfs,
                  uint32_t n_docs, const uint32_t* doc_lens,
                  const uint64_t* doc_ids, double avgdl,
                  const uint32_t* plan_off, const uint32_t* plan_tid,
                  const uint32_t* plan_mult, uint32_t nq, uint64_t k, double k1,
                  double b, uint32_t row_lo, uint32_t row_hi,
                  uint64_t* out_ids, double* out_scores, uint32_t* out_n,
                  uint64_t* postings_touched) {
    if (row_hi > n_docs) row_hi = n_docs;
    size_t nd = n_docs ? n_docs : 1;
    double* acc = (double*)calloc(nd, sizeof(double));
    unsigned char* seen = (unsigned char*)calloc(nd, 1);
    uint32_t* rows = (uint32_t*)malloc(nd * sizeof(uint32_t));
    if (!acc || !seen || !rows) {
        free(acc);
        free(seen);
        free(rows);
        return -1;
    }
    for (uint32_t q = 0; q < nq; ++q) {
        topk_one(term_offsets, posting_rows, posting_weights, idfs, n_docs,
                 doc_lens, doc_ids, avgdl, plan_tid + plan_off[q],
                 plan_mult + plan_off[q], plan_off[q + 1] - plan_off[q], k, k1,
                 b, row_lo, row_hi, acc, seen, rows, out_ids + (size_t)q * k,
                 out_scores + (size_t)q * k, out_n + q,
                 postings_touched ? postings_touched + q : 0);
    }
    free(acc);
    free(seen);
    free(rows);
    return 0;
}

/* ---- learned-sparse bridge: src/bridge.cpp:112-137 (+ collect :100-108) --
 * Query q owns q_idx/q_val[q_off[q] .. q_off[q+1]) (a validated
 * SparseVector: strictly increasing term ids, values > 0).  Terms >= n_terms
 * are skipped (:122); S[row] += w_q * W in ascending term-id order (:127);
 * postings_touched counts each term's whole list (:133), restricted here to
 * rows in [row_lo, row_hi) like or_topk. */
int or_bridge_topk_batch(const uint64_t* term_offsets, const uint32_t* posting_rows,
                         const double* posting_weights, uint32_t n_terms,
                         uint32_t n_docs, const uint64_t* doc_ids,
                         const uint64_t* q_off, const uint32_t* q_idx,
                         const double* q_val, uint32_t nq, uint64_t k,
                         uint32_t row_lo, uint32_t row_hi, uint64_t* out_ids,
                         double* out_scores, uint32_t* out_n,
                         uint64_t* postings_touched) {
    if (row_hi > n_docs) row_hi = n_docs;
    size_t nd = n_docs ? n_docs : 1;
    double* acc = (double*)calloc(nd, sizeof(double));
    unsigned char* seen = (unsigned char*)calloc(nd, 1);
    uint32_t* rows = (uint32_t*)malloc(nd * sizeof(uint32_t));
    if (!acc || !seen || !rows) {
        free(acc);
        free(seen);
        free(rows);
        return -1;
    }
    for (uint32_t q = 0; q < nq; ++q) {
        uint64_t touched = 0;
        uint32_t n_rows = 0;
        for (uint64_t i = q_off[q]; i < q_off[q + 1]; ++i) {
            uint32_t t = q_idx[i];
            if (t >= n_terms) continue;
            double wq = q_val[i];
            for (uint64_t j = term_offsets[t]; j < term_offsets[t + 1]; ++j) {
                uint32_t row = posting_rows[j];
                if (row < row_lo || row >= row_hi) continue;
                acc[row] += wq * posting_weights[j];
                if (!seen[row]) {
                    seen[row] = 1;
                    rows[n_rows++] = row;
                }
                ++touched;
            }
        }
        if (postings_touched) postings_touched[q] = touched;
        collect_best(acc, seen, rows, n_rows, doc_ids, k, out_ids + (size_t)q * k,
                     out_scores + (size_t)q * k, out_n + q);
    }
    free(acc);
    free(seen);
    free(rows);
    return 0;
}

/* ---- dense channel: src/dense.cpp:86-101 --------------------------------
 * dot = sum_j double(r_j) * q_j, j ascending; EVERY row ranked by
 * (score desc, id asc) (sort_and_truncate over all rows: no score filter). */
int or_dense_topk_batch(const float* data, const uint64_t* ids, uint64_t count,
                        uint32_t dim, const float* queries, uint32_t nq,
                        uint64_t k, uint64_t* out_ids, double* out_scores,
                        uint32_t* out_n) {
    uint64_t cap = k < count ? k : count;
    entry* heap = (entry*)malloc(sizeof(entry) * (cap ? cap : 1));
    if (!heap) return -1;
    for (uint32_t q = 0; q < nq; ++q) {
        const float* qv = queries + (size_t)q * dim;
        uint64_t hn = 0;
        for (uint64_t i = 0; i < count && cap; ++i) {
            const float* r = data + i * dim;
            double dot = 0.0;
            for (uint32_t j = 0; j < dim; ++j) dot += (double)r[j] * (double)qv[j];
            entry e = {ids[i], dot};
            if (hn < cap) {
                heap[hn] = e;
                sift_up(heap, hn++);
            } else if (better(&e, &heap[0])) {
                heap[0] = e;
                sift_down(heap, hn, 0);
            }
        }
        qsort(heap, hn, sizeof(entry), entry_cmp);
        for (uint64_t i = 0; i < hn; ++i) {
            out_ids[(size_t)q * k + i] = heap[i].id;
            out_scores[(size_t)q * k + i] = heap[i].score;
        }
        out_n[q] = (uint32_t)hn;
    }
    free(heap);
    return 0;
}

/* ---- cascade trigger: src/cascade.cpp:10-42, :79-84 --------------------- */
double or_confidence(const double* s, uint32_t n, int proxy, double eps) {
    if (n == 0 || s[0] <= 0.0) return 0.0;
    if (proxy == 0) { /* Margin */
        if (n < 2) return 0.0;
        return (s[0] - s[1]) / (s[0] > eps ? s[0] : eps);
    }
    double sum = 0.0;
    for (uint32_t i = 0; i < n; ++i) sum += s[i];
    if (proxy == 1) return s[0] / (sum > eps ? sum : eps); /* Top1Fraction */
    if (proxy == 2) {                                       /* EntropyComplement */
        if (n < 2 || sum <= 0.0) return 0.0;
        double h = 0.0;
        for (uint32_t i = 0; i < n; ++i) {
            double pi = s[i] / sum;
            if (pi > 0.0) h -= pi * log(pi);
        }
        return 1.0 - h / log((double)n);
    }
    return 0.0;
}
double or_margin(const double* scores, uint32_t n, double eps) {
    return or_confidence(scores, n, 0, eps);
}
int or_skip(double conf, double tau) { return conf >= tau; }

/* ---- temporal budget: src/temporal_index.cpp:9-17, :78-80 --------------- */
uint32_t or_k_star(double epsilon, double lambda) {
    if (!(epsilon > 0.0 && epsilon < 1.0)) return 0;
    if (!(lambda > 0.0)) return 0;
    double v = ceil(log(1.0 / epsilon) / lambda);
    if (v < 1.0) v = 1.0;
    return (uint32_t)v;
}
uint32_t or_temporal_budget(double epsilon, double lambda, uint32_t k_max,
                            uint32_t n_partitions) {
    uint32_t ks = or_k_star(epsilon, lambda);
    uint32_t b = ks < k_max ? ks : k_max;
    return b < n_partitions ? b : n_partitions;
}

/* ---- nDCG: src/eval.cpp:14-61 ------------------------------------------- */
static int grade_desc(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x > y ? -1 : (x < y ? 1 : 0);
}
double or_ndcg_at_k(const uint64_t* ids, uint32_t n, const uint64_t* rel_docs,
                    const uint32_t* rel_grades, uint32_t n_rel, uint64_t k,
                    int linear) {
    if (k == 0) return -2.0; /* reference throws invalid_argument */
    uint32_t* g = (uint32_t*)malloc(sizeof(uint32_t) * (n_rel ? n_rel : 1));
    uint32_t ng = 0;
    for (uint32_t i = 0; i < n_rel; ++i)
        if (rel_grades[i] > 0) g[ng++] = rel_grades[i];
    qsort(g, ng, sizeof(uint32_t), grade_desc);
    double ideal = 0.0;
    for (uint64_t i = 0; i < k && i < ng; ++i) {
        double gain = linear ? (double)g[i] : exp2((double)g[i]) - 1.0;
        ideal += gain / log2((double)(i + 2));
    }
    free(g);
    if (ideal <= 0.0) return -1.0;
    double dcg = 0.0;
    for (uint64_t i = 0; i < k && i < n; ++i) {
        uint32_t r = 0;
        for (uint32_t j = 0; j < n_rel; ++j)
            if (rel_docs[j] == ids[i]) r = rel_grades[j];
        if (r == 0) continue;
        double gain = linear ? (double)r : exp2((double)r) - 1.0;
        dcg += gain / log2((double)(i + 2));
    }
    return dcg / ideal;
}

/* ---- two-phase selector: src/twophase.cpp:9-64 -------------------------- */
void or_twophase_init(or_slot* slots, uint64_t capacity) {
    for (uint64_t i = 0; i < capacity; ++i) {
        slots[i].score = -INFINITY;
        slots[i].doc = 0;
        slots[i].valid = 0;
    }
}

int or_twophase_select(or_slot* slots, uint64_t capacity, int reset_sentinel,
                       const double* scores, uint64_t n, uint64_t k,
                       uint64_t* out_ids, double* out_scores, uint32_t* out_n) {
    if (k == 0 || k > capacity) return -1; /* twophase.cpp:20-22 */
    if (reset_sentinel) or_twophase_init(slots, capacity); /* :24-27 */
    uint64_t lanes = capacity / k;
    if (lanes < 1) lanes = 1;
    entry* local = (entry*)malloc(sizeof(entry) * (k + 1));
    for (uint64_t lane = 0; lane < lanes; ++lane) {
        uint64_t ln = 0;
        for (uint64_t d = lane; d < n; d += lanes) {
            if (scores[d] <= 0.0) continue;
            entry c = {d, scores[d]};
            uint64_t pos = 0; /* lower_bound under `better` */
            while (pos < ln && better(&local[pos], &c)) ++pos;
            if (ln < k || pos != ln) {
                memmove(&local[pos + 1], &local[pos], (ln - pos) * sizeof(entry));
                local[pos] = c;
                if (ln < k) ++ln;
            }
        }
        for (uint64_t i = 0; i < ln; ++i) {
            slots[lane * k + i].score = local[i].score;
            slots[lane * k + i].doc = local[i].id;
            slots[lane * k + i].valid = 1;
        }
    }
    free(local);
    /* phase 2 (:49-61): valid positive slots, sorted, deduplicated, first k */
    entry* c = (entry*)malloc(sizeof(entry) * capacity);
    uint64_t nc = 0;
    for (uint64_t i = 0; i < capacity; ++i)
        if (slots[i].valid && slots[i].score > 0.0) {
            c[nc].id = slots[i].doc;
            c[nc].score = slots[i].score;
            ++nc;
        }
    qsort(c, nc, sizeof(entry), entry_cmp);
    uint64_t w = 0;
    for (uint64_t i = 0; i < nc; ++i) {
        if (w && c[w - 1].id == c[i].id && c[w - 1].score == c[i].score) continue;
        c[w++] = c[i];
    }
    uint32_t m = 0;
    for (uint64_t i = 0; i < w && m < k; ++i, ++m) {
        out_ids[m] = c[i].id;
        out_scores[m] = c[i].score;
    }
    *out_n = m;
    free(c);
    return 0;
}
