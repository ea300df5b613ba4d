// Host-safe constants and argument structs shared by the kernels and the
// C-ABI host code (no device intrinsics here; see hm_device.cuh).
//
// HBM layout of an index (built once by hm_index_create, host/hm_index.cpp):
//   post[P+8]    u32 packed postings, term-major, rows strictly increasing:
//                 * LONG terms (df > kLongFactor * n_tiles, with a tile table):
//                   (tile-local row << 18) | code18   -- 14-bit row inside the
//                   kTile-row tile, code18 < n_codes names a (tf, doc_len)
//                   pair of the code table, code18 == kEscLong means "read tf[]
//                   and doc_lens[]";
//                 * SHORT terms: (global row << cb) | code_cb   (cb = min(8,
//                   32 - row_bits)); only the n_codes_short most frequent
//                   pairs are addressable, the all-ones code escapes.
//                 4 B per posting; +8 words of padding for 16-B bulk copies.
//   tf[P]        u32 raw term frequency (escapes and exact rescoring only)
//   term_off[V+1] u64, idf[V] f64 (exact), idf32[V] f32 (selection),
//   order_key[V] f64 (plan order), long_slot[V] i32 (-1 = short),
//   tile_tab[n_long][16*n_tiles+1] u32: offset, relative to the term start,
//                 of the first posting of every 1024-row sub-tile (long terms
//                 only); tile j starts at entry 16*j.
//   doc_lens[N] u32, doc_ids[N] u64, code_tf/code_len[kMaxCodes] u32.
//   bk[]         u32 BAKED long-term postings for one (k1, b) (bake_kernel),
//                 in their own index space: the range of long term `slot` in
//                 2048-row unit u (= the rows a search-kernel warp owns in one
//                 tile) is bk[bk_base[slot] + bk_uoff[slot][u] ..
//                 bk_base[slot] + bk_uoff[slot][u+1]), padded to a multiple
//                 of 4 words and 16-byte aligned.  Word = (q19 << 13) | off13:
//                   q19 = float_bits(w * 2^-ks) >> 7 -- the idf-free impact
//                         w = tf*(k1+1)/(tf + k1*(1-b+b*len/avgdl)) scaled
//                         into the 7 lowest normal binades (exponent field
//                         1..7) and truncated to 16 mantissa bits (relative
//                         error < 2^-16); q19 = 0 is a NULL posting (padding);
//                   off13 = (swz10(r) & 2047) * 4, r = tile-local row: the
//                         byte offset of the row's accumulator inside the unit,
//                         XOR-swizzled so that read-modify-writes of dense runs
//                         of rows (lane strides 1, 2, 4 .. 32) are
//                         bank-conflict-free.
//                 Decoding is one shift: float(word >> 6) is w * 2^-ks with
//                 the offset's top 7 bits below the kept mantissa bits (error
//                 < 2^-16), and a NULL decodes to a denormal that the kernel's
//                 flush-to-zero multiply turns into an exact 0.
#pragma once
#include <cstdint>

namespace hm {

constexpr int kThreads = 512;                 // consumer / plain CTA threads
constexpr int kWarps = kThreads / 32;
constexpr int kTileShift = 14;                // selection tile: 16384 rows
constexpr int kTile = 1 << kTileShift;
constexpr int kMaxTerms = 256;                // distinct terms per query
constexpr int kCap = 2048;                    // selection candidate list
constexpr int kPruneAt = 512;                 // prune the list beyond this
constexpr int kSurvCap = 512;                 // survivors rescored in fp64
constexpr int kExactCap = 1024;               // exact-kernel candidate list
constexpr int kMaxCodes = 4096;               // (tf, len) code table entries
constexpr uint32_t kCodeMask = kMaxCodes - 1; // long codes < kCodeMask; w32[kCodeMask] = 0
constexpr int kSubShift = 10;                 // sub-tile (one consumer warp's rows): 1024
constexpr int kSubPerTile = 1 << (14 - kSubShift);
constexpr int kLocalBits = 14;                // long-term posting: local row bits
constexpr int kCodeBitsLong = 32 - kLocalBits;
constexpr uint32_t kEscLong = (1u << kCodeBitsLong) - 1;
constexpr int kMaxK = 256;
constexpr uint32_t kNoTerm = 0xFFFFFFFFu;
#ifndef HM_SHORT_TAB_MIN_DF
#define HM_SHORT_TAB_MIN_DF 256
#endif
constexpr uint32_t kShortTabMinDf = HM_SHORT_TAB_MIN_DF;
constexpr uint32_t kNoTabRow = 0xFFFFFFFFu;
constexpr int kLongFactor = 32;               // long term: df > 32 * n_tiles
constexpr int kBakeMantBits = 16;             // baked impact: 3 exponent + 16 mantissa bits
constexpr int kBakeBinades = 7;               // normal exponent fields 1..7
constexpr int kUnitShift = 11;                // search-kernel warp unit: 2048 rows
constexpr int kUnitsPerTile = 1 << (kTileShift - kUnitShift);
constexpr int kSubPerUnit = 1 << (kUnitShift - kSubShift);
constexpr int kScoreShift = 61;               // fp32 selection scores are score * 2^-61
constexpr int kShortCodes = 1024;             // smem impact table of the first codes (short terms use < 256)
static_assert(kLocalBits == kTileShift, "local row field must cover one tile");

struct DevIndex {
    const uint32_t* post;
    const uint32_t* tf;
    const uint64_t* term_off;
    const double* idf;
    const float* idf32;
    const double* order_key;
    const int32_t* long_slot;
    const uint8_t* long_esc;   // [n_long] 1 if the long term has escaped postings
    const uint32_t* tile_tab;
    // short terms with df >= kShortTabMinDf: the offset (from the term's start)
    // of the first posting of every tile, [row][n_tiles + 1] (row from
    // short_tab_row, kNoTabRow otherwise) -- the kernels' per-query short-term
    // tables are filled from it instead of scanning the postings
    const uint32_t* short_tab;
    const uint32_t* short_tab_row;
    const uint32_t* doc_lens;
    const uint64_t* doc_ids;
    const uint32_t* code_tf;   // [kMaxCodes]
    const uint32_t* code_len;  // [kMaxCodes]
    uint32_t n_terms, n_docs, n_tiles;
    uint32_t code_bits;        // short-term code field width
    uint32_t esc_short;        // all-ones short code
    uint32_t n_codes;          // codes usable by long terms (< kMaxCodes)
    uint32_t n_codes_short;    // codes usable by short terms (< esc_short)
    double avgdl;
    const uint32_t* bk;        // baked long-term postings (see above)
    const uint64_t* bk_base;   // [n_long] start of each long term's baked ranges
    const uint32_t* bk_uoff;   // [n_long][n_units + 1] unit offsets relative to bk_base
    uint32_t n_units;          // n_tiles * kUnitsPerTile
    uint32_t bk_ks;            // impact scale exponent: stored value = w * 2^-ks
    const float* tmax;         // [n_terms] max idf-free impact of the term (baked; bounds of the seeded kernel)
    // dense probe arrays of the most frequent long terms (seeded kernel):
    // dense[d * n_docs + row] = the posting's (tf, len) code, kDenseAbsent if
    // the term lacks the row, kDenseEscape if the pair has no code
    const uint16_t* dense;
    const int32_t* dense_of_slot;  // [n_long] d or -1
};
constexpr uint16_t kDenseAbsent = 0xFFFF;
constexpr uint16_t kDenseEscape = 0xFFFE;
#ifndef HM_SEED_SCRATCH
#define HM_SEED_SCRATCH (2 * 131072)
#endif
constexpr uint32_t kSeedScratch = HM_SEED_SCRATCH;  // words per CTA (search_seed.cu: kSeedMaxDf scores + rows)
#ifndef HM_NE_PEND_CAP
#define HM_NE_PEND_CAP 8192
#endif
constexpr uint32_t kNePendCap = HM_NE_PEND_CAP;  // essential-term sweep: pending rows per warp
#ifndef HM_NE_MIN_TERMS
#define HM_NE_MIN_TERMS 8
#endif
constexpr uint32_t kNeMinTerms = HM_NE_MIN_TERMS;  // plans the essential-term sweep serves
constexpr int kMaxDense = 128;             // dense arrays: long terms with df >= n_docs / 32, largest first
constexpr int kDenseMinDiv = 32;

// swizzled position of a row (only bits 0-4 change, from bits 5-9); an involution
#ifdef __CUDACC__
#define HM_HD __host__ __device__ __forceinline__
#else
#define HM_HD inline
#endif
HM_HD uint32_t swz10(uint32_t r) { return r ^ ((r >> 5) & 31u); }

struct BatchArgs {
    uint32_t nq, k;
    const uint32_t* q_off;     // raw query tids (device)
    const uint32_t* q_tid;
    double k1, b;
    const double* tau;         // may be null
    double tau_default, eps;
    uint32_t row_lo, row_hi;
    uint32_t flags;
    // intra-query split (small batches): split > 1 makes query q a slab
    // query -- real query q % nq_real over the split's (q / nq_real)-th of
    // [row_lo, row_hi); plan arrays are per real query, results per slab
    // query (merged afterwards by merge_kernel)
    uint32_t split, nq_real;
    const uint32_t* slab_row;  // [split + 1] explicit slab boundaries (partitions), or null:
                               // equal slabs of [row_lo, row_hi)
    const float* w32;          // [kMaxCodes] idf-free impacts for (k1, b)
    // planner scratch (device)
    uint32_t* plan_tid;        // [q_off[nq]] plan of query i at q_off[i]
    uint32_t* plan_mult;
    uint32_t* plan_len;        // [nq]
    uint64_t* cost;            // [nq] sum of df over the plan (LPT key)
    uint32_t* order;           // [nq] queries, most expensive first
    uint64_t* cost_seed;       // [nq] the seeded pass's cost proxy: postings of the plan terms with at
                               // most kSeedScratch / 2 postings (its seeds and essential candidates)
    const uint32_t* order_seed;  // [nq] queries by cost_seed descending (the seeded pass's LPT), or null
    uint32_t* counters;        // [0]=work cursor (seeded or exhaustive), [1]=exact list size,
                               // [2]=work cursor exact, [3]=error flags,
                               // [4]=queries handed over, [5]=exhaustive cursor after the seeded pass,
                               // [6]=wide list size, [7]=essential-term sweep cursor,
                               // [8]=plans of kNeMinTerms..32 terms (16 words)
    uint32_t* exact_list;      // [nq]
    uint32_t* wide_list;       // [nq] queries with more than kMaxTerms distinct terms
                               // (counters[6] entries) for the wide path (wide.cu);
                               // null: such a query sets kErrTooManyTerms
    uint32_t* fb_list;         // [nq] 1 = the seeded kernel handed the query to the
                               // exhaustive kernel (which walks `order` with cursor
                               // counters[5] and skips the others); null: every query
    uint32_t* stab;            // per-CTA short-term tile tables
    uint32_t* seed_scratch;    // per-CTA seeded-pass scratch: 2 * seed_half words (scores, rows)
    uint64_t* ne_pend;         // essential-term sweep: per CTA and warp kNePendCap rows awaiting
                               // completion, (score bits << 32) | row
    const float* ext_bound;    // [nq_real] doc shards: lower bound on the k-th selection score of the
                               // union of the shards (MAX over the shards' out_bound), or null
    float* out_bound;          // [nq_real] the seeded pass's bound of this index (kFlagBoundOnly: only that)
    uint32_t seed_half;        // min(kSeedScratch / 2, n_docs): the largest seed set of the index
    uint32_t stab_stride;      // words per short term (>= n_tiles + 2)
    // results (device)
    uint64_t* out_ids;
    double* out_scores;
    uint32_t* out_n;
    double* out_conf;
    uint8_t* out_skip;
    uint64_t* out_post;
};

// The wide path (kernels/wide.cu): any k, any plan length, fp64 exhaustive.
struct WideState {
    uint64_t pre_hi, pre_lo;   // key prefix of the k-th document found so far
    uint64_t post;             // postings_touched of the query
    uint32_t kr;               // rank of the k-th document inside the prefix group
    uint32_t done, take_all;   // selection finished; every positive document qualifies
    uint32_t n_c;              // candidates emitted
};
struct WideCand {
    uint32_t g;                // query slot in the group (sort key 1)
    uint64_t bits;             // score bits (desc), 0 = padding
    uint64_t id;               // DocId (asc)
};
struct WideArgs {
    uint32_t G;                // queries in the group
    const uint32_t* qlist;     // [G] batch query indices
    uint32_t span;             // rows of the window
    double* scores;            // [G][span] fp64 scores
    uint32_t* hist;            // [G][256]
    WideState* st;             // [G]
    WideCand* cand;            // [G][k]
};

// doc-sharded search (hm_sharded_*): each shard's exact local top-k lists,
// device pointers readable from the merging device (its own HBM or a peer's
// over NVLink), for gather_merge_kernel (shard_merge.cu)
constexpr int kMaxShards = 16;
struct ShardLists {
    uint32_t G;
    const uint64_t* ids[kMaxShards];     // [nq][k]
    const double* scores[kMaxShards];    // [nq][k]
    const uint32_t* n[kMaxShards];       // [nq]
    const uint64_t* post[kMaxShards];    // [nq] or NULL
};

constexpr uint32_t kFlagBoundOnly = 512u;  // HM_FLAG_BOUND_ONLY
// an external bound (seed or sweep domain, score * 2^-61) used as a bound of
// the other domain: both are within delta < 2^-15 of the exact score
constexpr float kExtSlack = 1.0f - 1e-4f;
// doc shards' bound exchange (shard_merge.cu): every shard's [nq][k] best seed scores
struct BoundLists {
    uint32_t G;
    const float* b[kMaxShards];
};
constexpr uint32_t kErrTooManyTerms = 1u;
constexpr uint32_t kErrNoConverge = 2u;

}  // namespace hm
