// Host-safe constants and argument structs shared by the kernels and the
// C-ABI host code (no device intrinsics here; see hm_device.cuh).
#pragma once
#include <cstdint>

namespace hm {

constexpr int kThreads = 512;                 // threads per search CTA
constexpr int kWarps = kThreads / 32;
constexpr int kTileShift = 14;                // selection tile: 16384 rows
constexpr int kTile = 1 << kTileShift;
constexpr int kExactTileShift = 13;           // exact tile: 8192 rows (fp64)
constexpr int kExactTile = 1 << kExactTileShift;
constexpr int kMaxTerms = 256;                // distinct terms per query
constexpr int kCap = 2048;                    // selection candidate list
constexpr int kSurvCap = 512;                 // survivors rescored in fp64
constexpr int kExactCap = 1024;               // exact-kernel candidate list
constexpr int kMaxCodes = 256;                // (tf, len) code table entries
constexpr int kMaxK = 256;
constexpr uint32_t kNoTerm = 0xFFFFFFFFu;
constexpr int kLongFactor = 32;               // long term: df > 32 * n_tiles

struct DevIndex {
    const uint32_t* post;
    const uint32_t* tf;
    const uint64_t* term_off;
    const double* idf;
    const float* idf32;
    const double* order_key;
    const int32_t* long_slot;
    const uint32_t* tile_tab;
    const uint32_t* doc_lens;
    const uint64_t* doc_ids;
    const uint32_t* code_tf;   // [kMaxCodes]
    const uint32_t* code_len;  // [kMaxCodes]
    uint32_t n_terms, n_docs, n_tiles;
    uint32_t code_bits, n_codes, esc;
    double avgdl;
};

struct BatchArgs {
    uint32_t nq, k;
    const uint32_t* q_off;     // raw query tids (device)
    const uint32_t* q_tid;
    double k1, b;
    const double* tau;         // may be null
    double tau_default, eps;
    uint32_t row_lo, row_hi;
    uint32_t flags;
    const float* w32;          // [kMaxCodes] idf-free impacts for (k1, b)
    // planner scratch (device)
    uint32_t* plan_tid;        // [q_off[nq]] plan of query i at q_off[i]
    uint32_t* plan_mult;
    uint32_t* plan_len;        // [nq]
    uint64_t* cost;            // [nq] sum of df over the plan (LPT key)
    uint32_t* order;           // [nq] queries, most expensive first
    uint32_t* counters;        // [0]=work cursor approx, [1]=exact list size,
                               // [2]=work cursor exact, [3]=error flags
    uint32_t* exact_list;      // [nq]
    // results (device)
    uint64_t* out_ids;
    double* out_scores;
    uint32_t* out_n;
    double* out_conf;
    uint8_t* out_skip;
    uint64_t* out_post;
};

constexpr uint32_t kErrTooManyTerms = 1u;

}  // namespace hm
