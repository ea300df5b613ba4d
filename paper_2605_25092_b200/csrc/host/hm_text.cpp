// Query strings -> term ids: the host half of make_plan (src/csr_index.cpp:
// 31-48, the vocab lookup) and of the query reader's whitespace split
// (load_queries_tsv, src/io.cpp:389-391: `std::istringstream >> term`).
//
// hm_vocab holds the index's terms (tid = position, the CsrIndex's `terms`)
// in one byte arena with an open-addressing hash table of (hash, tid) slots;
// hm_vocab_resolve splits every query on the C locale's whitespace and looks
// each token up (unknown -> 0xFFFFFFFF, which the planner drops exactly as
// make_plan does), the batch cut into contiguous query ranges over the
// threads of a persistent pool (each range resolved once into a per-thread
// buffer, then copied to its place once the offsets are known).
#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "hm_b200.h"
#include "hm_host.h"
#include "worker_pool.hpp"

struct hm_vocab {
    std::vector<char> arena;
    std::vector<uint64_t> off;   // [n + 1] term bytes in the arena
    std::vector<uint64_t> slot;  // (hash32 << 32) | (tid + 1); 0 = empty
    uint64_t mask = 0;
};

namespace {

inline uint64_t hash_bytes(const char* s, size_t n) {
    // 64-bit multiply-xorshift over 8-byte words (the tail zero-padded)
    uint64_t h = 0x9E3779B97F4A7C15ull ^ (n * 0xFF51AFD7ED558CCDull);
    size_t i = 0;
    for (; i + 8 <= n; i += 8) {
        uint64_t w;
        std::memcpy(&w, s + i, 8);
        h = (h ^ w) * 0xC4CEB9FE1A85EC53ull;
        h ^= h >> 29;
    }
    if (i < n) {
        uint64_t w = 0;
        std::memcpy(&w, s + i, n - i);
        h = (h ^ w) * 0xC4CEB9FE1A85EC53ull;
        h ^= h >> 29;
    }
    h *= 0xFF51AFD7ED558CCDull;
    return h ^ (h >> 32);
}

// std::isspace in the "C" locale (what istringstream >> skips)
inline bool is_ws(unsigned char c) { return c == ' ' || (c >= '\t' && c <= '\r'); }

inline uint32_t lookup(const hm_vocab& v, const char* s, size_t n) {
    const uint64_t h = hash_bytes(s, n);
    const uint64_t tag = h >> 32;
    for (uint64_t i = h & v.mask;; i = (i + 1) & v.mask) {
        const uint64_t e = v.slot[i];
        if (e == 0) return 0xFFFFFFFFu;
        if ((e >> 32) != tag) continue;
        const uint32_t t = static_cast<uint32_t>(e) - 1;
        const uint64_t a = v.off[t], b = v.off[t + 1];
        if (b - a == n && std::memcmp(v.arena.data() + a, s, n) == 0) return t;
    }
}

// tokens of text[lo, hi): calls f(ptr, len) for each
template <typename F>
inline void for_tokens(const char* text, uint64_t lo, uint64_t hi, F&& f) {
    uint64_t i = lo;
    for (;;) {
        while (i < hi && is_ws(static_cast<unsigned char>(text[i]))) ++i;
        if (i >= hi) return;
        const uint64_t s = i;
        while (i < hi && !is_ws(static_cast<unsigned char>(text[i]))) ++i;
        f(text + s, static_cast<size_t>(i - s));
    }
}

}  // namespace

extern "C" {

int hm_vocab_create(const char* const* terms, const uint32_t* lens, uint32_t n, hm_vocab** out) {
    return hm_host::guard([&] {
        if (!out || (n && !terms)) throw std::invalid_argument("null argument");
        auto* v = new hm_vocab();
        try {
            v->off.resize(n + 1ull);
            uint64_t tot = 0;
            for (uint32_t t = 0; t < n; ++t) {
                v->off[t] = tot;
                tot += lens ? lens[t] : std::strlen(terms[t]);
            }
            v->off[n] = tot;
            v->arena.resize(std::max<uint64_t>(tot, 1));
            for (uint32_t t = 0; t < n; ++t)
                std::memcpy(v->arena.data() + v->off[t], terms[t], v->off[t + 1] - v->off[t]);
            uint64_t cap = 16;
            while (cap < 2ull * n) cap <<= 1;
            v->slot.assign(cap, 0);
            v->mask = cap - 1;
            for (uint32_t t = 0; t < n; ++t) {
                const char* s = v->arena.data() + v->off[t];
                const size_t len = v->off[t + 1] - v->off[t];
                if (lookup(*v, s, len) != 0xFFFFFFFFu) throw std::invalid_argument("duplicate term in vocabulary");
                const uint64_t h = hash_bytes(s, len);
                uint64_t i = h & v->mask;
                while (v->slot[i]) i = (i + 1) & v->mask;
                v->slot[i] = ((h >> 32) << 32) | (static_cast<uint64_t>(t) + 1);
            }
        } catch (...) {
            delete v;
            throw;
        }
        *out = v;
    });
}

void hm_vocab_destroy(hm_vocab* v) { delete v; }

int hm_vocab_resolve(const hm_vocab* v, uint32_t nq, const char* text, const uint64_t* text_off, uint32_t* q_off,
                     uint32_t* q_tid, uint64_t tid_cap, uint64_t* n_tids, uint32_t n_threads) {
    return hm_host::guard([&] {
        if (!v || !q_off || (nq && (!text || !text_off))) throw std::invalid_argument("null argument");
        unsigned T = std::min(n_threads ? n_threads : hm_host::worker_pool().size(), hm_host::worker_pool().size());
        if (nq < 1024) T = 1;  // a handful of queries: not worth waking the pool
        T = std::min<unsigned>(T, std::max(nq, 1u));
        // pass 1 (parallel): every query range resolved into its own buffer
        std::vector<std::vector<uint32_t>> loc(T);
        std::vector<uint32_t> cnt(nq + 1ull, 0);
        auto resolve = [&](unsigned t) {
            const uint32_t a = static_cast<uint32_t>(static_cast<uint64_t>(nq) * t / T);
            const uint32_t b = static_cast<uint32_t>(static_cast<uint64_t>(nq) * (t + 1) / T);
            std::vector<uint32_t>& o = loc[t];
            o.reserve(static_cast<size_t>(text_off[b] - text_off[a]) / 4 + 16);
            for (uint32_t q = a; q < b; ++q) {
                const size_t before = o.size();
                for_tokens(text, text_off[q], text_off[q + 1],
                           [&](const char* s, size_t n) { o.push_back(lookup(*v, s, n)); });
                cnt[q] = static_cast<uint32_t>(o.size() - before);
            }
        };
        if (T == 1) resolve(0);
        else hm_host::worker_pool().run(T, resolve);
        uint64_t tot = 0;
        for (uint32_t q = 0; q < nq; ++q) {
            q_off[q] = static_cast<uint32_t>(tot);
            tot += cnt[q];
            if (tot > 0xFFFFFFFFull) throw std::out_of_range("more than 2^32 query terms in one batch");
        }
        q_off[nq] = static_cast<uint32_t>(tot);
        if (n_tids) *n_tids = tot;
        if (tot > tid_cap) throw std::out_of_range("q_tid capacity too small (needed count in n_tids)");
        if (tot && !q_tid) throw std::invalid_argument("q_tid is required");
        // pass 2: each buffer copied to its place
        auto place = [&](unsigned t) {
            const uint32_t a = static_cast<uint32_t>(static_cast<uint64_t>(nq) * t / T);
            if (!loc[t].empty()) std::memcpy(q_tid + q_off[a], loc[t].data(), loc[t].size() * sizeof(uint32_t));
        };
        if (T == 1) place(0);
        else hm_host::worker_pool().run(T, place);
    });
}

uint32_t hm_vocab_size(const hm_vocab* v) { return v ? static_cast<uint32_t>(v->off.size() - 1) : 0; }

}  // extern "C"
