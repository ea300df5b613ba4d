// Shared pieces of the C++ drop-ins (csrc/dropin/*.cpp): C-ABI status ->
// the reference's exception types, content fingerprints of the
// reference's index objects, and the LRU cache of their device copies.
//
// A device copy is keyed by the object's address and a fingerprint of its
// arrays (addresses, sizes, a strided sample of the contents), so an object
// destroyed and rebuilt at the same address -- even into recycled buffers of
// the same sizes -- is uploaded again instead of served stale.  The cache
// holds at most `cap` copies; a copy evicted while a batch still uses it
// lives until that batch drops its shared_ptr.
#pragma once
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <list>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "hm_b200.h"

namespace hm_dropin {

inline void throw_on(int rc) {
    if (rc == HM_OK) return;
    const std::string msg = hm_last_error();
    if (rc == HM_ERR_INVALID) throw std::invalid_argument(msg);
    if (rc == HM_ERR_RANGE) throw std::out_of_range(msg);
    throw std::runtime_error(msg);
}

inline uint64_t mix(uint64_t h, uint64_t v) {
    h ^= v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
    return h * 0xFF51AFD7ED558CCDull;
}

// address, size and ~n evenly spaced elements (bit patterns) of an array
template <typename T>
uint64_t sample(uint64_t h, const std::vector<T>& v, std::size_t n = 1024) {
    h = mix(h, reinterpret_cast<uintptr_t>(v.data()));
    h = mix(h, v.size());
    if (v.empty()) return h;
    const std::size_t step = std::max<std::size_t>(1, v.size() / n);
    auto bits = [](const T& x) {
        uint64_t b = 0;
        std::memcpy(&b, &x, std::min(sizeof(T), sizeof b));
        return b;
    };
    for (std::size_t i = 0; i < v.size(); i += step) h = mix(h, bits(v[i]));
    return mix(h, bits(v.back()));
}

template <typename Entry>
class LruCache {
public:
    using Ptr = std::shared_ptr<Entry>;
    explicit LruCache(std::size_t cap) : cap_(cap) {}
    // the copy of `key` whose fingerprint is `fp`; build(Entry&) makes a new one
    template <typename Build>
    Ptr get(const void* key, uint64_t fp, Build&& build) {
        std::lock_guard<std::mutex> lk(mu_);
        for (auto it = lru_.begin(); it != lru_.end(); ++it) {
            if ((*it)->key != key) continue;
            if ((*it)->fp == fp) {
                lru_.splice(lru_.begin(), lru_, it);
                return lru_.front();
            }
            lru_.erase(it);  // same address, other content
            break;
        }
        auto e = std::make_shared<Entry>();
        e->key = key;
        e->fp = fp;
        build(*e);
        lru_.push_front(e);
        while (lru_.size() > cap_) lru_.pop_back();
        return e;
    }
    std::size_t size() {
        std::lock_guard<std::mutex> lk(mu_);
        return lru_.size();
    }
    void clear() {
        std::lock_guard<std::mutex> lk(mu_);
        lru_.clear();
    }

private:
    std::mutex mu_;
    std::list<Ptr> lru_;
    std::size_t cap_;
};

}  // namespace hm_dropin
