// A persistent host worker pool (header-only): the C ABI's query-string
// resolution (hm_text.cpp) and the C++ drop-ins' per-batch host work.
// run(T, f) calls f(0 .. T-1) -- f(0) on the caller -- and returns when all
// are done; one run at a time.  Spawning threads per call cost more than the
// work itself (≈1 ms per 10K-query batch).
#pragma once
#include <algorithm>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include <unistd.h>

namespace hm_host {

class Pool {
public:
    explicit Pool(unsigned n) {
        for (unsigned i = 1; i < n; ++i) th_.emplace_back([this, i] { loop(i); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> l(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    Pool(const Pool&) = delete;
    Pool& operator=(const Pool&) = delete;
    unsigned size() const { return static_cast<unsigned>(th_.size()) + 1; }
    void run(unsigned T, const std::function<void(unsigned)>& f) {  // 1 <= T <= size()
        std::lock_guard<std::mutex> one(run_mu_);
        {
            std::lock_guard<std::mutex> l(mu_);
            job_ = &f;
            job_t_ = T;
            pending_ = T - 1;
            ++gen_;
        }
        cv_.notify_all();
        f(0);
        std::unique_lock<std::mutex> l(mu_);
        done_.wait(l, [&] { return pending_ == 0; });
        job_ = nullptr;
    }

private:
    void loop(unsigned id) {
        uint64_t seen = 0;
        std::unique_lock<std::mutex> l(mu_);
        for (;;) {
            cv_.wait(l, [&] { return stop_ || gen_ != seen; });
            if (stop_) return;
            seen = gen_;
            if (id >= job_t_) continue;
            const std::function<void(unsigned)>* f = job_;
            l.unlock();
            (*f)(id);
            l.lock();
            if (--pending_ == 0) done_.notify_all();
        }
    }
    std::vector<std::thread> th_;
    std::mutex mu_, run_mu_;
    std::condition_variable cv_, done_;
    const std::function<void(unsigned)>* job_ = nullptr;
    unsigned job_t_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

// The process's pool, created on first use; a forked child (which inherits
// the object but not its threads) gets a fresh one.  Never destroyed: the idle
// workers end with the process.
inline Pool& worker_pool() {
    static std::mutex mu;
    static Pool* p = nullptr;
    static pid_t owner = 0;
    std::lock_guard<std::mutex> l(mu);
    if (!p || owner != getpid()) {
        p = new Pool(std::max(1u, std::min(std::thread::hardware_concurrency(), 16u)));
        owner = getpid();
    }
    return *p;
}

// f(a, b) over [0, n) cut into the pool's threads (serially below `min_n`)
template <typename F>
inline void parallel_ranges(std::size_t n, std::size_t min_n, F&& f) {
    const unsigned T = n >= min_n ? std::min<std::size_t>(worker_pool().size(), std::max<std::size_t>(n, 1)) : 1u;
    if (T <= 1) {
        f(std::size_t{0}, n);
        return;
    }
    const std::function<void(unsigned)> job = [&](unsigned t) { f(n * t / T, n * (t + 1) / T); };
    worker_pool().run(T, job);
}

}  // namespace hm_host
