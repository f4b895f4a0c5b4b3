// tal_par.hpp -- host thread parallelism for the mesh preprocessing.
//
// Every parallel step here produces the same bits as its serial form: loops
// write disjoint outputs, reductions are exact (integers, min/max), and the
// sort orders keys that are unique (ties broken by index), so the merge order
// of the sorted runs cannot matter.  Threads: std::thread::hardware_concurrency
// (the process affinity), capped by TAL_PREP_THREADS.
#pragma once
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <cstdlib>
#include <sched.h>
#include <thread>
#include <vector>

namespace tal {

inline int prep_threads()
{
    static const int n = [] {
        int t = (int)std::thread::hardware_concurrency();
        cpu_set_t set;
        if (sched_getaffinity(0, sizeof set, &set) == 0)
            t = CPU_COUNT(&set);
        if (const char *e = std::getenv("TAL_PREP_THREADS"))
            t = std::atoi(e);
        return std::max(1, std::min(t, 64));
    }();
    return n;
}

// Persistent worker pool: run(T, f) calls f(t) for t in [0, T), t = 0 on the
// caller, the rest on parked workers (no thread creation per call -- the
// seam's pipelined copies issue dozens of small parallel steps per call).
// Nested or concurrent use (a worker calling run, or two host threads at
// once) degrades to a serial loop in the caller, so it can never deadlock.
class WorkerPool {
  public:
    static WorkerPool &get()
    {
        static WorkerPool pool(prep_threads());
        return pool;
    }
    template <class F>
    void run(int T, F &&f)
    {
        T = std::min(T, n_);
        if (T <= 1 || in_worker()) {
            for (int t = 0; t < T; ++t)
                f(t);
            return;
        }
        std::unique_lock<std::mutex> busy(busy_, std::try_to_lock);
        if (!busy.owns_lock()) {
            for (int t = 0; t < T; ++t)
                f(t);
            return;
        }
        {
            std::lock_guard<std::mutex> lk(m_);
            job_ = [&f](int t) { f(t); };
            want_ = T;
            next_ = 1;
            left_ = T - 1;
            ++gen_;
        }
        cv_.notify_all();
        in_worker() = true;  // a nested run() from f(0) goes serial
        f(0);
        in_worker() = false;
        std::unique_lock<std::mutex> lk(m_);
        done_.wait(lk, [&] { return left_ == 0; });
        job_ = nullptr;
    }
    ~WorkerPool()
    {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto &t : th_)
            t.join();
    }

  private:
    explicit WorkerPool(int n) : n_(std::max(1, n))
    {
        for (int i = 1; i < n_; ++i)
            th_.emplace_back([this] { loop(); });
    }
    static bool &in_worker()
    {
        thread_local bool w = false;
        return w;
    }
    void loop()
    {
        in_worker() = true;
        uint64_t seen = 0;
        for (;;) {
            std::function<void(int)> job;
            int t = -1;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return stop_ || (gen_ != seen && next_ < want_); });
                if (stop_)
                    return;
                t = next_++;
                if (next_ >= want_)
                    seen = gen_;
                job = job_;
            }
            job(t);
            std::lock_guard<std::mutex> lk(m_);
            if (--left_ == 0)
                done_.notify_all();
        }
    }
    int n_;
    std::vector<std::thread> th_;
    std::mutex m_, busy_;
    std::condition_variable cv_, done_;
    std::function<void(int)> job_;
    uint64_t gen_ = 0;
    int want_ = 0, next_ = 0, left_ = 0;
    bool stop_ = false;
};

// f(begin, end, thread) over [0, n) in contiguous blocks, one per thread;
// serial below 'grain' items.
template <class F>
void parallel_for(int64_t n, F f, int64_t grain = 1 << 14)
{
    const int T = (int)std::min<int64_t>(prep_threads(), std::max<int64_t>(1, n / std::max<int64_t>(grain, 1)));
    if (T <= 1) {
        if (n > 0)
            f((int64_t)0, n, 0);
        return;
    }
    WorkerPool::get().run(T, [&](int t) { f(n * t / T, n * (t + 1) / T, t); });
}

// dynamic scheduling over [0, n) for uneven items: f(i, thread)
template <class F>
void parallel_items(int64_t n, F f, int64_t block = 16)
{
    const int T = (int)std::min<int64_t>(prep_threads(), std::max<int64_t>(1, (n + block - 1) / block));
    if (T <= 1) {
        for (int64_t i = 0; i < n; ++i)
            f(i, 0);
        return;
    }
    std::atomic<int64_t> next{0};
    WorkerPool::get().run(T, [&](int t) {
        for (;;) {
            const int64_t b = next.fetch_add(block);
            if (b >= n)
                return;
            for (int64_t i = b, e = std::min(n, b + block); i < e; ++i)
                f(i, t);
        }
    });
}

// sort of unique keys: per-thread std::sort runs, then a parallel multiway
// merge -- thread k owns the key range [split_k, split_k+1) (splitters from
// the run boundaries' samples), gathers its slice of every run and merges
// the slices pairwise.  Keys must be unique under 'less' (results are then
// the serial std::sort's bits whatever the thread count).
template <class T, class Less>
void psort(std::vector<T> &v, Less less)
{
    const int64_t n = (int64_t)v.size();
    const int P = prep_threads();
    if (n < (1 << 16) || P <= 1) {
        std::sort(v.begin(), v.end(), less);
        return;
    }
    std::vector<int64_t> cut((size_t)P + 1);
    for (int i = 0; i <= P; ++i)
        cut[i] = n * i / P;
    parallel_items(P, [&](int64_t i, int) { std::sort(v.begin() + cut[i], v.begin() + cut[i + 1], less); }, 1);
    // splitters: every run's elements at its own P-quantiles, sorted, every P-th
    std::vector<T> sample;
    for (int r = 0; r < P; ++r)
        for (int q = 1; q < P; ++q)
            sample.push_back(v[cut[r] + (cut[r + 1] - cut[r]) * q / P]);
    std::sort(sample.begin(), sample.end(), less);
    std::vector<T> split;
    for (int k = 1; k < P; ++k)
        split.push_back(sample[(size_t)k * (P - 1) - 1]);
    // bound[k][r]: first index of run r with key >= split_k (k = 0: run start, k = P: run end)
    std::vector<std::vector<int64_t>> bound((size_t)P + 1, std::vector<int64_t>((size_t)P));
    for (int r = 0; r < P; ++r) {
        bound[0][r] = cut[r];
        bound[P][r] = cut[r + 1];
        for (int k = 1; k < P; ++k)
            bound[k][r] = std::lower_bound(v.begin() + cut[r], v.begin() + cut[r + 1], split[k - 1], less) -
                          v.begin();
    }
    std::vector<int64_t> obeg((size_t)P + 1, 0);
    for (int k = 0; k < P; ++k) {
        int64_t m = 0;
        for (int r = 0; r < P; ++r)
            m += bound[k + 1][r] - bound[k][r];
        obeg[k + 1] = obeg[k] + m;
    }
    std::vector<T> out;
    out.reserve((size_t)n);
    out.resize((size_t)n);  // (trivial T: the fill below is the only real cost)
    parallel_items(P, [&](int64_t k, int) {
        // copy the slices, then merge adjacent sorted segments pairwise
        std::vector<int64_t> seg{obeg[k]};
        int64_t at = obeg[k];
        for (int r = 0; r < P; ++r) {
            at = std::copy(v.begin() + bound[k][r], v.begin() + bound[k + 1][r], out.begin() + at) - out.begin();
            seg.push_back(at);
        }
        while (seg.size() > 2) {
            std::vector<int64_t> nxt{seg[0]};
            for (size_t i = 0; i + 2 < seg.size(); i += 2) {
                std::inplace_merge(out.begin() + seg[i], out.begin() + seg[i + 1], out.begin() + seg[i + 2], less);
                nxt.push_back(seg[i + 2]);
            }
            if (seg.size() % 2 == 0)
                nxt.push_back(seg.back());
            seg.swap(nxt);
        }
    }, 1);
    v.swap(out);
}

}  // namespace tal
