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
#include <cstdint>
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
    std::vector<std::thread> th;
    th.reserve((size_t)T);
    for (int t = 0; t < T; ++t) {
        const int64_t b = n * t / T, e = n * (t + 1) / T;
        th.emplace_back([=, &f] { f(b, e, t); });
    }
    for (auto &x : th)
        x.join();
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
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
            for (;;) {
                const int64_t b = next.fetch_add(block);
                if (b >= n)
                    return;
                for (int64_t i = b, e = std::min(n, b + block); i < e; ++i)
                    f(i, t);
            }
        });
    for (auto &x : th)
        x.join();
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
