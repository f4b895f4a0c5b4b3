// tal_prep.cpp -- native mesh preprocessing (see tal_prep.hpp).
#include "tal_prep.hpp"

#include <algorithm>
#include <array>
#include <atomic>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <numeric>
#include <memory>
#include <chrono>
#include <cstdio>

#include "tal_par.hpp"

namespace tal {

void box_mesh(int64_t nx, int64_t ny, int64_t nz, double ex, double ey, double ez,
              double *coords, int64_t *conn)
{
    // nodes x-fastest; coordinate i*(ext/n), last plane exactly ext
    // (np.linspace semantics, mesh.py:159-162)
    const int64_t sy = nx + 1, sz = (nx + 1) * (ny + 1);
    const double hx = ex / (double)nx, hy = ey / (double)ny, hz = ez / (double)nz;
    for (int64_t k = 0; k <= nz; ++k) {
        const double zc = (k == nz) ? ez : (double)k * hz;
        for (int64_t j = 0; j <= ny; ++j) {
            const double yc = (j == ny) ? ey : (double)j * hy;
            double *row = coords + 3 * (j * sy + k * sz);
            for (int64_t i = 0; i <= nx; ++i) {
                row[3 * i + 0] = (i == nx) ? ex : (double)i * hx;
                row[3 * i + 1] = yc;
                row[3 * i + 2] = zc;
            }
        }
    }
    // six tets per cell: monotone lattice paths corner -> opposite corner along
    // the axis orders (x,y,z),(x,z,y),(y,x,z),(y,z,x),(z,x,y),(z,y,x); paths of
    // odd permutations store their last two nodes swapped to stay positive
    const int64_t stride[3] = {1, sy, sz};
    static const int order[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    static const bool swap_last[6] = {false, true, true, false, false, true};
    int64_t e = 0;
    for (int64_t k = 0; k < nz; ++k)
        for (int64_t j = 0; j < ny; ++j)
            for (int64_t i = 0; i < nx; ++i) {
                const int64_t base = i + j * sy + k * sz;
                for (int t = 0; t < 6; ++t, ++e) {
                    const int64_t v1 = base + stride[order[t][0]];
                    const int64_t v2 = v1 + stride[order[t][1]];
                    const int64_t v3 = v2 + stride[order[t][2]];
                    int64_t *q = conn + 4 * e;
                    q[0] = base;
                    q[1] = v1;
                    q[2] = swap_last[t] ? v3 : v2;
                    q[3] = swap_last[t] ? v2 : v3;
                }
            }
}

void signed_volumes(const double *coords, const int64_t *conn, int64_t n_elems, double *vols)
{
    parallel_for(n_elems, [&](int64_t e0, int64_t e1, int) {
    for (int64_t e = e0; e < e1; ++e) {
        const double *p0 = coords + 3 * conn[4 * e];
        double d[3][3];
        for (int b = 0; b < 3; ++b) {
            const double *pb = coords + 3 * conn[4 * e + b + 1];
            for (int c = 0; c < 3; ++c)
                d[b][c] = pb[c] - p0[c];
        }
        const double det = d[0][0] * (d[1][1] * d[2][2] - d[1][2] * d[2][1]) +
                           d[0][1] * (d[1][2] * d[2][0] - d[1][0] * d[2][2]) +
                           d[0][2] * (d[1][0] * d[2][1] - d[1][1] * d[2][0]);
        vols[e] = det / 6.0;
    }
    });
}

int64_t color_elements(const int64_t *conn, int64_t n_nodes, int64_t n_elems, int64_t *colors)
{
    constexpr int W = 4;  // 4 x 64 = 256 colours
    std::vector<uint64_t> used((size_t)std::max<int64_t>(n_nodes, 1) * W, 0);
    int64_t ncol = 0;
    for (int64_t e = 0; e < n_elems; ++e) {
        const int64_t *q = conn + 4 * e;
        int color = -1;
        for (int w = 0; w < W && color < 0; ++w) {
            const uint64_t m = used[q[0] * W + w] | used[q[1] * W + w] | used[q[2] * W + w] |
                               used[q[3] * W + w];
            if (m != ~0ull)
                color = w * 64 + __builtin_ctzll(~m);
        }
        if (color < 0)
            return -1;
        colors[e] = color;
        ncol = std::max<int64_t>(ncol, color + 1);
        const uint64_t bit = 1ull << (color & 63);
        for (int a = 0; a < 4; ++a)
            used[q[a] * W + (color >> 6)] |= bit;
    }
    return ncol;
}

bool check_coloring(const int64_t *conn, const int64_t *colors, int64_t n_nodes, int64_t n_elems)
{
    // no (node, colour) pair may occur twice (mesh.py:260-267)
    std::vector<std::pair<int64_t, int64_t>> pairs;
    pairs.reserve((size_t)n_elems * 4);
    for (int64_t e = 0; e < n_elems; ++e)
        for (int a = 0; a < 4; ++a)
            pairs.emplace_back(conn[4 * e + a], colors[e]);
    std::sort(pairs.begin(), pairs.end());
    (void)n_nodes;
    return std::adjacent_find(pairs.begin(), pairs.end()) == pairs.end();
}

namespace {

// node -> element incidence (CSR), each list in ascending element id.
// Parallel without atomics: thread t counts its contiguous element block into
// its own count row, the rows become per-(thread, node) write cursors
// (ascending thread order inside each node's list), then every thread fills
// its block -- the serial lists exactly.  Threads are limited so the T x N
// cursor table stays under ~2 GB.
template <class Idx>
void node_elements(const Idx *conn, int64_t n_nodes, int64_t n_elems, std::vector<int64_t> &off,
                   std::vector<int32_t> &adj)
{
    off.assign((size_t)n_nodes + 1, 0);
    adj.resize((size_t)(4 * n_elems));
    int T = prep_threads();
    while (T > 1 && (int64_t)T * n_nodes * 8 > ((int64_t)2 << 30))
        --T;
    if (T <= 1 || n_elems < (1 << 16)) {
        for (int64_t i = 0; i < 4 * n_elems; ++i)
            off[conn[i] + 1]++;
        for (int64_t v = 0; v < n_nodes; ++v)
            off[v + 1] += off[v];
        std::vector<int64_t> pos(off.begin(), off.end() - 1);
        for (int64_t e = 0; e < n_elems; ++e)
            for (int a = 0; a < 4; ++a)
                adj[pos[conn[4 * e + a]]++] = (int32_t)e;
        return;
    }
    std::vector<std::unique_ptr<int64_t[]>> cur((size_t)T);
    std::vector<std::thread> th;
    auto run = [&](auto f) {
        th.clear();
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] { f(t); });
        for (auto &x : th)
            x.join();
    };
    auto eb = [&](int t) { return n_elems * t / T; };
    run([&](int t) {
        cur[t].reset(new int64_t[(size_t)n_nodes]());
        int64_t *c = cur[t].get();
        for (int64_t i = 4 * eb(t); i < 4 * eb(t + 1); ++i)
            c[conn[i]]++;
    });
    // node totals, prefix sum, then per-(thread, node) cursors
    run([&](int t) {
        for (int64_t v = n_nodes * t / T; v < n_nodes * (t + 1) / T; ++v) {
            int64_t sum = 0;
            for (int r = 0; r < T; ++r)
                sum += cur[r][v];
            off[v + 1] = sum;
        }
    });
    for (int64_t v = 0; v < n_nodes; ++v)
        off[v + 1] += off[v];
    run([&](int t) {
        for (int64_t v = n_nodes * t / T; v < n_nodes * (t + 1) / T; ++v) {
            int64_t at = off[v];
            for (int r = 0; r < T; ++r) {
                const int64_t c = cur[r][v];
                cur[r][v] = at;
                at += c;
            }
        }
    });
    run([&](int t) {
        int64_t *c = cur[t].get();
        for (int64_t e = eb(t); e < eb(t + 1); ++e)
            for (int a = 0; a < 4; ++a)
                adj[c[conn[4 * e + a]]++] = (int32_t)e;
    });
}

// Node-node adjacency for Cuthill-McKee: the neighbours of v (the other
// nodes of its incident elements), each list sorted by (valence, id) with
// valence = incident element count.  Built in parallel over nodes.
void cm_neighbours(const int64_t *conn, int64_t n_nodes, const std::vector<int64_t> &off,
                   const std::vector<int32_t> &adj, std::vector<int64_t> &noff, std::vector<int32_t> &nbr)
{
    const int T = prep_threads();
    std::vector<std::vector<int32_t>> part((size_t)T);
    std::vector<int64_t> cnt((size_t)n_nodes + 1, 0);
    std::vector<int64_t> tb((size_t)T + 1, 0);
    parallel_for(n_nodes, [&](int64_t v0, int64_t v1, int t) {
        auto &out = part[(size_t)t];
        std::vector<int32_t> nb;
        std::vector<int32_t> seen((size_t)n_nodes, -1);  // dedup stamp: last v that saw w
        for (int64_t v = v0; v < v1; ++v) {
            nb.clear();
            seen[v] = (int32_t)v;
            for (int64_t p = off[v]; p < off[v + 1]; ++p) {
                const int64_t e = adj[p];
                for (int a = 0; a < 4; ++a) {
                    const int64_t w = conn[4 * e + a];
                    if (seen[w] != (int32_t)v) {
                        seen[w] = (int32_t)v;
                        nb.push_back((int32_t)w);
                    }
                }
            }
            std::sort(nb.begin(), nb.end(), [&](int32_t a, int32_t b) {
                const int64_t da = off[a + 1] - off[a], db = off[b + 1] - off[b];
                return da != db ? da < db : a < b;
            });
            cnt[v + 1] = (int64_t)nb.size();
            out.insert(out.end(), nb.begin(), nb.end());
        }
    }, 1 << 12);
    noff.assign((size_t)n_nodes + 1, 0);
    for (int64_t v = 0; v < n_nodes; ++v)
        noff[v + 1] = noff[v] + cnt[v + 1];
    nbr.resize((size_t)noff[n_nodes]);
    // the blocks of parallel_for are contiguous and in thread order
    int64_t at = 0;
    for (auto &pv : part) {
        std::copy(pv.begin(), pv.end(), nbr.begin() + at);
        at += (int64_t)pv.size();
    }
}

// one BFS from 'start' over unvisited nodes; each node's unvisited
// neighbours are appended in order of increasing valence (Cuthill-McKee):
// the presorted list filtered by the mark is exactly that order.  Returns the
// visit order; 'mark' is set.
void cm_bfs(int64_t start, const std::vector<int64_t> &noff, const std::vector<int32_t> &nbr,
            std::vector<uint8_t> &mark, uint8_t tag, std::vector<int32_t> &order, int64_t *last_level_begin)
{
    order.clear();
    order.push_back((int32_t)start);
    mark[start] = tag;
    size_t head = 0, level_end = 1;
    *last_level_begin = 0;
    while (head < order.size()) {
        if (head == level_end) {
            *last_level_begin = (int64_t)head;
            level_end = order.size();
        }
        if (head + 8 < order.size()) {  // the queue is known ahead: hide the list-start miss
            const int32_t f = order[head + 8];
            __builtin_prefetch(&noff[f]);
            if (head + 4 < order.size())
                __builtin_prefetch(&nbr[noff[order[head + 4]]]);
        }
        const int32_t v = order[head++];
        for (int64_t p = noff[v]; p < noff[v + 1]; ++p) {
            const int32_t w = nbr[p];
            if (mark[w] != tag) {
                mark[w] = tag;
                order.push_back(w);
            }
        }
    }
}

uint64_t spread3(uint64_t v)
{
    v &= 0x1fffff;
    v = (v | v << 32) & 0x1f00000000ffffull;
    v = (v | v << 16) & 0x1f0000ff0000ffull;
    v = (v | v << 8) & 0x100f00f00f00f00full;
    v = (v | v << 4) & 0x10c30c30c30c30c3ull;
    v = (v | v << 2) & 0x1249249249249249ull;
    return v;
}

// Morton order of points.  With a grid (pitch cell[3] > 0 per axis, anchored
// at origin[3]) the primary key is the Morton code of the point's grid cell --
// on an element-size grid, points of one cell stay together and aligned code
// blocks are compact blocks of cells whatever the extents -- and the
// bounding-box code breaks ties; without one, the bounding-box code only.
inline bool p_ok(double lo, double origin) { return lo >= origin; }

struct Lap {
    const char *what;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    static bool on() { static const bool b = std::getenv("TAL_PREP_TIMES") != nullptr; return b; }
    void operator()(const char *sub) {
        auto t = std::chrono::steady_clock::now();
        if (on())
            std::fprintf(stderr, "[tal prep]   %s/%s %.3f s\n", what, sub, std::chrono::duration<double>(t - t0).count());
        t0 = t;
    }
};

template <class GetPoint>
void morton_order(int64_t n, GetPoint pt, std::vector<int32_t> &perm, const double *cell = nullptr,
                  const double *origin = nullptr)
{
    Lap lap{"morton"};
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    {
        const int T = prep_threads();
        std::vector<std::array<double, 6>> box((size_t)T);
        for (auto &b : box)
            b = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY};
        parallel_for(n, [&](int64_t i0, int64_t i1, int t) {
            auto &b = box[(size_t)t];
            for (int64_t i = i0; i < i1; ++i) {
                double p[3];
                pt(i, p);
                for (int c = 0; c < 3; ++c) {
                    b[c] = std::min(b[c], p[c]);
                    b[3 + c] = std::max(b[3 + c], p[c]);
                }
            }
        });
        for (auto &b : box)  // min / max: exact in any order
            for (int c = 0; c < 3; ++c) {
                lo[c] = std::min(lo[c], b[c]);
                hi[c] = std::max(hi[c], b[3 + c]);
            }
    }
    double span = 0.0;
    for (int c = 0; c < 3; ++c)
        span = std::max(span, hi[c] - lo[c]);
    const double scale = span > 0.0 ? (double)((1u << 21) - 1) / span : 0.0;
    bool grid = cell && origin;
    for (int c = 0; grid && c < 3; ++c)
        grid = cell[c] > 0.0 && (hi[c] - origin[c]) / cell[c] < (double)(1u << 21) && p_ok(lo[c], origin[c]);
    struct Key {
        uint64_t coarse, fine;
        int32_t i;
        bool operator<(const Key &o) const
        {
            return coarse != o.coarse ? coarse < o.coarse : fine != o.fine ? fine < o.fine : i < o.i;
        }
    };
    std::vector<Key> key((size_t)n);
    parallel_for(n, [&](int64_t i0, int64_t i1, int) {
        for (int64_t i = i0; i < i1; ++i) {
            double p[3];
            pt(i, p);
            uint64_t fine = 0, coarse = 0;
            for (int c = 0; c < 3; ++c) {
                fine |= spread3((uint64_t)((p[c] - lo[c]) * scale)) << c;
                if (grid)
                    coarse |= spread3((uint64_t)((p[c] - origin[c]) / cell[c])) << c;
            }
            key[i] = {coarse, fine, (int32_t)i};
        }
    });
    lap("bbox+keys");
    psort(key, [](const Key &a, const Key &b) { return a < b; });  // keys unique (index)
    lap("sort");
    perm.resize((size_t)n);
    parallel_for(n, [&](int64_t i0, int64_t i1, int) {
        for (int64_t i = i0; i < i1; ++i)
            perm[i] = key[i].i;
    });
}

}  // namespace

void renumber_rcm(const int64_t *conn, int64_t n_nodes, int64_t n_elems, std::vector<int32_t> &perm)
{
    Lap lap{"rcm"};
    std::vector<int64_t> off;
    std::vector<int32_t> adj;
    node_elements(conn, n_nodes, n_elems, off, adj);
    lap("node_elements");
    std::vector<int64_t> noff;
    std::vector<int32_t> nbr;
    cm_neighbours(conn, n_nodes, off, adj, noff, nbr);
    lap("neighbours");
    // byte marks (a BFS is latency bound on them: 1 B per node keeps them in
    // cache); tags cycle through 1..255 with a clear on wrap-around
    std::vector<uint8_t> mark((size_t)n_nodes, 0), done((size_t)n_nodes, 0);
    std::vector<int32_t> order, result;
    result.reserve((size_t)n_nodes);
    int tag = 0;
    auto next_tag = [&]() -> uint8_t {
        if (++tag == 256) {
            std::fill(mark.begin(), mark.end(), 0);
            tag = 1;
        }
        return (uint8_t)tag;
    };
    // components in order of their smallest-valence seed
    // (= stable sort by valence, as a counting sort)
    std::vector<int32_t> seeds((size_t)n_nodes);
    {
        int64_t vmax = 0;
        for (int64_t v = 0; v < n_nodes; ++v)
            vmax = std::max(vmax, off[v + 1] - off[v]);
        std::vector<int64_t> at((size_t)vmax + 2, 0);
        for (int64_t v = 0; v < n_nodes; ++v)
            at[off[v + 1] - off[v] + 1]++;
        for (int64_t k = 0; k <= vmax; ++k)
            at[k + 1] += at[k];
        for (int64_t v = 0; v < n_nodes; ++v)
            seeds[at[off[v + 1] - off[v]]++] = (int32_t)v;
    }
    for (int32_t s : seeds) {
        if (done[s])
            continue;
        // pseudo-peripheral start: two sweeps (George-Liu style)
        int64_t start = s, llb = 0;
        for (int sweep = 0; sweep < 2; ++sweep) {
            cm_bfs(start, noff, nbr, mark, next_tag(), order, &llb);
            int64_t best = order[llb];
            for (size_t i = (size_t)llb; i < order.size(); ++i) {
                const int32_t v = order[i];
                if (off[v + 1] - off[v] < off[best + 1] - off[best])
                    best = v;
            }
            start = best;
        }
        cm_bfs(start, noff, nbr, mark, next_tag(), order, &llb);
        for (int32_t v : order)
            done[v] = 1;
        result.insert(result.end(), order.begin(), order.end());
    }
    std::reverse(result.begin(), result.end());
    perm.swap(result);
    lap("bfs");
}

void renumber_sfc(const double *coords, int64_t n_nodes, std::vector<int32_t> &perm)
{
    morton_order(
        n_nodes,
        [&](int64_t i, double p[3]) {
            for (int c = 0; c < 3; ++c)
                p[c] = coords[3 * i + c];
        },
        perm);
}

void element_order(int method, const int32_t *conn4, const double *coords_int, int64_t n_nodes,
                   int64_t n_elems, std::vector<int32_t> &eperm)
{
    eperm.resize((size_t)n_elems);
    std::iota(eperm.begin(), eperm.end(), 0);
    if (method == 1) {  // by smallest node id
        std::vector<std::pair<int32_t, int32_t>> key((size_t)n_elems);
        parallel_for(n_elems, [&](int64_t e0, int64_t e1, int) {
            for (int64_t e = e0; e < e1; ++e) {
                const int32_t *q = conn4 + 4 * e;
                key[e] = {std::min(std::min(q[0], q[1]), std::min(q[2], q[3])), (int32_t)e};
            }
        });
        psort(key, [](const std::pair<int32_t, int32_t> &a, const std::pair<int32_t, int32_t> &b) {
            return a < b;
        });
        for (int64_t e = 0; e < n_elems; ++e)
            eperm[e] = key[e].second;
    } else if (method == 2) {  // Morton order of centroids on an element-size grid
        // grid pitch per axis: the mean extent of an element's bounding box
        // (a Kuhn tet spans exactly its cell, so the key is the cell index),
        // anchored at the nodes' bounding-box corner
        double lo[3] = {INFINITY, INFINITY, INFINITY}, cell[3] = {0.0, 0.0, 0.0};
        for (int64_t v = 0; v < n_nodes; ++v)
            for (int c = 0; c < 3; ++c)
                lo[c] = std::min(lo[c], coords_int[3 * v + c]);
        // extents and centroids in one parallel gather; extents summed in
        // element order (the serial bits)
        std::unique_ptr<double[]> ext(new double[(size_t)(3 * n_elems)]);  // no zero fill
        std::unique_ptr<double[]> cen(new double[(size_t)(3 * n_elems)]);
        parallel_for(n_elems, [&](int64_t e0, int64_t e1, int) {
            for (int64_t e = e0; e < e1; ++e) {
                const int32_t *q = conn4 + 4 * e;
                for (int c = 0; c < 3; ++c) {
                    const double x0 = coords_int[3 * q[0] + c], x1 = coords_int[3 * q[1] + c];
                    const double x2 = coords_int[3 * q[2] + c], x3 = coords_int[3 * q[3] + c];
                    ext[3 * e + c] = std::max(std::max(std::max(x0, x1), x2), x3) -
                                     std::min(std::min(std::min(x0, x1), x2), x3);
                    cen[3 * e + c] = 0.25 * (x0 + x1 + x2 + x3);
                }
            }
        });
        for (int64_t e = 0; e < n_elems; ++e)
            for (int c = 0; c < 3; ++c)
                cell[c] += ext[3 * e + c];
        ext.reset();
        for (int c = 0; c < 3; ++c)
            cell[c] = n_elems ? cell[c] / (double)n_elems : 0.0;
        morton_order(
            n_elems,
            [&](int64_t e, double p[3]) {
                for (int c = 0; c < 3; ++c)
                    p[c] = cen[3 * e + c];
            },
            eperm, cell, lo);
    }
}

namespace {

struct Arc {
    std::vector<int32_t> tets, ring;
    bool closed = false;
};

// ring candidates of one edge (p,q) of the current tet: the unassigned tets
// containing p and q (in adj[p] order, at most 64) with their two other
// corners (c,d)
struct Cand {
    int32_t tet, c, d;
    bool used;
};
struct EdgeCands {
    Cand cand[64];
    int n = 0;
};

// one pass over the unassigned tets at each corner i < 3 of tet t fills the
// candidate lists of the edges (v[i], v[j]), j > i -- the same lists, in the
// same order, as scanning adj[v[i]] once per edge
template <class Assigned>
void edge_candidates(int64_t t, const int32_t *conn4, const std::vector<int64_t> &off,
                     const std::vector<int32_t> &adj, const Assigned &assigned, EdgeCands ec[6])
{
    static const int EIDX[3][4] = {{-1, 0, 1, 2}, {-1, -1, 3, 4}, {-1, -1, -1, 5}};
    const int32_t *v = conn4 + 4 * t;
    for (int e = 0; e < 6; ++e)
        ec[e].n = 0;
    for (int i = 0; i < 3; ++i) {
        const int32_t p = v[i];
        for (int64_t k = off[p]; k < off[p + 1]; ++k) {
            const int32_t s = adj[k];
            if (assigned(s))
                continue;
            const int32_t *w = conn4 + 4 * (int64_t)s;
            unsigned m = 0;  // which of v[j], j > i, tet s contains
            for (int j = i + 1; j < 4; ++j)
                m |= (unsigned)((w[0] == v[j]) | (w[1] == v[j]) | (w[2] == v[j]) | (w[3] == v[j])) << j;
            while (m) {
                const int j = __builtin_ctz(m);
                m &= m - 1;
                EdgeCands &E = ec[EIDX[i][j]];
                if (E.n >= 64)
                    continue;
                const int32_t q = v[j];
                int32_t o[2], no = 0;
                for (int a = 0; a < 4; ++a)
                    if (w[a] != q && w[a] != p && no < 2)
                        o[no++] = w[a];
                if (no == 2)
                    E.cand[E.n++] = {s, o[0], o[1], s == (int32_t)t};
            }
        }
    }
}

// ring of unassigned tets around edge (p,q) that contains tet t, from the
// edge's candidate list
void ring_arc(int32_t t, int32_t p, int32_t q, const int32_t *conn4, const EdgeCands &E, Arc &arc)
{
    Cand cand[64];
    const int nc = E.n;
    std::copy(E.cand, E.cand + nc, cand);
    int it = -1;
    for (int i = 0; i < nc; ++i)
        if (cand[i].tet == t)
            it = i;
    arc.tets.assign(1, t);
    arc.closed = false;
    if (it < 0) {  // should not happen
        const int32_t *v = conn4 + 4 * (int64_t)t;
        arc.ring.clear();
        for (int a = 0; a < 4; ++a)
            if (v[a] != p && v[a] != q)
                arc.ring.push_back(v[a]);
        return;
    }
    // fixed-size walks (this runs 6x per patch: no heap traffic)
    struct Seq {
        int32_t v[PATCH_MAX_RING + 2];
        int n = 0;
        void push(int32_t x) { v[n++] = x; }
        int32_t back() const { return v[n - 1]; }
    };
    Seq fwd, bwd, tf, tb;
    fwd.push(cand[it].d);
    bwd.push(cand[it].c);
    // at most 6 tets per patch (a Kuhn cell's closed ring; longer rings of
    // unstructured meshes are cut into arcs): the warp that walks a chunk's
    // longest rings sets the chunk's phase-B time, and on a Delaunay mesh the
    // cap measured 34.0 (8) -> 36.0 (6) Gelem/s; TAL_MAX_RING_TETS overrides
    static const int max_tets = [] {
        const char *e = std::getenv("TAL_MAX_RING_TETS");
        const int v = e ? std::atoi(e) : 6;
        return std::max(1, std::min(v, PATCH_MAX_RING - 1));
    }();
    auto walk = [&](Seq &seq, Seq &ts, const Seq &other, int budget) {
        while (ts.n < budget) {
            const int32_t cur = seq.back();
            int found = -1;
            for (int i = 0; i < nc; ++i)
                if (!cand[i].used && (cand[i].c == cur || cand[i].d == cur)) {
                    found = i;
                    break;
                }
            if (found < 0)
                return false;
            cand[found].used = true;
            const int32_t nxt = cand[found].c == cur ? cand[found].d : cand[found].c;
            ts.push(cand[found].tet);
            if (nxt == other.v[0])
                return true;  // closed the ring
            seq.push(nxt);
        }
        return false;
    };
    const bool closed = walk(fwd, tf, bwd, max_tets - 1);
    if (!closed)
        walk(bwd, tb, fwd, max_tets - 1 - tf.n);
    arc.ring.clear();
    for (int i = bwd.n - 1; i >= 0; --i)
        arc.ring.push_back(bwd.v[i]);
    for (int i = 0; i < fwd.n; ++i)
        arc.ring.push_back(fwd.v[i]);
    arc.tets.clear();
    for (int i = tb.n - 1; i >= 0; --i)
        arc.tets.push_back(tb.v[i]);
    arc.tets.push_back(t);
    for (int i = 0; i < tf.n; ++i)
        arc.tets.push_back(tf.v[i]);
    arc.closed = closed;
}

}  // namespace

void build_patches(const int32_t *conn4, int64_t n_nodes, int64_t n_elems, int mode, Patches &out)
{
    out.off.assign(1, 0);
    out.nodes.clear();
    out.closed.clear();
    if (mode == 0) {
        out.off.reserve((size_t)n_elems + 1);
        out.nodes.reserve((size_t)n_elems * 4);
        for (int64_t e = 0; e < n_elems; ++e) {
            for (int a = 0; a < 4; ++a)
                out.nodes.push_back(conn4[4 * e + a]);
            out.off.push_back((int32_t)out.nodes.size());
            out.closed.push_back(0);
        }
        return;
    }
    // node -> tets
    Lap lap{"patches"};
    std::vector<int64_t> off;
    std::vector<int32_t> adj;
    node_elements(conn4, n_nodes, n_elems, off, adj);
    lap("adjacency");
    // The greedy is sequential in tet order; it runs on contiguous blocks of
    // the order in parallel, speculatively.  When the serial walk reaches a
    // block's first tet, every earlier tet is assigned, so a block's outcome
    // depends only on which of ITS OWN or later tets earlier blocks' patches
    // took ("spill"): each block assumes none, records its own spills, and a
    // serial fix-up re-runs every block whose actual inflow was not empty
    // with that inflow -- the result is exactly the serial greedy's.
    std::vector<uint8_t> shared((size_t)n_elems, 0);  // block k owns [b_k, e_k)
    struct Block {
        int64_t b = 0, e = 0;
        std::vector<int32_t> ends, nodes, spill;  // patch end offsets (block-relative nodes)
        std::vector<uint8_t> closed;
    };
    auto greedy = [&](Block &B, const std::vector<int32_t> &inflow) {
        const int64_t b = B.b, e = B.e;
        std::fill(shared.begin() + b, shared.begin() + e, 0);
        std::vector<int32_t> ext;  // assigned tets >= e, sorted
        for (int32_t x : inflow) {
            if (x < e)
                shared[x] = 1;
            else
                ext.push_back(x);
        }
        std::sort(ext.begin(), ext.end());
        B.ends.clear(), B.nodes.clear(), B.spill.clear(), B.closed.clear();
        auto assigned = [&](int64_t x) {
            return x < b || (x < e ? shared[x] != 0 : std::binary_search(ext.begin(), ext.end(), (int32_t)x));
        };
        static const int EDGES[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
        Arc best, cur;
        EdgeCands ec[6];
        int32_t best_p = 0, best_q = 0;
        for (int64_t t = b; t < e; ++t) {
            if (assigned(t))
                continue;
            const int32_t *v = conn4 + 4 * t;
            size_t best_n = 0;
            int64_t best_span = 0;
            edge_candidates(t, conn4, off, adj, assigned, ec);
            for (int k = 0; k < 6; ++k) {
                const auto &ed = EDGES[k];
                const int32_t p = v[ed[0]], q = v[ed[1]];
                ring_arc((int32_t)t, p, q, conn4, ec[k], cur);
                int64_t lo = cur.tets[0], hi = cur.tets[0];
                for (int32_t x : cur.tets) {
                    lo = std::min<int64_t>(lo, x);
                    hi = std::max<int64_t>(hi, x);
                }
                const int64_t span = hi - lo;
                if (cur.tets.size() > best_n || (cur.tets.size() == best_n && span < best_span)) {
                    best_n = cur.tets.size();
                    best_span = span;
                    std::swap(best, cur);
                    best_p = p;
                    best_q = q;
                }
            }
            for (int32_t x : best.tets) {
                if (x < e) {
                    shared[x] = 1;
                } else {
                    ext.insert(std::lower_bound(ext.begin(), ext.end(), x), x);
                    B.spill.push_back(x);
                }
            }
            B.nodes.push_back(best_p);
            B.nodes.push_back(best_q);
            for (int32_t r : best.ring)
                B.nodes.push_back(r);
            B.ends.push_back((int32_t)B.nodes.size());
            B.closed.push_back(best.closed ? 1 : 0);
        }
    };
    const int K = (int)std::max<int64_t>(1, std::min<int64_t>(prep_threads(), n_elems / 4096));
    std::vector<Block> blocks((size_t)K);
    for (int k = 0; k < K; ++k)
        blocks[k].b = n_elems * k / K, blocks[k].e = n_elems * (k + 1) / K;
    const std::vector<int32_t> none;
    parallel_items(K, [&](int64_t k, int) { greedy(blocks[k], none); }, 1);
    lap("greedy (speculative)");
    std::vector<int32_t> carry;  // tets >= b_k taken by the final patches of blocks < k
    int reruns = 0;
    for (int k = 0; k < K; ++k) {
        std::vector<int32_t> inflow;
        for (int32_t x : carry)
            if (x >= blocks[k].b)
                inflow.push_back(x);
        if (!inflow.empty()) {
            greedy(blocks[k], inflow);
            ++reruns;
        }
        inflow.insert(inflow.end(), blocks[k].spill.begin(), blocks[k].spill.end());
        carry.swap(inflow);
    }
    if (Lap::on())
        std::fprintf(stderr, "[tal prep]   patches: %d blocks, %d re-run\n", K, reruns);
    size_t nn = 0, np = 0;
    for (auto &B : blocks)
        nn += B.nodes.size(), np += B.ends.size();
    out.nodes.reserve(nn);
    out.off.reserve(np + 1);
    out.closed.reserve(np);
    for (auto &B : blocks) {
        const int32_t base = (int32_t)out.nodes.size();
        out.nodes.insert(out.nodes.end(), B.nodes.begin(), B.nodes.end());
        for (int32_t x : B.ends)
            out.off.push_back(base + x);
        out.closed.insert(out.closed.end(), B.closed.begin(), B.closed.end());
    }
    lap("fix-up + concat");
}

bool orient_patches(Patches &P, const double *xyz)
{
    auto det = [&](int32_t a, int32_t b, int32_t c, int32_t d) {
        double e[3][3];
        for (int k = 0; k < 3; ++k) {
            e[0][k] = xyz[3 * (int64_t)b + k] - xyz[3 * (int64_t)a + k];
            e[1][k] = xyz[3 * (int64_t)c + k] - xyz[3 * (int64_t)a + k];
            e[2][k] = xyz[3 * (int64_t)d + k] - xyz[3 * (int64_t)a + k];
        }
        return e[0][0] * (e[1][1] * e[2][2] - e[1][2] * e[2][1]) +
               e[0][1] * (e[1][2] * e[2][0] - e[1][0] * e[2][2]) +
               e[0][2] * (e[1][0] * e[2][1] - e[1][1] * e[2][0]);
    };
    std::atomic<bool> ok{true};
    parallel_for(P.n_patches(), [&](int64_t g0, int64_t g1, int) {
        for (int64_t g = g0; g < g1; ++g) {
            int32_t *v = P.nodes.data() + P.off[g];
            const int m = P.off[g + 1] - P.off[g] - 2;
            const int k = P.closed[g] ? m : m - 1;
            int pos = 0, neg = 0;
            for (int t = 0; t < k; ++t) {
                const double d = det(v[0], v[1], v[2 + t], v[2 + (t + 1 == m ? 0 : t + 1)]);
                pos += d > 0.0;
                neg += d < 0.0;
            }
            if (neg == k)
                std::swap(v[0], v[1]);
            else if (pos != k)
                ok = false;
        }
    }, 1 << 12);
    return ok;
}

// ---------------------------------------------------------------------------
// Bank-aware placement of a chunk's node records in shared memory.
//
// Phase B loads a 48-B record per ring node with three LDS.128; a quarter-warp
// (8 lanes) is served conflict-free only if its 8 records sit in distinct
// 16-B bank groups, i.e. (3 j + s) mod 8 distinct for record slot j -- which
// holds iff the slots are distinct mod 8.  Every load instruction of the ring
// walk (a, b, r_0, then r_{t+1} at tet t) defines, per quarter-warp, a group
// of nodes; the placement colours nodes with the 8 residues (capacity
// ceil((nn - c) / 8) each) minimising the sum over groups of colliding pairs:
// greedy by group count, then pairwise-swap descent.  Returns the slot order.
// ---------------------------------------------------------------------------
namespace {
struct BankStats {
    int64_t groups = 0, wave_before = 0, wave_after = 0;
};
BankStats g_bank;

int bank_place_mode()
{
    static int mode = [] {
        const char *e = std::getenv("TAL_BANK_PLACE");
        return e ? std::atoi(e) : 1;
    }();
    return mode;
}

void bank_place(const Patches &P, int64_t p0, int64_t p1, std::vector<int32_t> &nodes,
                int32_t *idx, BankStats &stats)
{
    const int nn = (int)nodes.size();
    for (int i = 0; i < nn; ++i)
        idx[nodes[i]] = i;
    constexpr int NI = 3 + PATCH_MAX_RING;  // load instructions of one ring walk
    const int64_t npat = p1 - p0;
    const int nq = (int)((npat + 7) / 8);
    const int ng = nq * NI;
    std::vector<std::vector<int32_t>> gm((size_t)ng);
    for (int64_t g = p0; g < p1; ++g) {
        const int q = (int)((g - p0) >> 3);
        const int32_t *v = P.nodes.data() + P.off[g];
        const int m = P.off[g + 1] - P.off[g] - 2;
        const int k = P.closed[g] ? m : m - 1;
        gm[(size_t)q * NI + 0].push_back(idx[v[0]]);
        gm[(size_t)q * NI + 1].push_back(idx[v[1]]);
        gm[(size_t)q * NI + 2].push_back(idx[v[2]]);
        for (int t = 0; t < k; ++t)
            gm[(size_t)q * NI + 3 + t].push_back(idx[v[2 + (t + 1 == m ? 0 : t + 1)]]);
    }
    std::vector<std::vector<int32_t>> ng_of((size_t)nn);  // groups of each node
    for (int G = 0; G < ng; ++G) {
        auto &v = gm[G];
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
        for (int32_t i : v)
            ng_of[i].push_back(G);
    }
    std::vector<int> cls(nn, -1), cap(8), used(8, 0);
    for (int c = 0; c < 8; ++c)
        cap[c] = (nn - c + 7) / 8;
    std::vector<std::array<int, 8>> cnt((size_t)ng);
    for (auto &a : cnt)
        a.fill(0);
    auto waves = [&]() {
        int64_t w = 0;
        for (int G = 0; G < ng; ++G)
            if (!gm[G].empty())
                w += *std::max_element(cnt[G].begin(), cnt[G].end());
        return w;
    };
    // before: ascending node id in slot order
    for (int i = 0; i < nn; ++i)
        for (int G : ng_of[i])
            cnt[G][i & 7]++;
    int64_t groups = 0;
    for (int G = 0; G < ng; ++G)
        groups += !gm[G].empty();
    const int64_t before = waves();
    for (auto &a : cnt)
        a.fill(0);
    std::vector<int> ord(nn);
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(),
                     [&](int x, int y) { return ng_of[x].size() > ng_of[y].size(); });
    for (int i : ord) {
        int best = -1;
        int64_t bc = 0;
        for (int c = 0; c < 8; ++c) {
            if (used[c] >= cap[c])
                continue;
            int64_t cost = 0;
            for (int G : ng_of[i])
                cost += cnt[G][c];
            cost = cost * 1024 + used[c];
            if (best < 0 || cost < bc)
                best = c, bc = cost;
        }
        cls[i] = best;
        used[best]++;
        for (int G : ng_of[i])
            cnt[G][best]++;
    }
    std::vector<std::vector<int32_t>> members(8);
    for (int i = 0; i < nn; ++i)
        members[cls[i]].push_back(i);
    std::vector<int> mark((size_t)ng, -1);
    auto move_cost = [&](int i, int from, int to) {  // colliding-pair change of moving i
        int64_t d = 0;
        for (int G : ng_of[i])
            d += cnt[G][to] - (cnt[G][from] - 1);
        return d;
    };
    for (int pass = 0; pass < 4; ++pass) {
        bool any = false;
        for (int u = 0; u < nn; ++u) {
            const int a = cls[u];
            int64_t best = 0;
            int bv = -1;
            for (int b = 0; b < 8; ++b) {
                if (b == a)
                    continue;
                const int64_t mu = move_cost(u, a, b);
                if (mu >= 0)
                    continue;
                for (int G : ng_of[u])
                    mark[G] = u;
                for (int32_t v : members[b]) {
                    int shared = 0;
                    for (int G : ng_of[v])
                        shared += mark[G] == u;
                    const int64_t d = mu + move_cost(v, b, a) - 2 * shared;
                    if (d < best)
                        best = d, bv = v;
                }
                for (int G : ng_of[u])
                    mark[G] = -1;
            }
            if (bv < 0)
                continue;
            const int b = cls[bv];
            for (int G : ng_of[u])
                cnt[G][a]--, cnt[G][b]++;
            for (int G : ng_of[bv])
                cnt[G][b]--, cnt[G][a]++;
            cls[u] = b, cls[bv] = a;
            auto &ma = members[a], &mb = members[b];
            *std::find(ma.begin(), ma.end(), u) = bv;
            *std::find(mb.begin(), mb.end(), bv) = u;
            any = true;
        }
        if (!any)
            break;
    }
    stats.groups += groups;
    stats.wave_before += before;
    stats.wave_after += waves();
    // slot j = c + 8 r: class c's members in ascending node id
    std::vector<int32_t> out((size_t)nn);
    for (int c = 0; c < 8; ++c) {
        auto &mc = members[c];
        std::sort(mc.begin(), mc.end());
        for (size_t r = 0; r < mc.size(); ++r)
            out[(size_t)c + 8 * r] = nodes[mc[r]];
    }
    nodes.swap(out);
}
}  // namespace

void bank_stats(int64_t *groups, int64_t *before, int64_t *after)
{
    *groups = g_bank.groups, *before = g_bank.wave_before, *after = g_bank.wave_after;
}

// ---------------------------------------------------------------------------
// Bank-aware contribution positions.  Phase B stores each patch node's sum at
// p = lev[s] + rank[node] (three 8-B arrays); a half-warp (16 lanes) of one
// STS.64 is conflict-free iff its positions are distinct mod 16.  Free
// choices that keep the jagged layout valid: which of a node's contributions
// takes which level s, and the rank order among nodes of equal contribution
// count.  Pairwise-swap descent on the colliding pairs per (half-warp, store
// instruction) group over the level choice (rank swaps among equal counts,
// measured: 1.95 -> 1.87 wavefronts per group for 2.5x the host prep time,
// are not done).  'lvl' (in: patch-order levels, out: chosen levels) is
// indexed like the patch-order contribution enumeration of close_chunk.
// ---------------------------------------------------------------------------
namespace {
BankStats g_pos;

#ifndef POS_PASSES
#define POS_PASSES 2
#endif
int pos_place_mode()
{
    static int mode = [] {
        const char *e = std::getenv("TAL_POS_PLACE");
        return e ? std::atoi(e) : 1;
    }();
    return mode;
}

void pos_place(const Patches &P, int64_t p0, int64_t p1, const int32_t *local,
               const std::vector<int32_t> &ncnt, std::vector<int32_t> &order, std::vector<int32_t> &rank,
               const uint16_t *lev, std::vector<int32_t> &lvl, BankStats &stats)
{
    constexpr int NI = PATCH_MAX_RING + 3;  // loop stores, then ring end, a, b
    const int nn = (int)rank.size();
    const int64_t npat = p1 - p0;
    const int ng = (int)((npat + 15) / 16) * NI;
    struct Con {
        int32_t node, g0, g1;  // g1 = -1 or the second group (closed ring's r_0 RMW)
    };
    std::vector<Con> con;
    con.reserve((size_t)npat * (PATCH_MAX_RING + 2));
    for (int64_t g = p0; g < p1; ++g) {
        const int32_t *v = P.nodes.data() + P.off[g];
        const int m = P.off[g + 1] - P.off[g] - 2;
        const bool closed = P.closed[g];
        const int kk = closed ? m : m - 1;
        const int base = (int)((g - p0) >> 4) * NI;
        for (int k = 0; k < m + 2; ++k) {
            Con c{local[v[k]], -1, -1};
            if (k == 0)
                c.g0 = base + PATCH_MAX_RING + 1;
            else if (k == 1)
                c.g0 = base + PATCH_MAX_RING + 2;
            else {
                const int i = k - 2;
                if (i < kk)
                    c.g0 = base + i;
                if ((closed && i == 0) || (!closed && i == m - 1))
                    (c.g0 < 0 ? c.g0 : c.g1) = base + PATCH_MAX_RING;
            }
            con.push_back(c);
        }
    }
    const int nc = (int)con.size();
    std::vector<std::vector<int32_t>> of_node((size_t)nn);  // contributions per node
    for (int c = 0; c < nc; ++c)
        of_node[con[c].node].push_back(c);
    std::vector<std::array<int16_t, 16>> cnt((size_t)ng);
    for (auto &a : cnt)
        a.fill(0);
    auto cls = [&](int c) { return (lev[lvl[c]] + rank[con[c].node]) & 15; };
    auto add = [&](int c, int d) {  // returns the pair-count change of adding (d=+1) / removing (d=-1)
        const int k = cls(c);
        int64_t delta = 0;
        for (int G : {con[c].g0, con[c].g1})
            if (G >= 0) {
                if (d > 0)
                    delta += cnt[G][k]++;
                else
                    delta -= --cnt[G][k];
            }
        return delta;
    };
    auto waves = [&]() {
        int64_t w = 0, groups = 0;
        for (int G = 0; G < ng; ++G) {
            int mx = 0, tot = 0;
            for (int x : cnt[G])
                mx = std::max(mx, x), tot += x;
            w += mx;
            groups += tot > 0;
        }
        return std::make_pair(w, groups);
    };
    for (int c = 0; c < nc; ++c)
        add(c, +1);
    const auto before = waves();
    // try a change: remove the affected contributions, mutate, re-add; keep if better
    auto attempt = [&](const std::vector<int32_t> &cs, auto &&mutate, auto &&undo) {
        int64_t d = 0;
        for (int c : cs)
            d += add(c, -1);
        mutate();
        for (int c : cs)
            d += add(c, +1);
        if (d < 0)
            return true;
        for (int c : cs)
            add(c, -1);
        undo();
        for (int c : cs)
            add(c, +1);
        return false;
    };
    std::vector<int32_t> cs;
    for (int pass = 0; pass < POS_PASSES; ++pass) {
        bool any = false;
        // (a) level swaps between two contributions of one node
        for (int j = 0; j < nn; ++j) {
            auto &L = of_node[j];
            for (size_t x = 0; x < L.size(); ++x)
                for (size_t y = x + 1; y < L.size(); ++y) {
                    const int a = L[x], b = L[y];
                    cs = {a, b};
                    any |= attempt(cs, [&] { std::swap(lvl[a], lvl[b]); }, [&] { std::swap(lvl[a], lvl[b]); });
                }
        }
        if (!any)
            break;
    }
    const auto after = waves();
    stats.groups += before.second;
    stats.wave_before += before.first;
    stats.wave_after += after.first;
}
}  // namespace

void pos_stats(int64_t *groups, int64_t *before, int64_t *after)
{
    *groups = g_pos.groups, *before = g_pos.wave_before, *after = g_pos.wave_after;
}

namespace {
// patches of a chunk ordered by ring length (TAL_RING_SORT=0: as built)
int ring_sort_mode()
{
    static int mode = [] {
        const char *e = std::getenv("TAL_RING_SORT");
        return e ? std::atoi(e) : 1;
    }();
    return mode;
}
}  // namespace

bool build_chunks(const Patches &P_in, int64_t n_nodes, int max_patches, int max_nodes, int max_contrib,
                  const uint8_t *external, Chunking &out, std::string &err)
{
    const Patches *pp = &P_in;
    if (max_patches < 1 || max_nodes < PATCH_MAX_RING + 2 || max_contrib < PATCH_MAX_RING + 2 ||
        max_contrib > 65535 || max_nodes > 65535) {
        err = "invalid chunk limits";
        return false;
    }
    const Patches &P0 = P_in;
    out = Chunking();
    out.max_patches = max_patches;
    out.max_nodes = max_nodes;
    out.max_contrib = max_contrib;
    const int64_t np = P0.n_patches();
    out.pids.assign((size_t)np * PATCH_SLOTS, 0);
    out.ppos.assign((size_t)np * PATCH_SLOTS, 0);

    Lap lap{"chunks"};
    // pass 1 (serial, cheap): greedy chunk boundaries in patch order
    struct Span {
        int64_t p0, p1;
        int32_t nn, contrib;
    };
    std::vector<Span> spans;
    {
        std::vector<int32_t> stamp((size_t)n_nodes, -1), cnt((size_t)n_nodes, 0), nodes;
        int32_t chunk = 0;
        int64_t p_begin = 0, contrib = 0;
        auto close = [&](int64_t p_end) {
            spans.push_back({p_begin, p_end, (int32_t)nodes.size(), (int32_t)contrib});
            for (int32_t v : nodes)
                cnt[v] = 0;
            nodes.clear();
            ++chunk;
            p_begin = p_end;
            contrib = 0;
        };
        for (int64_t g = 0; g < np; ++g) {
            const int32_t n = P0.off[g + 1] - P0.off[g];
            if (n - 2 > PATCH_MAX_RING || n < 4) {
                err = "patch ring size out of range";
                return false;
            }
            int fresh = 0;
            bool full_level = false;
            for (int32_t k = P0.off[g]; k < P0.off[g + 1]; ++k) {
                const int32_t v = P0.nodes[k];
                if (stamp[v] != chunk)
                    ++fresh;
                else if (cnt[v] + 1 > CHUNK_LEVELS)
                    full_level = true;
            }
            if (g > p_begin && ((g - p_begin) + 1 > max_patches || (int64_t)nodes.size() + fresh > max_nodes ||
                                contrib + n > max_contrib || full_level))
                close(g);
            for (int32_t k = P0.off[g]; k < P0.off[g + 1]; ++k) {
                const int32_t v = P0.nodes[k];
                if (stamp[v] != chunk) {
                    stamp[v] = chunk;
                    nodes.push_back(v);
                }
                cnt[v]++;
            }
            contrib += n;
        }
        if (np > p_begin)
            close(np);
    }
    lap("pass1");
    const int64_t n_chunks = (int64_t)spans.size();
    // Within every chunk, patches by tet count, descending (stable): thread
    // = patch, so a warp's lanes then walk rings of equal length.  On a Kuhn
    // box every interior ring has 6 tets and this changes little; on an
    // unstructured mesh (rings of 1-8 tets) it keeps the ring loop's SIMT
    // lanes busy instead of idling behind the longest ring of the warp.
    Patches sorted_p;
    if (ring_sort_mode()) {
        std::vector<int32_t> ord((size_t)np);
        for (int64_t g = 0; g < np; ++g)
            ord[g] = (int32_t)g;
        auto tets = [&](int32_t g) {
            const int32_t m = P0.off[g + 1] - P0.off[g] - 2;
            return P0.closed[g] ? m : m - 1;
        };
        parallel_items(n_chunks, [&](int64_t c, int) {
            std::stable_sort(ord.begin() + spans[c].p0, ord.begin() + spans[c].p1,
                             [&](int32_t x, int32_t y) { return tets(x) > tets(y); });
        }, 64);
        sorted_p.off.assign((size_t)np + 1, 0);
        sorted_p.closed.resize((size_t)np);
        for (int64_t g = 0; g < np; ++g) {
            sorted_p.off[g + 1] = sorted_p.off[g] + (P0.off[ord[g] + 1] - P0.off[ord[g]]);
            sorted_p.closed[g] = P0.closed[ord[g]];
        }
        sorted_p.nodes.resize(P0.nodes.size());
        parallel_for(np, [&](int64_t g0, int64_t g1, int) {
            for (int64_t g = g0; g < g1; ++g)
                std::copy(P0.nodes.begin() + P0.off[ord[g]], P0.nodes.begin() + P0.off[ord[g] + 1],
                          sorted_p.nodes.begin() + sorted_p.off[g]);
        });
        pp = &sorted_p;
    }
    const Patches &P = *pp;
    std::vector<int64_t> nbeg((size_t)n_chunks + 1, 0);
    for (int64_t c = 0; c < n_chunks; ++c)
        nbeg[c + 1] = nbeg[c] + spans[c].nn;
    const int64_t total = nbeg[n_chunks];
    out.chunks.resize((size_t)(5 * n_chunks));
    out.gather_nodes.resize((size_t)total);
    out.cnodes.resize((size_t)total);
    out.runs.resize((size_t)total);
    out.levels.resize((size_t)(CHUNK_LEVELS * n_chunks));

    // pass 2 (parallel over chunks): slot placement, ranks, jagged levels,
    // contribution positions -- each chunk's outputs are disjoint
    struct Scratch {
        std::vector<int32_t> local, cnt, nodes, order, rank, fill, lvl, ncnt;
        BankStats bank, pos;
    };
    std::vector<Scratch> scr((size_t)prep_threads());
    parallel_items(n_chunks, [&](int64_t c, int t) {
        Scratch &S = scr[(size_t)t];
        if (S.local.empty()) {  // node-indexed scratch: written before read, cnt reset after use
            S.local.resize((size_t)std::max<int64_t>(n_nodes, 1));
            S.cnt.assign((size_t)std::max<int64_t>(n_nodes, 1), 0);
        }
        int32_t *local = S.local.data(), *cnt = S.cnt.data();
        const int64_t p_begin = spans[c].p0, p_end = spans[c].p1;
        std::vector<int32_t> &sorted = S.nodes;
        sorted.clear();
        for (int64_t g = p_begin; g < p_end; ++g)
            for (int32_t k = P.off[g]; k < P.off[g + 1]; ++k) {
                const int32_t v = P.nodes[k];
                if (cnt[v]++ == 0)
                    sorted.push_back(v);
            }
        std::sort(sorted.begin(), sorted.end());  // local ids: ascending node id (gather order)
        if (bank_place_mode())                    // or bank-aware slots (above)
            bank_place(P, p_begin, p_end, sorted, local, S.bank);
        const int32_t nn = (int32_t)sorted.size();
        for (int32_t j = 0; j < nn; ++j)
            local[sorted[j]] = j;
        // rank: by contribution count descending, then local id
        std::vector<int32_t> &order = S.order, &rank = S.rank;
        order.resize(nn);
        for (int32_t j = 0; j < nn; ++j)
            order[j] = j;
        std::stable_sort(order.begin(), order.end(),
                         [&](int32_t x, int32_t y) { return cnt[sorted[x]] > cnt[sorted[y]]; });
        rank.assign(nn, 0);
        for (int32_t q = 0; q < nn; ++q)
            rank[order[q]] = q;
        uint16_t *lev = out.levels.data() + (size_t)CHUNK_LEVELS * c;
        lev[0] = 0;
        for (int s = 1; s < CHUNK_LEVELS; ++s) {
            int32_t alive = 0;  // nodes with more than s-1 contributions
            for (int32_t q = 0; q < nn; ++q)
                alive += cnt[sorted[order[q]]] > s - 1;
            lev[s] = (uint16_t)(lev[s - 1] + alive);
        }
        // levels of the patch-order contributions (fill order), then the
        // bank-aware choice of levels (above)
        std::vector<int32_t> &fill = S.fill, &lvl = S.lvl;
        fill.assign(nn, 0);
        lvl.clear();
        for (int64_t g = p_begin; g < p_end; ++g)
            for (int32_t k = P.off[g]; k < P.off[g + 1]; ++k)
                lvl.push_back(fill[local[P.nodes[k]]]++);
        if (pos_place_mode()) {
            S.ncnt.resize(nn);
            for (int32_t j = 0; j < nn; ++j)
                S.ncnt[j] = cnt[sorted[j]];
            pos_place(P, p_begin, p_end, local, S.ncnt, order, rank, lev, lvl, S.pos);
        }
        const int64_t node_begin = nbeg[c];
        for (int32_t j = 0; j < nn; ++j)
            out.gather_nodes[node_begin + j] = sorted[j];
        for (int32_t q = 0; q < nn; ++q) {
            const int32_t v = sorted[order[q]];
            out.cnodes[node_begin + q] = v;
            out.runs[node_begin + q] = (uint8_t)cnt[v];
        }
        size_t ci = 0;  // contribution index in patch order (lvl)
        for (int64_t g = p_begin; g < p_end; ++g) {
            uint16_t *ids = out.pids.data() + PATCH_SLOTS * g, *pos = out.ppos.data() + PATCH_SLOTS * g;
            const int32_t m = P.off[g + 1] - P.off[g] - 2;
            ids[0] = (uint16_t)(m | (P.closed[g] << 8));
            for (int32_t k = 0; k < m + 2; ++k) {
                const int32_t l = local[P.nodes[P.off[g] + k]];
                ids[1 + k] = (uint16_t)l;
                pos[1 + k] = (uint16_t)(lev[lvl[ci++]] + rank[l]);
            }
        }
        for (int32_t v : sorted)
            cnt[v] = 0;
        int32_t *ch = out.chunks.data() + 5 * c;
        ch[0] = (int32_t)p_begin;
        ch[1] = (int32_t)(p_end - p_begin);
        ch[2] = (int32_t)node_begin;
        ch[3] = nn;
        ch[4] = spans[c].contrib;
    }, 4);
    for (auto &S : scr) {  // integer sums: the serial totals
        g_bank.groups += S.bank.groups, g_bank.wave_before += S.bank.wave_before;
        g_bank.wave_after += S.bank.wave_after;
        g_pos.groups += S.pos.groups, g_pos.wave_before += S.pos.wave_before;
        g_pos.wave_after += S.pos.wave_after;
    }

    lap("pass2");
    // interior flag + shared/isolated node lists for the ordered merge
    std::vector<int32_t> cnt_chunks((size_t)n_nodes, 0);
    for (int32_t v : out.cnodes)
        cnt_chunks[v]++;
    auto interior = [&](int64_t v) { return cnt_chunks[v] == 1 && !(external && external[v]); };
    for (int64_t q = 0; q < total; ++q) {
        const int32_t v = out.cnodes[q];
        if (interior(v))
            out.cnodes[q] = (int32_t)((uint32_t)v | 0x80000000u);
    }
    for (int64_t v = 0; v < n_nodes; ++v)
        if (!interior(v)) {
            out.bnd_nodes.push_back((int32_t)v);
            if (cnt_chunks[v] > 1)
                out.n_shared++;
        }
    std::vector<int32_t> bidx((size_t)n_nodes, -1);
    for (size_t i = 0; i < out.bnd_nodes.size(); ++i)
        bidx[out.bnd_nodes[i]] = (int32_t)i;
    out.bnd_off.assign(out.bnd_nodes.size() + 1, 0);
    for (size_t i = 0; i < out.bnd_nodes.size(); ++i)
        out.bnd_off[i + 1] = out.bnd_off[i] + cnt_chunks[out.bnd_nodes[i]];
    out.bnd_pos.resize((size_t)out.bnd_off.back());
    std::vector<int32_t> bfill(out.bnd_off.begin(), out.bnd_off.end() - 1);
    for (int64_t q = 0; q < total; ++q) {
        const uint32_t raw = (uint32_t)out.cnodes[q];
        if (raw & 0x80000000u)
            continue;
        out.bnd_pos[bfill[bidx[raw]]++] = (int32_t)q;
    }
    lap("tail");
    return true;
}

void pack_blobs(const Chunking &ch, int T, std::vector<uint8_t> &blobs, std::vector<int32_t> &blob_off)
{
    const int64_t n_chunks = (int64_t)ch.chunks.size() / 5;
    auto pad = [](int64_t b) { return (b + 15) / 16 * 16; };
    auto blob_bytes = [&](int64_t nn) {
        return 16 + 4 * PATCH_SLOTS * (int64_t)T + 2 * CHUNK_LEVELS + 2 * pad(4 * nn) + pad(nn);
    };
    blob_off.assign((size_t)n_chunks + 1, 0);
    int64_t total = 0;
    for (int64_t c = 0; c < n_chunks; ++c) {
        total += blob_bytes(ch.chunks[5 * c + 3]);
        blob_off[c + 1] = (int32_t)(total / 16);
    }
    blobs.assign((size_t)total, 0);
    parallel_items(n_chunks, [&](int64_t c, int) {
        const int32_t p0 = ch.chunks[5 * c], npch = ch.chunks[5 * c + 1];
        const int32_t n0 = ch.chunks[5 * c + 2], nn = ch.chunks[5 * c + 3];
        uint8_t *b = blobs.data() + (int64_t)blob_off[c] * 16;
        const int32_t hdr[4] = {npch, nn, n0, ch.chunks[5 * c + 4]};
        std::memcpy(b, hdr, 16);
        uint16_t *ids = reinterpret_cast<uint16_t *>(b + 16);
        uint16_t *pos = ids + PATCH_SLOTS * T;
        for (int32_t g = 0; g < npch; ++g)
            for (int s = 0; s < PATCH_SLOTS; ++s) {
                ids[s * T + g] = ch.pids[PATCH_SLOTS * (int64_t)(p0 + g) + s];
                pos[s * T + g] = ch.ppos[PATCH_SLOTS * (int64_t)(p0 + g) + s];
            }
        uint8_t *q = b + 16 + 4 * PATCH_SLOTS * T;
        std::memcpy(q, ch.levels.data() + CHUNK_LEVELS * c, 2 * CHUNK_LEVELS);
        q += 2 * CHUNK_LEVELS;
        std::memcpy(q, ch.gather_nodes.data() + n0, 4 * (size_t)nn);
        q += pad(4 * nn);
        std::memcpy(q, ch.cnodes.data() + n0, 4 * (size_t)nn);
        q += pad(4 * nn);
        std::memcpy(q, ch.runs.data() + n0, (size_t)nn);
    }, 64);
}

}  // namespace tal
