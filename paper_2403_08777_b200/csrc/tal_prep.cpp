// tal_prep.cpp -- native mesh preprocessing (see tal_prep.hpp).
#include "tal_prep.hpp"

#include <algorithm>
#include <array>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <numeric>

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
    for (int64_t e = 0; e < n_elems; ++e) {
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

// node -> element incidence (CSR)
void node_elements(const int64_t *conn, int64_t n_nodes, int64_t n_elems,
                   std::vector<int64_t> &off, std::vector<int32_t> &adj)
{
    off.assign((size_t)n_nodes + 1, 0);
    for (int64_t i = 0; i < 4 * n_elems; ++i)
        off[conn[i] + 1]++;
    for (int64_t v = 0; v < n_nodes; ++v)
        off[v + 1] += off[v];
    adj.resize((size_t)(4 * n_elems));
    std::vector<int64_t> pos(off.begin(), off.end() - 1);
    for (int64_t e = 0; e < n_elems; ++e)
        for (int a = 0; a < 4; ++a)
            adj[pos[conn[4 * e + a]]++] = (int32_t)e;
}

// one BFS from 'start' over unvisited nodes; neighbours of a node are the
// other nodes of its incident elements; neighbours are appended in order of
// increasing valence (Cuthill-McKee).  Returns the visit order; 'mark' is set.
void cm_bfs(int64_t start, const int64_t *conn, const std::vector<int64_t> &off,
            const std::vector<int32_t> &adj, std::vector<int32_t> &mark, int32_t tag,
            std::vector<int32_t> &order, int64_t *last_level_begin)
{
    order.clear();
    order.push_back((int32_t)start);
    mark[start] = tag;
    size_t head = 0, level_end = 1;
    *last_level_begin = 0;
    std::vector<int32_t> nb;
    while (head < order.size()) {
        if (head == level_end) {
            *last_level_begin = (int64_t)head;
            level_end = order.size();
        }
        const int32_t v = order[head++];
        nb.clear();
        for (int64_t p = off[v]; p < off[v + 1]; ++p) {
            const int64_t e = adj[p];
            for (int a = 0; a < 4; ++a) {
                const int64_t w = conn[4 * e + a];
                if (mark[w] != tag) {
                    mark[w] = tag;
                    nb.push_back((int32_t)w);
                }
            }
        }
        std::sort(nb.begin(), nb.end(), [&](int32_t a, int32_t b) {
            const int64_t da = off[a + 1] - off[a], db = off[b + 1] - off[b];
            return da != db ? da < db : a < b;
        });
        order.insert(order.end(), nb.begin(), nb.end());
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

template <class GetPoint>
void morton_order(int64_t n, GetPoint pt, std::vector<int32_t> &perm, const double *cell = nullptr,
                  const double *origin = nullptr)
{
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = 0; i < n; ++i) {
        double p[3];
        pt(i, p);
        for (int c = 0; c < 3; ++c) {
            lo[c] = std::min(lo[c], p[c]);
            hi[c] = std::max(hi[c], p[c]);
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
    for (int64_t i = 0; i < n; ++i) {
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
    std::sort(key.begin(), key.end());
    perm.resize((size_t)n);
    for (int64_t i = 0; i < n; ++i)
        perm[i] = key[i].i;
}

}  // namespace

void renumber_rcm(const int64_t *conn, int64_t n_nodes, int64_t n_elems, std::vector<int32_t> &perm)
{
    std::vector<int64_t> off;
    std::vector<int32_t> adj;
    node_elements(conn, n_nodes, n_elems, off, adj);
    std::vector<int32_t> mark((size_t)n_nodes, 0), done((size_t)n_nodes, 0);
    std::vector<int32_t> order, result;
    result.reserve((size_t)n_nodes);
    int32_t tag = 0;
    // components in order of their smallest-valence seed
    std::vector<int32_t> seeds((size_t)n_nodes);
    std::iota(seeds.begin(), seeds.end(), 0);
    std::stable_sort(seeds.begin(), seeds.end(), [&](int32_t a, int32_t b) {
        return off[a + 1] - off[a] < off[b + 1] - off[b];
    });
    for (int32_t s : seeds) {
        if (done[s])
            continue;
        // pseudo-peripheral start: two sweeps (George-Liu style)
        int64_t start = s, llb = 0;
        for (int sweep = 0; sweep < 2; ++sweep) {
            cm_bfs(start, conn, off, adj, mark, ++tag, order, &llb);
            int64_t best = order[llb];
            for (size_t i = (size_t)llb; i < order.size(); ++i) {
                const int32_t v = order[i];
                if (off[v + 1] - off[v] < off[best + 1] - off[best])
                    best = v;
            }
            start = best;
        }
        cm_bfs(start, conn, off, adj, mark, ++tag, order, &llb);
        for (int32_t v : order)
            done[v] = 1;
        result.insert(result.end(), order.begin(), order.end());
    }
    std::reverse(result.begin(), result.end());
    perm.swap(result);
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
        for (int64_t e = 0; e < n_elems; ++e) {
            const int32_t *q = conn4 + 4 * e;
            key[e] = {std::min(std::min(q[0], q[1]), std::min(q[2], q[3])), (int32_t)e};
        }
        std::sort(key.begin(), key.end());
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
        for (int64_t e = 0; e < n_elems; ++e) {
            const int32_t *q = conn4 + 4 * e;
            for (int c = 0; c < 3; ++c) {
                double a = coords_int[3 * q[0] + c], b = a;
                for (int k = 1; k < 4; ++k) {
                    a = std::min(a, coords_int[3 * q[k] + c]);
                    b = std::max(b, coords_int[3 * q[k] + c]);
                }
                cell[c] += b - a;
            }
        }
        for (int c = 0; c < 3; ++c)
            cell[c] = n_elems ? cell[c] / (double)n_elems : 0.0;
        morton_order(
            n_elems,
            [&](int64_t e, double p[3]) {
                const int32_t *q = conn4 + 4 * e;
                for (int c = 0; c < 3; ++c)
                    p[c] = 0.25 * (coords_int[3 * q[0] + c] + coords_int[3 * q[1] + c] +
                                   coords_int[3 * q[2] + c] + coords_int[3 * q[3] + c]);
            },
            eperm, cell, lo);
    }
}

namespace {

struct Arc {
    std::vector<int32_t> tets, ring;
    bool closed = false;
};

// ring of unassigned tets around edge (p,q) that contains tet t
void ring_arc(int32_t t, int32_t p, int32_t q, const int32_t *conn4, const std::vector<int64_t> &off,
              const std::vector<int32_t> &adj, const std::vector<uint8_t> &assigned, Arc &arc)
{
    // candidate tets: unassigned, contain p and q; their ring edge (c,d)
    struct Cand {
        int32_t tet, c, d;
        bool used;
    };
    Cand cand[64];
    int nc = 0;
    for (int64_t k = off[p]; k < off[p + 1] && nc < 64; ++k) {
        const int32_t s = adj[k];
        if (assigned[s])
            continue;
        const int32_t *v = conn4 + 4 * (int64_t)s;
        bool hq = false;
        int32_t o[2], no = 0;
        for (int a = 0; a < 4; ++a) {
            if (v[a] == q)
                hq = true;
            else if (v[a] != p && no < 2)
                o[no++] = v[a];
        }
        if (hq && no == 2)
            cand[nc++] = {s, o[0], o[1], s == t};
    }
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
    std::vector<int32_t> fwd{cand[it].d}, bwd{cand[it].c};
    std::vector<int32_t> tf, tb;
    const int max_tets = PATCH_MAX_RING - 1;
    auto walk = [&](std::vector<int32_t> &seq, std::vector<int32_t> &ts, int budget) {
        while ((int)ts.size() < budget) {
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
            ts.push_back(cand[found].tet);
            if (nxt == (&seq == &fwd ? bwd.front() : fwd.front()))
                return true;  // closed the ring
            seq.push_back(nxt);
        }
        return false;
    };
    const bool closed = walk(fwd, tf, max_tets - 1);
    if (!closed)
        walk(bwd, tb, max_tets - 1 - (int)tf.size());
    arc.ring.clear();
    for (auto i = bwd.rbegin(); i != bwd.rend(); ++i)
        arc.ring.push_back(*i);
    for (int32_t v : fwd)
        arc.ring.push_back(v);
    arc.tets.clear();
    for (auto i = tb.rbegin(); i != tb.rend(); ++i)
        arc.tets.push_back(*i);
    arc.tets.push_back(t);
    for (int32_t s : tf)
        arc.tets.push_back(s);
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
    std::vector<int64_t> off((size_t)n_nodes + 1, 0);
    for (int64_t i = 0; i < 4 * n_elems; ++i)
        off[conn4[i] + 1]++;
    for (int64_t v = 0; v < n_nodes; ++v)
        off[v + 1] += off[v];
    std::vector<int32_t> adj((size_t)(4 * n_elems));
    {
        std::vector<int64_t> pos(off.begin(), off.end() - 1);
        for (int64_t e = 0; e < n_elems; ++e)
            for (int a = 0; a < 4; ++a)
                adj[pos[conn4[4 * e + a]]++] = (int32_t)e;
    }
    std::vector<uint8_t> assigned((size_t)n_elems, 0);
    static const int EDGES[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
    Arc best, cur;
    int32_t best_p = 0, best_q = 0;
    for (int64_t t = 0; t < n_elems; ++t) {
        if (assigned[t])
            continue;
        const int32_t *v = conn4 + 4 * t;
        size_t best_n = 0;
        int64_t best_span = 0;
        for (auto &ed : EDGES) {
            const int32_t p = v[ed[0]], q = v[ed[1]];
            ring_arc((int32_t)t, p, q, conn4, off, adj, assigned, cur);
            int64_t lo = cur.tets[0], hi = cur.tets[0];
            for (int32_t s : cur.tets) {
                lo = std::min<int64_t>(lo, s);
                hi = std::max<int64_t>(hi, s);
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
        for (int32_t s : best.tets)
            assigned[s] = 1;
        out.nodes.push_back(best_p);
        out.nodes.push_back(best_q);
        for (int32_t r : best.ring)
            out.nodes.push_back(r);
        out.off.push_back((int32_t)out.nodes.size());
        out.closed.push_back(best.closed ? 1 : 0);
    }
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
                std::vector<int32_t> &idx)
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
    g_bank.groups += groups;
    g_bank.wave_before += before;
    g_bank.wave_after += waves();
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

void pos_place(const Patches &P, int64_t p0, int64_t p1, const std::vector<int32_t> &local,
               const std::vector<int32_t> &ncnt, std::vector<int32_t> &order, std::vector<int32_t> &rank,
               const uint16_t *lev, std::vector<int32_t> &lvl)
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
    g_pos.groups += before.second;
    g_pos.wave_before += before.first;
    g_pos.wave_after += after.first;
}
}  // namespace

void pos_stats(int64_t *groups, int64_t *before, int64_t *after)
{
    *groups = g_pos.groups, *before = g_pos.wave_before, *after = g_pos.wave_after;
}

bool build_chunks(const Patches &P, int64_t n_nodes, int max_patches, int max_nodes, int max_contrib,
                  const uint8_t *external, Chunking &out, std::string &err)
{
    if (max_patches < 1 || max_nodes < PATCH_MAX_RING + 2 || max_contrib < PATCH_MAX_RING + 2 ||
        max_contrib > 65535 || max_nodes > 65535) {
        err = "invalid chunk limits";
        return false;
    }
    out = Chunking();
    out.max_patches = max_patches;
    out.max_nodes = max_nodes;
    out.max_contrib = max_contrib;
    const int64_t np = P.n_patches();
    out.pids.assign((size_t)np * PATCH_SLOTS, 0);
    out.ppos.assign((size_t)np * PATCH_SLOTS, 0);
    std::vector<int32_t> stamp((size_t)n_nodes, -1), local((size_t)n_nodes, 0), cnt((size_t)n_nodes, 0);
    std::vector<int32_t> cnt_chunks((size_t)n_nodes, 0);
    std::vector<int32_t> nodes, order, rank, fill, lvl, ncnt;
    int32_t chunk = 0;
    int64_t p_begin = 0, contrib = 0;

    auto close_chunk = [&](int64_t p_end) {
        std::vector<int32_t> sorted(nodes);
        std::sort(sorted.begin(), sorted.end());  // local ids: ascending node id (gather order)
        if (bank_place_mode())                    // or bank-aware slots (above)
            bank_place(P, p_begin, p_end, sorted, local);
        const int32_t nn = (int32_t)sorted.size();
        for (int32_t j = 0; j < nn; ++j)
            local[sorted[j]] = j;
        // rank: by contribution count descending, then local id
        order.resize(nn);
        for (int32_t j = 0; j < nn; ++j)
            order[j] = j;
        std::stable_sort(order.begin(), order.end(),
                         [&](int32_t x, int32_t y) { return cnt[sorted[x]] > cnt[sorted[y]]; });
        rank.assign(nn, 0);
        for (int32_t q = 0; q < nn; ++q)
            rank[order[q]] = q;
        uint16_t lev[CHUNK_LEVELS] = {0};
        for (int s = 1; s < CHUNK_LEVELS; ++s) {
            int32_t alive = 0;  // nodes with more than s-1 contributions
            for (int32_t q = 0; q < nn; ++q)
                alive += cnt[sorted[order[q]]] > s - 1;
            lev[s] = (uint16_t)(lev[s - 1] + alive);
        }
        // levels of the patch-order contributions (fill order), then the
        // bank-aware choice of levels / equal-count ranks (above)
        fill.assign(nn, 0);
        lvl.clear();
        for (int64_t g = p_begin; g < p_end; ++g)
            for (int32_t k = P.off[g]; k < P.off[g + 1]; ++k)
                lvl.push_back(fill[local[P.nodes[k]]]++);
        if (pos_place_mode()) {
            ncnt.resize(nn);
            for (int32_t j = 0; j < nn; ++j)
                ncnt[j] = cnt[sorted[j]];
            pos_place(P, p_begin, p_end, local, ncnt, order, rank, lev, lvl);
        }
        const size_t node_begin = out.cnodes.size();
        for (int32_t j = 0; j < nn; ++j)
            out.gather_nodes.push_back(sorted[j]);
        for (int32_t q = 0; q < nn; ++q) {
            const int32_t v = sorted[order[q]];
            out.cnodes.push_back(v);
            out.runs.push_back((uint8_t)cnt[v]);
            cnt_chunks[v]++;
        }
        for (int s = 0; s < CHUNK_LEVELS; ++s)
            out.levels.push_back(lev[s]);
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
        out.chunks.push_back((int32_t)p_begin);
        out.chunks.push_back((int32_t)(p_end - p_begin));
        out.chunks.push_back((int32_t)node_begin);
        out.chunks.push_back(nn);
        out.chunks.push_back((int32_t)contrib);
        nodes.clear();
        ++chunk;
        p_begin = p_end;
        contrib = 0;
    };

    for (int64_t g = 0; g < np; ++g) {
        const int32_t n = P.off[g + 1] - P.off[g];
        if (n - 2 > PATCH_MAX_RING || n < 4) {
            err = "patch ring size out of range";
            return false;
        }
        int fresh = 0;
        bool full_level = false;
        for (int32_t k = P.off[g]; k < P.off[g + 1]; ++k) {
            const int32_t v = P.nodes[k];
            if (stamp[v] != chunk)
                ++fresh;
            else if (cnt[v] + 1 > CHUNK_LEVELS)
                full_level = true;
        }
        if (g > p_begin && ((g - p_begin) + 1 > max_patches || (int64_t)nodes.size() + fresh > max_nodes ||
                            contrib + n > max_contrib || full_level))
            close_chunk(g);
        for (int32_t k = P.off[g]; k < P.off[g + 1]; ++k) {
            const int32_t v = P.nodes[k];
            if (stamp[v] != chunk) {
                stamp[v] = chunk;
                nodes.push_back(v);
            }
            cnt[v]++;
        }
        contrib += n;
    }
    if (np > p_begin)
        close_chunk(np);

    // interior flag + shared/isolated node lists for the ordered merge
    const int64_t total = (int64_t)out.cnodes.size();
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
    for (int64_t c = 0; c < n_chunks; ++c) {
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
    }
}

}  // namespace tal
