// tal_prep.cpp -- native mesh preprocessing (see tal_prep.hpp).
#include "tal_prep.hpp"

#include <algorithm>
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

template <class GetPoint>
void morton_order(int64_t n, GetPoint pt, std::vector<int32_t> &perm)
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
    std::vector<std::pair<uint64_t, int32_t>> key((size_t)n);
    for (int64_t i = 0; i < n; ++i) {
        double p[3];
        pt(i, p);
        uint64_t code = 0;
        for (int c = 0; c < 3; ++c)
            code |= spread3((uint64_t)((p[c] - lo[c]) * scale)) << c;
        key[i] = {code, (int32_t)i};
    }
    std::sort(key.begin(), key.end());
    perm.resize((size_t)n);
    for (int64_t i = 0; i < n; ++i)
        perm[i] = key[i].second;
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
    (void)n_nodes;
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
    } else if (method == 2) {  // Morton order of centroids
        morton_order(
            n_elems,
            [&](int64_t e, double p[3]) {
                const int32_t *q = conn4 + 4 * e;
                for (int c = 0; c < 3; ++c)
                    p[c] = 0.25 * (coords_int[3 * q[0] + c] + coords_int[3 * q[1] + c] +
                                   coords_int[3 * q[2] + c] + coords_int[3 * q[3] + c]);
            },
            eperm);
    }
}

bool build_chunks(const int32_t *conn4, int64_t n_nodes, int64_t n_elems, int chunk_elems,
                  int chunk_nodes, Chunking &out, std::string &err)
{
    if (chunk_elems < 1 || chunk_elems > 1024 || chunk_nodes < 4 || chunk_nodes > 2048) {
        err = "chunk_elems must be in [1,1024] and chunk_nodes in [4,2048]";
        return false;
    }
    if (4 * chunk_elems > 65535) {
        err = "chunk_elems too large for 16-bit slots";
        return false;
    }
    out = Chunking();
    out.chunk_elems = chunk_elems;
    out.max_nodes = chunk_nodes;
    out.lconn.resize((size_t)n_elems * 4);
    out.csr_slots.resize((size_t)n_elems * 4);
    std::vector<int32_t> stamp((size_t)n_nodes, -1), local((size_t)n_nodes, 0);
    std::vector<int32_t> cnt_chunks((size_t)n_nodes, 0);
    std::vector<int32_t> nodes;  // current chunk's nodes (first-seen order)
    std::vector<int32_t> counts;
    nodes.reserve(chunk_nodes);
    int32_t chunk = 0;
    int64_t e_begin = 0;

    auto close_chunk = [&](int64_t e_end) {
        // sort the chunk's nodes ascending (coalesced staging loads), then
        // rewrite local ids and build the chunk-local node->slot CSR
        std::vector<int32_t> sorted(nodes);
        std::sort(sorted.begin(), sorted.end());
        for (size_t j = 0; j < sorted.size(); ++j)
            local[sorted[j]] = (int32_t)j;
        const int32_t nn = (int32_t)sorted.size(), ne = (int32_t)(e_end - e_begin);
        counts.assign((size_t)nn + 1, 0);
        for (int64_t e = e_begin; e < e_end; ++e)
            for (int a = 0; a < 4; ++a) {
                const int32_t l = local[conn4[4 * e + a]];
                out.lconn[4 * e + a] = (uint16_t)l;
                counts[l + 1]++;
            }
        for (int32_t j = 0; j < nn; ++j)
            counts[j + 1] += counts[j];
        const size_t node_begin = out.chunk_nodes.size();
        for (int32_t j = 0; j < nn; ++j) {
            out.chunk_nodes.push_back(sorted[j]);
            out.csr_off.push_back((uint16_t)counts[j]);
            cnt_chunks[sorted[j]]++;
        }
        std::vector<int32_t> fill(counts.begin(), counts.end() - 1);
        for (int64_t e = e_begin; e < e_end; ++e)  // element order within each node
            for (int a = 0; a < 4; ++a) {
                const int32_t l = out.lconn[4 * e + a];
                out.csr_slots[4 * e_begin + fill[l]++] =
                    (uint16_t)(a * chunk_elems + (int32_t)(e - e_begin));
            }
        out.chunks.push_back((int32_t)e_begin);
        out.chunks.push_back(ne);
        out.chunks.push_back((int32_t)node_begin);
        out.chunks.push_back(nn);
        nodes.clear();
        ++chunk;
        e_begin = e_end;
    };

    for (int64_t e = 0; e < n_elems; ++e) {
        const int32_t *q = conn4 + 4 * e;
        int fresh = 0;
        for (int a = 0; a < 4; ++a) {
            bool dup = false;
            for (int b = 0; b < a; ++b)
                dup |= (q[b] == q[a]);
            if (!dup && stamp[q[a]] != chunk)
                ++fresh;
        }
        if (e > e_begin && ((e - e_begin) + 1 > chunk_elems ||
                            (int64_t)nodes.size() + fresh > chunk_nodes))
            close_chunk(e);
        for (int a = 0; a < 4; ++a)
            if (stamp[q[a]] != chunk) {
                stamp[q[a]] = chunk;
                nodes.push_back(q[a]);
            }
    }
    if (n_elems > e_begin)
        close_chunk(n_elems);

    // interior flag + shared/isolated node lists for the ordered merge
    const int64_t total = (int64_t)out.chunk_nodes.size();
    std::vector<int32_t> pos_count((size_t)n_nodes + 1, 0);
    for (int64_t p = 0; p < total; ++p) {
        const int32_t v = out.chunk_nodes[p];
        if (cnt_chunks[v] == 1)
            out.chunk_nodes[p] = (int32_t)((uint32_t)v | 0x80000000u);
    }
    for (int64_t v = 0; v < n_nodes; ++v)
        if (cnt_chunks[v] != 1) {
            out.bnd_nodes.push_back((int32_t)v);
            if (cnt_chunks[v] > 1)
                out.n_shared++;
        }
    // positions per boundary node, in chunk order
    std::vector<int32_t> bidx((size_t)n_nodes, -1);
    for (size_t i = 0; i < out.bnd_nodes.size(); ++i)
        bidx[out.bnd_nodes[i]] = (int32_t)i;
    out.bnd_off.assign(out.bnd_nodes.size() + 1, 0);
    for (size_t i = 0; i < out.bnd_nodes.size(); ++i)
        out.bnd_off[i + 1] = out.bnd_off[i] + cnt_chunks[out.bnd_nodes[i]];
    out.bnd_pos.resize((size_t)out.bnd_off.back());
    std::vector<int32_t> bfill(out.bnd_off.begin(), out.bnd_off.end() - 1);
    for (int64_t p = 0; p < total; ++p) {
        const uint32_t raw = (uint32_t)out.chunk_nodes[p];
        if (raw & 0x80000000u)
            continue;
        const int32_t b = bidx[raw];
        out.bnd_pos[bfill[b]++] = (int32_t)p;
    }
    return true;
}

}  // namespace tal
