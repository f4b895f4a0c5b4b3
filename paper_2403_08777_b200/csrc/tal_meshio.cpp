// tal_meshio.cpp -- native mesh IO and partitioning.
//
//  * The reference's text format (mesh.py:280-371, save_mesh / load_mesh):
//    "nodes <n>", n lines "x y z" (%.17g), "elems <m>", m lines of 4
//    zero-based node ids; '#' starts a comment, blank lines are skipped;
//    inverted elements are re-oriented on load (last two nodes swapped) and
//    counted.  Formatting runs in parallel blocks written in order (bytes
//    identical to the reference's writer); parsing is one pass over the
//    mapped file with line numbers kept for the errors.
//  * A binary format for large meshes ("TALMESH1"): a 64-byte little-endian
//    header {magic, version, n_nodes, n_elems, flags, content hash} followed
//    by coords (f64, n x 3) and connectivity (i64, m x 4): one read per
//    array, exact round trip, the hash checked on load.
//  * Recursive coordinate bisection (distributed.py MeshPartition): the
//    parts of a point set, bit-identical to the numpy statement of the
//    algorithm it replaces (stable sort along the widest axis, cut at
//    size * floor(k/2) / k), sub-problems run in parallel.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "tal_meshio.hpp"
#include "tal_par.hpp"
#include "tal_prep.hpp"

namespace tal {

namespace {

struct Line {
    int64_t no;           // 1-based line number
    const char *b, *e;    // content without comment / surrounding blanks
};

// split [b, e) into whitespace-separated tokens (at most 'cap'); returns count
int tokens(const char *b, const char *e, const char **tb, const char **te, int cap)
{
    int n = 0;
    while (b < e) {
        while (b < e && (*b == ' ' || *b == '\t' || *b == '\r' || *b == '\v' || *b == '\f'))
            ++b;
        if (b >= e)
            break;
        const char *s = b;
        while (b < e && !(*b == ' ' || *b == '\t' || *b == '\r' || *b == '\v' || *b == '\f'))
            ++b;
        if (n < cap)
            tb[n] = s, te[n] = b;
        ++n;
    }
    return n;
}

bool parse_double(const char *b, const char *e, double *out)
{
    char buf[128];
    const size_t n = (size_t)(e - b);
    if (n == 0 || n >= sizeof buf)
        return false;
    std::memcpy(buf, b, n);
    buf[n] = 0;
    if (buf[0] == '0' && (buf[1] == 'x' || buf[1] == 'X'))  // hex floats: not Python float()
        return false;
    char *end = nullptr;
    errno = 0;
    *out = std::strtod(buf, &end);
    return end == buf + n;
}

bool parse_int(const char *b, const char *e, int64_t *out)
{
    char buf[64];
    const size_t n = (size_t)(e - b);
    if (n == 0 || n >= sizeof buf)
        return false;
    std::memcpy(buf, b, n);
    buf[n] = 0;
    char *end = nullptr;
    errno = 0;
    *out = std::strtoll(buf, &end, 10);
    return end == buf + n && errno == 0;
}

std::string tok_text(const Line &l)
{
    std::string s(l.b, l.e);
    // collapse runs of blanks like ' '.join(parts)
    std::string o;
    bool sp = false;
    for (char c : s) {
        const bool w = c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f';
        if (w) {
            sp = !o.empty();
        } else {
            if (sp)
                o += ' ';
            o += c;
            sp = false;
        }
    }
    return o;
}

}  // namespace

MeshText::~MeshText() = default;

bool load_mesh_text(const char *path, MeshText &m, std::string &err, int64_t &err_line)
{
    err_line = 0;
    FILE *f = std::fopen(path, "rb");
    if (!f) {
        err = std::string("cannot open ") + path + ": " + std::strerror(errno);
        return false;
    }
    std::vector<char> data;
    {
        std::fseek(f, 0, SEEK_END);
        const long sz = std::ftell(f);
        std::fseek(f, 0, SEEK_SET);
        data.resize((size_t)std::max(sz, 0L));
        if (sz > 0 && std::fread(data.data(), 1, (size_t)sz, f) != (size_t)sz) {
            std::fclose(f);
            err = std::string("read error on ") + path;
            return false;
        }
        std::fclose(f);
    }
    // non-blank lines (comment-stripped), with their numbers
    std::vector<Line> lines;
    {
        const char *p = data.data(), *end = p + data.size();
        int64_t no = 0;
        while (p < end) {
            const char *nl = (const char *)std::memchr(p, '\n', (size_t)(end - p));
            const char *le = nl ? nl : end;
            ++no;
            const char *hash = (const char *)std::memchr(p, '#', (size_t)(le - p));
            const char *ce = hash ? hash : le;
            const char *b = p;
            while (b < ce && std::isspace((unsigned char)*b))
                ++b;
            const char *e = ce;
            while (e > b && std::isspace((unsigned char)e[-1]))
                --e;
            if (b < e)
                lines.push_back({no, b, e});
            p = nl ? nl + 1 : end;
        }
    }
    size_t pos = 0;
    auto take = [&](const char *what, Line &l) {
        if (pos >= lines.size()) {
            err = std::string("unexpected end of file, expected ") + what;
            err_line = lines.empty() ? 1 : lines.back().no;
            return false;
        }
        l = lines[pos++];
        return true;
    };
    const char *tb[8], *te[8];
    Line l;
    auto header = [&](const char *word, const char *what, const char *noun, int64_t &count) {
        if (!take(what, l))
            return false;
        const int nt = tokens(l.b, l.e, tb, te, 8);
        if (nt != 2 || (size_t)(te[0] - tb[0]) != std::strlen(word) ||
            std::strncmp(tb[0], word, std::strlen(word)) != 0) {
            err = std::string("expected '") + word + " <" + (word[0] == 'n' ? "n" : "m") + ">', got '" +
                  tok_text(l) + "'";
            err_line = l.no;
            return false;
        }
        if (!parse_int(tb[1], te[1], &count) || count < 0) {
            err = std::string("bad ") + noun + " count '" + std::string(tb[1], te[1]) + "'";
            err_line = l.no;
            return false;
        }
        return true;
    };
    int64_t n = 0, e = 0;
    if (!header("nodes", "'nodes <n>'", "node", n))
        return false;
    // lines are parsed as the reference reads them: the first bad one among
    // those present wins, then a missing one (end of file)
    const int64_t nav = std::min<int64_t>(n, (int64_t)(lines.size() - pos));
    m.coords.resize((size_t)(3 * n));
    // parse the n coordinate lines in parallel; the first error (lowest line) wins
    std::vector<int64_t> bad_at((size_t)prep_threads(), -1);
    std::vector<std::string> bad_msg((size_t)prep_threads());
    const size_t c0 = pos;
    parallel_for(nav, [&](int64_t i0, int64_t i1, int t) {
        const char *b2[8], *e2[8];
        for (int64_t i = i0; i < i1; ++i) {
            const Line &q = lines[c0 + i];
            const int nt = tokens(q.b, q.e, b2, e2, 8);
            if (nt != 3) {
                bad_at[t] = i, bad_msg[t] = "expected 3 coordinates, got " + std::to_string(nt);
                return;
            }
            for (int c = 0; c < 3; ++c)
                if (!parse_double(b2[c], e2[c], &m.coords[3 * i + c])) {
                    bad_at[t] = i, bad_msg[t] = "bad coordinate in '" + tok_text(q) + "'";
                    return;
                }
        }
    }, 1 << 12);
    for (size_t t = 0; t < bad_at.size(); ++t)
        if (bad_at[t] >= 0) {
            err = bad_msg[t], err_line = lines[c0 + bad_at[t]].no;
            return false;
        }
    if (nav < n) {
        pos = lines.size();
        take("a coordinate line", l);
        return false;
    }
    pos += (size_t)n;
    if (!header("elems", "'elems <m>'", "element", e))
        return false;
    const int64_t eav = std::min<int64_t>(e, (int64_t)(lines.size() - pos));
    m.conn.resize((size_t)(4 * e));
    std::fill(bad_at.begin(), bad_at.end(), -1);
    const size_t e0 = pos;
    parallel_for(eav, [&](int64_t i0, int64_t i1, int t) {
        const char *b2[8], *e2[8];
        for (int64_t i = i0; i < i1; ++i) {
            const Line &q = lines[e0 + i];
            const int nt = tokens(q.b, q.e, b2, e2, 8);
            if (nt != 4) {
                bad_at[t] = i, bad_msg[t] = "expected 4 node indices, got " + std::to_string(nt);
                return;
            }
            for (int c = 0; c < 4; ++c)
                if (!parse_int(b2[c], e2[c], &m.conn[4 * i + c])) {
                    bad_at[t] = i, bad_msg[t] = "bad node index in '" + tok_text(q) + "'";
                    return;
                }
        }
    }, 1 << 12);
    for (size_t t = 0; t < bad_at.size(); ++t)
        if (bad_at[t] >= 0) {
            err = bad_msg[t], err_line = lines[e0 + bad_at[t]].no;
            return false;
        }
    if (eav < e) {
        pos = lines.size();
        take("an element line", l);
        return false;
    }
    pos += (size_t)e;
    if (pos != lines.size()) {
        err = "trailing content after element section";
        err_line = lines[pos].no;
        return false;
    }
    for (int64_t i = 0; i < 4 * e; ++i)
        if (m.conn[i] < 0 || m.conn[i] >= n) {
            err = "connectivity index out of range [0, n_nodes)";
            return false;  // err_line 0: a plain ValueError, as the reference raises
        }
    // re-orient inverted elements (mesh.py:360-370)
    std::vector<double> vols((size_t)e);
    signed_volumes(m.coords.data(), m.conn.data(), e, vols.data());
    m.n_reoriented = 0;
    for (int64_t k = 0; k < e; ++k)
        if (vols[k] < 0.0) {
            std::swap(m.conn[4 * k + 2], m.conn[4 * k + 3]);
            ++m.n_reoriented;
        }
    m.n_nodes = n, m.n_elems = e;
    return true;
}

bool save_mesh_text(const char *path, const double *coords, const int64_t *conn, int64_t n, int64_t e,
                    std::string &err)
{
    FILE *f = std::fopen(path, "wb");
    if (!f) {
        err = std::string("cannot open ") + path + ": " + std::strerror(errno);
        return false;
    }
    // blocks formatted in parallel, written in order
    const int64_t BLK = 1 << 16;
    bool ok = true;
    auto emit = [&](int64_t count, auto fmt) {
        const int64_t nb = (count + BLK - 1) / BLK;
        for (int64_t g0 = 0; g0 < nb && ok; g0 += 64) {
            const int64_t g1 = std::min(nb, g0 + 64);
            std::vector<std::string> out((size_t)(g1 - g0));
            parallel_items(g1 - g0, [&](int64_t j, int) {
                std::string &s = out[(size_t)j];
                char buf[160];
                for (int64_t i = (g0 + j) * BLK, ie = std::min(count, (g0 + j + 1) * BLK); i < ie; ++i) {
                    const int len = fmt(i, buf);
                    s.append(buf, (size_t)len);
                }
            }, 1);
            for (auto &s : out)
                if (std::fwrite(s.data(), 1, s.size(), f) != s.size())
                    ok = false;
        }
    };
    std::fprintf(f, "nodes %lld\n", (long long)n);
    emit(n, [&](int64_t i, char *buf) {
        return std::snprintf(buf, 160, "%.17g %.17g %.17g\n", coords[3 * i], coords[3 * i + 1], coords[3 * i + 2]);
    });
    std::fprintf(f, "elems %lld\n", (long long)e);
    emit(e, [&](int64_t i, char *buf) {
        return std::snprintf(buf, 160, "%lld %lld %lld %lld\n", (long long)conn[4 * i], (long long)conn[4 * i + 1],
                             (long long)conn[4 * i + 2], (long long)conn[4 * i + 3]);
    });
    if (std::fclose(f) != 0 || !ok) {
        err = std::string("write error on ") + path;
        return false;
    }
    return true;
}

// ---- binary ----------------------------------------------------------------
namespace {
constexpr char BIN_MAGIC[8] = {'T', 'A', 'L', 'M', 'E', 'S', 'H', '1'};
struct BinHeader {
    char magic[8];
    uint32_t version, flags;
    int64_t n_nodes, n_elems;
    uint64_t hash;
    uint8_t pad[24];
};
static_assert(sizeof(BinHeader) == 64, "binary mesh header is 64 bytes");

uint64_t mix_hash(const void *p, size_t bytes, uint64_t seed)
{
    // order-fixed block hash (parallel blocks, combined in block order)
    const size_t B = 1 << 20, nb = (bytes + B - 1) / B;
    std::vector<uint64_t> hb(nb);
    parallel_items((int64_t)nb, [&](int64_t b, int) {
        const uint8_t *q = (const uint8_t *)p + b * B;
        const size_t n = std::min(B, bytes - b * B);
        uint64_t x = 0x9e3779b97f4a7c15ull ^ (uint64_t)b;
        size_t i = 0;
        for (; i + 8 <= n; i += 8) {
            uint64_t w;
            std::memcpy(&w, q + i, 8);
            x = (x ^ w) * 0xff51afd7ed558ccdull;
            x ^= x >> 29;
        }
        for (; i < n; ++i)
            x = (x ^ q[i]) * 0xc4ceb9fe1a85ec53ull;
        hb[(size_t)b] = x;
    }, 4);
    uint64_t h = seed ^ bytes;
    for (uint64_t x : hb)
        h = (h ^ x) * 0x100000001b3ull + 0x9e3779b97f4a7c15ull;
    return h;
}
}  // namespace

bool save_mesh_binary(const char *path, const double *coords, const int64_t *conn, int64_t n, int64_t e,
                      std::string &err)
{
    BinHeader h{};
    std::memcpy(h.magic, BIN_MAGIC, 8);
    h.version = 1;
    h.n_nodes = n, h.n_elems = e;
    h.hash = mix_hash(conn, sizeof(int64_t) * 4 * (size_t)e, mix_hash(coords, sizeof(double) * 3 * (size_t)n, 1));
    FILE *f = std::fopen(path, "wb");
    if (!f) {
        err = std::string("cannot open ") + path + ": " + std::strerror(errno);
        return false;
    }
    bool ok = std::fwrite(&h, sizeof h, 1, f) == 1;
    ok = ok && (n == 0 || std::fwrite(coords, sizeof(double) * 3, (size_t)n, f) == (size_t)n);
    ok = ok && (e == 0 || std::fwrite(conn, sizeof(int64_t) * 4, (size_t)e, f) == (size_t)e);
    if (std::fclose(f) != 0 || !ok) {
        err = std::string("write error on ") + path;
        return false;
    }
    return true;
}

int probe_mesh_binary(const char *path, int64_t *n, int64_t *e)
{
    FILE *f = std::fopen(path, "rb");
    if (!f)
        return -1;
    BinHeader h{};
    const bool ok = std::fread(&h, sizeof h, 1, f) == 1;
    std::fclose(f);
    if (!ok || std::memcmp(h.magic, BIN_MAGIC, 8) != 0)
        return 0;
    *n = h.n_nodes, *e = h.n_elems;
    return 1;
}

bool load_mesh_binary(const char *path, double *coords, const int64_t n, int64_t *conn, const int64_t e,
                      std::string &err)
{
    FILE *f = std::fopen(path, "rb");
    if (!f) {
        err = std::string("cannot open ") + path + ": " + std::strerror(errno);
        return false;
    }
    BinHeader h{};
    bool ok = std::fread(&h, sizeof h, 1, f) == 1 && std::memcmp(h.magic, BIN_MAGIC, 8) == 0 && h.version == 1 &&
              h.n_nodes == n && h.n_elems == e;
    ok = ok && (n == 0 || std::fread(coords, sizeof(double) * 3, (size_t)n, f) == (size_t)n);
    ok = ok && (e == 0 || std::fread(conn, sizeof(int64_t) * 4, (size_t)e, f) == (size_t)e);
    char extra;
    const bool trailing = ok && std::fread(&extra, 1, 1, f) == 1;
    std::fclose(f);
    if (!ok || trailing) {
        err = std::string(path) + ": not a complete TALMESH1 file of the announced size";
        return false;
    }
    const uint64_t hh =
        mix_hash(conn, sizeof(int64_t) * 4 * (size_t)e, mix_hash(coords, sizeof(double) * 3 * (size_t)n, 1));
    if (hh != h.hash) {
        err = std::string(path) + ": content hash mismatch (corrupted file)";
        return false;
    }
    return true;
}

// ---- recursive coordinate bisection ---------------------------------------
void rcb_parts(const double *pts, int64_t n, int world, int32_t *part)
{
    struct Task {
        std::vector<int64_t> idx;
        int first, k;
    };
    std::vector<int64_t> all((size_t)n);
    std::iota(all.begin(), all.end(), 0);
    std::vector<Task> level(1);
    level[0].idx.swap(all);
    level[0].first = 0;
    level[0].k = world;
    while (!level.empty()) {
        std::vector<Task> next_level((size_t)2 * level.size());
        std::vector<uint8_t> used(next_level.size(), 0);
        parallel_items((int64_t)level.size(), [&](int64_t j, int) {
            Task &T = level[(size_t)j];
            if (T.k == 1 || T.idx.empty()) {
                for (int64_t i : T.idx)
                    part[i] = T.first;
                return;
            }
            const int kl = T.k / 2;
            double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
            for (int64_t i : T.idx)
                for (int c = 0; c < 3; ++c) {
                    lo[c] = std::min(lo[c], pts[3 * i + c]);
                    hi[c] = std::max(hi[c], pts[3 * i + c]);
                }
            int ax = 0;  // numpy argmax: the first maximal extent
            for (int c = 1; c < 3; ++c)
                if (hi[c] - lo[c] > hi[ax] - lo[ax])
                    ax = c;
            // numpy argsort(kind="stable") of the axis values, ties in subset order
            std::vector<int64_t> ord(T.idx.size());
            std::iota(ord.begin(), ord.end(), 0);
            std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) {
                return pts[3 * T.idx[a] + ax] < pts[3 * T.idx[b] + ax];
            });
            const size_t cut = (T.idx.size() * (size_t)kl) / (size_t)T.k;
            Task &L = next_level[2 * j], &R = next_level[2 * j + 1];
            L.idx.resize(cut), R.idx.resize(T.idx.size() - cut);
            for (size_t i = 0; i < cut; ++i)
                L.idx[i] = T.idx[ord[i]];
            for (size_t i = cut; i < ord.size(); ++i)
                R.idx[i - cut] = T.idx[ord[i]];
            L.first = T.first, L.k = kl;
            R.first = T.first + kl, R.k = T.k - kl;
            used[2 * j] = used[2 * j + 1] = 1;
            std::vector<int64_t>().swap(T.idx);
        }, 1);
        std::vector<Task> keep;
        for (size_t j = 0; j < next_level.size(); ++j)
            if (used[j])
                keep.push_back(std::move(next_level[j]));
        level.swap(keep);
    }
}

}  // namespace tal
