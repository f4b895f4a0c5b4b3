// tal_meshio.hpp -- native mesh IO and RCB partitioning (tal_meshio.cpp).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace tal {

struct MeshText {
    std::vector<double> coords;  // n x 3
    std::vector<int64_t> conn;   // m x 4
    int64_t n_nodes = 0, n_elems = 0, n_reoriented = 0;
    ~MeshText();
};
// The reference's text format (mesh.py:280-371).  On a format error returns
// false with err and err_line (> 0: the offending 1-based line).
bool load_mesh_text(const char *path, MeshText &m, std::string &err, int64_t &err_line);
bool save_mesh_text(const char *path, const double *coords, const int64_t *conn, int64_t n, int64_t e,
                    std::string &err);
// Binary "TALMESH1": 64-byte header + coords (f64) + conn (i64) + hash check.
bool save_mesh_binary(const char *path, const double *coords, const int64_t *conn, int64_t n, int64_t e,
                      std::string &err);
// 1: a TALMESH1 file (sizes returned), 0: not one, -1: cannot open
int probe_mesh_binary(const char *path, int64_t *n, int64_t *e);
bool load_mesh_binary(const char *path, double *coords, int64_t n, int64_t *conn, int64_t e, std::string &err);
// Recursive coordinate bisection of n points into 'world' parts.
void rcb_parts(const double *pts, int64_t n, int world, int32_t *part);

}  // namespace tal
