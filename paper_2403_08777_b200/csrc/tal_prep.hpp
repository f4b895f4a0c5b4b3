// tal_prep.hpp -- native host-side mesh preprocessing for the device layout.
//
// Everything here runs once per mesh upload (the reference does its own
// once-per-mesh work -- Mesh validation mesh.py:50-75, colouring
// variants.py:565-570 -- before its timer starts, variants.py:572).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace tal {

// Kuhn 6-tet split of an nx*ny*nz box (mesh.py:145-184).
void box_mesh(int64_t nx, int64_t ny, int64_t nz, double ex, double ey, double ez,
              double *coords, int64_t *conn);

void signed_volumes(const double *coords, const int64_t *conn, int64_t n_elems, double *vols);

// Greedy lowest-free colouring in element order (mesh.py:235-257).
// Returns number of colours, or -1 if more than 256 colours would be needed.
int64_t color_elements(const int64_t *conn, int64_t n_nodes, int64_t n_elems, int64_t *colors);
bool check_coloring(const int64_t *conn, const int64_t *colors, int64_t n_nodes, int64_t n_elems);

// perm[new] = old.
void renumber_rcm(const int64_t *conn, int64_t n_nodes, int64_t n_elems, std::vector<int32_t> &perm);
void renumber_sfc(const double *coords, int64_t n_nodes, std::vector<int32_t> &perm);
// element order eperm[new] = old for the given TAL_EORDER_*, on internal conn.
void element_order(int method, const int32_t *conn4, const double *coords_int, int64_t n_nodes,
                   int64_t n_elems, std::vector<int32_t> &eperm);

// CTA chunking for the private scatter.
struct Chunking {
    int chunk_elems = 0, max_nodes = 0;
    std::vector<int32_t> chunks;       // 4 per chunk: elem_begin, n_elem, node_begin, n_node
    std::vector<int32_t> chunk_nodes;  // node id | (1u<<31 if the node is interior to the chunk)
    std::vector<uint16_t> csr_off;     // per chunk node: first slot index (chunk-relative)
    std::vector<uint16_t> csr_slots;   // 4 per element: slot = corner*chunk_elems + e_local
    std::vector<uint16_t> lconn;       // 4 per element: chunk-local node ids
    // deterministic merge: for nodes in >1 chunk (and isolated nodes), the
    // chunk-node positions holding their partial sums, in chunk order
    std::vector<int32_t> bnd_nodes, bnd_off, bnd_pos;
    int64_t n_shared = 0;
};
bool build_chunks(const int32_t *conn4, int64_t n_nodes, int64_t n_elems, int chunk_elems,
                  int chunk_nodes, Chunking &out, std::string &err);

}  // namespace tal
