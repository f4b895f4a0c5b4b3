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

// Patches: the unit of work of one thread in the private scatter.  A patch
// is the ring of tets around one edge (a,b): ring nodes r_0..r_{m-1}, tet i =
// (a, b, r_i, r_{i+1}) for i < k, with k = m for a closed ring (r_m = r_0)
// and k = m - 1 for an open one.  A lone tet (c0,c1,c2,c3) is the open ring
// a=c0, b=c1, r=(c2,c3).  Tets keep no corner order: the symmetric-rule
// element operator is invariant under corner permutation (|det|, sgn det).
constexpr int PATCH_SLOTS = 12;                    // u16 slots per patch table row
constexpr int PATCH_MAX_RING = PATCH_SLOTS - 3;     // ring nodes per patch (m|closed, a, b, r..)
struct Patches {
    std::vector<int32_t> off;    // n_patches + 1, into nodes
    std::vector<int32_t> nodes;  // a, b, r_0 .. r_{m-1}
    std::vector<uint8_t> closed;
    int64_t n_patches() const { return (int64_t)off.size() - 1; }
};
// mode 0: one patch per tet; mode 1: greedy edge stars (largest ring of
// still-unassigned tets around one of the current tet's edges; ties -> the
// most compact tet-index span), tets visited in the given order.
void build_patches(const int32_t *conn4, int64_t n_nodes, int64_t n_elems, int mode, Patches &out);
// Orient every patch so that all of its tets (a, b, r_t, r_t+1) have det > 0
// (swap a and b where all are negative).  Returns false if some patch has a
// tet with det <= 0 left (degenerate / inverted / mixed ring): the kernel
// must then keep the sign-generic arithmetic.  xyz: internal coords (AoS).
bool orient_patches(Patches &p, const double *xyz);

// CTA chunking of the patch sequence for the private scatter.  Each node's
// contributions inside a chunk (one per patch that touches it) are laid out
// "jagged diagonal": nodes ranked by contribution count (descending), level s
// holds the s-th contribution of every node with more than s of them, so the
// node-per-thread reduction reads lane-contiguous addresses.
constexpr int CHUNK_LEVELS = 32;  // max patches per node within one chunk
struct Chunking {
    int max_patches = 0, max_nodes = 0, max_contrib = 0;
    // 5 per chunk: patch_begin, n_patch, node_begin, n_node, n_contrib
    std::vector<int32_t> chunks;
    std::vector<int32_t> gather_nodes;  // per chunk node, local-id order: node id
    std::vector<int32_t> cnodes;        // per chunk node, rank order: node id | bit31 interior
    std::vector<uint8_t> runs;          // per chunk node, rank order: contribution count
    std::vector<uint16_t> levels;       // CHUNK_LEVELS per chunk: jagged level offsets
    std::vector<uint16_t> pids, ppos;   // PATCH_SLOTS per patch: ids {m|closed<<8, a, b, r..}, positions
    // deterministic merge: for nodes in >1 chunk (and isolated nodes), the
    // chunk-node entries (node_begin + rank) holding their partial sums, in chunk order
    std::vector<int32_t> bnd_nodes, bnd_off, bnd_pos;
    int64_t n_shared = 0;
};
// external[v] != 0 marks nodes whose sums other processes complete (e.g. the
// interface planes of a domain decomposition): never "interior" to a chunk,
// so they are always accumulated (REDs / ordered partials), never stored.
bool build_chunks(const Patches &p, int64_t n_nodes, int max_patches, int max_nodes, int max_contrib,
                  const uint8_t *external, Chunking &out, std::string &err);
// Estimated LDS.128 wavefronts of the ring walk's record loads, summed over
// all chunks built so far (quarter-warp groups, before/after bank placement).
void bank_stats(int64_t *groups, int64_t *before, int64_t *after);
// Same for the phase-B contribution stores (half-warp STS.64 groups, before /
// after the bank-aware level and rank choice).
void pos_stats(int64_t *groups, int64_t *before, int64_t *after);
// One contiguous 16-B aligned record per chunk (layout: tal_kernels.cuh,
// patch tables transposed with stride 'cta_threads'); blob_off in 16-B units.
void pack_blobs(const Chunking &ch, int cta_threads, std::vector<uint8_t> &blobs,
                std::vector<int32_t> &blob_off);

}  // namespace tal
