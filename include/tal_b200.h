/*
 * tal_b200.h -- C-ABI of the B200-native P1-tetrahedron momentum-RHS assembly.
 *
 * Drop-in boundary for the reference package tet-assembly-lab 0.1.0
 * (/root/reference/pkg/src/tet_assembly_lab).  The reference has no native
 * code: its hot path is the numba function
 *     _rsp_kernels.assemble_elements(coords, conn, u, rho, mu, cvre, pmat,
 *                                    ids, rhs)            (_rsp_kernels.py:20-21)
 * called by the Python operator
 *     variants.assemble_rsp(mesh, u, params, cfg) -> AssemblyResult
 *                                                        (variants.py:553-616)
 * This header is what that seam binds to instead (ctypes).
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch types.  Host arrays are C-order:
 *    coords (n_nodes,3) f64, conn (n_elems,4) int64, u/rhs (n_nodes,3) f64 --
 *    exactly the reference Mesh / velocity layout (mesh.py:36-47,
 *    kernel.py:194-200).
 *  - Every function returns a status: TAL_OK (0) or a TAL_E* code.  The
 *    message of the last failure on the calling thread is tal_last_error().
 *    TAL_EINVAL maps to Python ValueError (the reference raises ValueError
 *    for bad shapes / non-finite input / bad config), everything else to
 *    RuntimeError.  No C++ exception crosses the ABI.
 *  - A handle owns one CUDA device's copy of one mesh (device-resident,
 *    renumbered, SoA FP64) plus the per-field buffers.  Calls on one handle
 *    must be serialised by the caller; distinct handles are independent.
 *  - There is NO CPU fallback: without a usable sm_100 device every compute
 *    entry point fails with TAL_ECUDA.
 */
#ifndef TAL_B200_H
#define TAL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TAL_ABI_VERSION 1

/* status codes */
#define TAL_OK 0
#define TAL_EINVAL 1 /* bad argument / input          -> ValueError   */
#define TAL_ECUDA 2  /* CUDA failure / no device      -> RuntimeError */
#define TAL_ENOMEM 3 /* host or device allocation     -> MemoryError  */
#define TAL_ESTATE 4 /* call order (e.g. no mesh yet) -> RuntimeError */
#define TAL_EINTERNAL 5 /* unexpected internal failure  -> RuntimeError */
#define TAL_EIO 6       /* file system error            -> OSError      */

/* scatter strategies (the reference RunConfig.scatter, variants.py:74-101,
 * offers 'private' and 'colored'; the GPU adds two atomic forms) */
#define TAL_SCATTER_PRIVATE 0        /* CTA-private smem sums, ordered merge: bitwise reproducible */
#define TAL_SCATTER_COLORED 1        /* colour-by-colour plain read-modify-write: bitwise reproducible */
#define TAL_SCATTER_ATOMIC 2         /* 12 FP64 REDs per element */
#define TAL_SCATTER_PRIVATE_ATOMIC 3 /* CTA-private smem sums, FP64 RED per shared node */
#define TAL_SCATTER_SEQUENTIAL 4     /* reference order: the numba kernel's operation order (no
                                        FMA contraction) summed node by node in ascending element
                                        id -- bitwise identical to the reference's one-thread
                                        assemble_rsp; parity/debug path (4x the arithmetic) */

/* code shapes of the paper's study (variants.py:28-60 VariantId).
 * RSP is the production path (all scatter modes above); B and RS are the
 * baseline and restructured+specialised shapes, one thread per element:
 * scatter 'atomic'/'private-atomic' -> FP64 REDs, 'private'/'colored' ->
 * colour-by-colour plain stores (bitwise reproducible, needs a colouring). */
#define TAL_VARIANT_B 0
#define TAL_VARIANT_RS 1
#define TAL_VARIANT_RSP 2
#define TAL_VARIANT_P 3 /* study only: B with literal trip counts, privatised arrays (PAPER.md "P") */

/* node renumbering applied at upload (inverted on every host read-back) */
#define TAL_RENUMBER_NONE 0
#define TAL_RENUMBER_RCM 1 /* reverse Cuthill-McKee on the node graph */
#define TAL_RENUMBER_SFC 2 /* Morton (Z-order) of node coordinates */

/* element order used to cut CTA chunks */
#define TAL_EORDER_KEEP 0 /* as given */
#define TAL_EORDER_NODE 1 /* by smallest (renumbered) node id */
#define TAL_EORDER_SFC 2  /* Morton order of element centroids */

typedef struct tal_handle tal_handle;

typedef struct {
    double rho;       /* PhysParams.rho       (kernel.py:36)   */
    double mu;        /* PhysParams.mu        (kernel.py:37)   */
    double c_vreman;  /* PhysParams.c_vreman  (kernel.py:38)   */
    double pmat[16];  /* P^T P of the 4-point rule, row-major (variants.py:559) */
} tal_params;

typedef struct {
    int renumber;        /* TAL_RENUMBER_*                              */
    int element_order;   /* TAL_EORDER_*                                */
    int cta_patches;     /* patches per CTA chunk: <= 64 -> 64-thread CTAs, else 128 (max 128) */
    int chunk_nodes;     /* max unique nodes per CTA chunk (<= 144 | 256)  */
    int validate;        /* 1: reject out-of-range ids / non-positive volume */
    int build_colors;    /* 1: colour (greedy, element order) if colors==NULL */
    int patch_mode;      /* 0: one tet per patch; 1: edge-star patches (rings of
                            tets around an edge, e.g. the 6 tets of a Kuhn cell) */
} tal_mesh_opts;

typedef struct {
    int64_t n_nodes, n_elems;
    int64_t n_colors;        /* 0 if no colouring available              */
    int64_t n_patches;       /* thread work units of the private scatter  */
    int64_t n_chunks;        /* CTA chunks of the private scatter        */
    int64_t n_chunk_nodes;   /* sum over chunks of unique nodes          */
    int64_t n_shared_nodes;  /* nodes touched by >1 chunk                */
    int64_t device_bytes;    /* device memory held by the handle         */
    double prep_seconds;     /* host preprocessing time of the upload    */
} tal_mesh_info;

typedef struct {
    /* CUDA-event times in milliseconds of the last tal_assemble call */
    double h2d_ms, pack_ms, kernel_ms, unpack_ms, d2h_ms, total_ms;
    int64_t kernel_launches; /* kernels (of this library) launched by that call */
} tal_timings;

typedef struct {
    /* device pointers in the handle's internal (renumbered) node order */
    double *ux, *uy, *uz; /* velocity components, n_nodes each, stride u_stride doubles */
    double *rx, *ry, *rz; /* assembled RHS components            */
    const int32_t *perm;  /* internal -> caller node id (NULL = identity) */
    const int32_t *iperm; /* caller -> internal node id (NULL = identity) */
    int64_t u_stride;     /* element stride of ux/uy/uz (node records: 6) */
} tal_buffers;

/* ---- library / device ---------------------------------------------------- */
const char *tal_last_error(void);
int tal_abi_version(void);
int tal_device_count(int *count);
/* one tal_handle per (device, mesh) */
int tal_create(int device, tal_handle **out);
int tal_destroy(tal_handle *h);
/* pinned host memory for copy-overlapped end-to-end use */
int tal_host_alloc(int64_t bytes, void **out);
int tal_host_free(void *p);
/* page-lock / release an existing host buffer (cudaHostRegister): the seam
 * and the host round trips then DMA it directly */
int tal_host_register(void *p, int64_t bytes);
int tal_host_unregister(void *p);

/* ---- mesh ------------------------------------------------------------------ */
/* Replaces the per-call coords/conn arguments of assemble_elements
 * (_rsp_kernels.py:20-21) with a one-time upload.  colors may be NULL
 * (mesh.py:43-47: Mesh.colors is optional). */
int tal_upload_mesh(tal_handle *h, const double *coords, const int64_t *conn,
                    int64_t n_nodes, int64_t n_elems, const int64_t *colors,
                    const tal_mesh_opts *opts);
/* As tal_upload_mesh; 'external' (caller ids) are nodes whose sums other
 * ranks complete (interface planes of a domain decomposition): they are never
 * stored as chunk-interior, always accumulated, so a peer may add into them. */
int tal_upload_mesh_ex(tal_handle *h, const double *coords, const int64_t *conn,
                       int64_t n_nodes, int64_t n_elems, const int64_t *colors,
                       const tal_mesh_opts *opts, const int64_t *external,
                       int64_t n_external);
int tal_mesh_info_get(tal_handle *h, tal_mesh_info *out);
/* Host-only dry run of an upload: renumbering, element order, patches and CTA
 * chunks as tal_upload_mesh would build them; fills n_nodes, n_elems,
 * n_patches, n_chunks, n_chunk_nodes, n_shared_nodes, prep_seconds (no
 * device needed -- layout quality checks and planning). */
int tal_plan_layout(const double *coords, const int64_t *conn, int64_t n_nodes,
                    int64_t n_elems, const tal_mesh_opts *opts, tal_mesh_info *out);
int tal_default_mesh_opts(tal_mesh_opts *out);
/* Host-only dump of the private-scatter chunk blobs tal_upload_mesh_ex would
 * build (layout: csrc/tal_kernels.cuh at k_assemble_private), for inspection
 * and CPU-side layout tests.  Call once with NULL buffers to get sizes[0] =
 * blob bytes, [1] = blob_off entries (16-B units, n_chunks+1), [2] = CTA
 * threads (table stride), [3] = perm entries (internal -> caller node id; 0 =
 * identity); then again with buffers of those sizes. */
int tal_plan_blobs(const double *coords, const int64_t *conn, int64_t n_nodes,
                   int64_t n_elems, const tal_mesh_opts *opts, int64_t sizes[4],
                   uint8_t *blobs, int32_t *blob_off, int32_t *perm);
/* Layout diagnostic, summed over every chunking built in this process:
 * out[0] = quarter-warp record-load groups of the ring walk, out[1] / out[2] =
 * estimated shared-memory wavefronts of those loads with ascending-id slots /
 * with the bank-aware placement used; out[3..5] = the same for the half-warp
 * contribution stores (STS.64) before / after the bank-aware level and rank
 * choice.  Ideal = out[0] / out[3].  TAL_BANK_PLACE=0 / TAL_POS_PLACE=0 in the
 * environment disable the two placements. */
int tal_layout_bank_stats(int64_t out[6]);

/* ---- assembly ------------------------------------------------------------- */
/* End-to-end drop-in for assemble_rsp's kernel loop (variants.py:572-615):
 * host u (n_nodes,3) in caller numbering -> host rhs (n_nodes,3), overwritten.
 * Synchronous.  t may be NULL. */
int tal_assemble(tal_handle *h, const double *u, const tal_params *p,
                 double *rhs, int scatter, tal_timings *t);

/* tal_assemble for any code shape (TAL_VARIANT_*): the assemble_baseline /
 * assemble_rs / assemble_rsp entry points (variants.py:522-616). */
int tal_assemble_variant(tal_handle *h, const double *u, const tal_params *p,
                         double *rhs, int variant, int scatter, tal_timings *t);

/* Pipelined host round trip for streams of fields (time loops with host-side
 * I/O, ensembles): enqueues H2D(u) -> assembly -> D2H(rhs) on internal
 * streams and returns; at most three calls are in flight (a fourth call first
 * waits for the oldest), so the H2D of field n+1 and the D2H of result n-1
 * overlap the assembly of field n and each other.  u and rhs must stay untouched until
 * tal_wait(ticket) (pinned host memory, tal_host_alloc, gives full overlap). */
int tal_assemble_async(tal_handle *h, const double *u, const tal_params *p,
                       double *rhs, int scatter, int64_t *ticket);
int tal_wait(tal_handle *h, int64_t ticket);

/* Device-resident path (no host copies).  'stream' is a cudaStream_t (or 0).
 * tal_set_velocity_*: caller-numbered AoS (n_nodes,3) -> internal SoA.
 * tal_run: assemble internal u -> internal rhs (overwrites).  Asynchronous.
 * tal_get_rhs_*: internal SoA -> caller-numbered AoS (n_nodes,3). */
int tal_buffers_get(tal_handle *h, tal_buffers *out);
int tal_set_velocity_host(tal_handle *h, const double *u, void *stream);
int tal_set_velocity_device(tal_handle *h, const double *d_u, void *stream);
int tal_run(tal_handle *h, const tal_params *p, int scatter, void *stream,
            int64_t *kernel_launches);
/* Optional P1 pressure-gradient term r_a += int p dN_a/dx_i (SURVEY.md section
 * 8 f4; NOT part of the reference operator, kernel.py:7-10 -- its parity is
 * pinned by this repo's own oracle only).  p: (n_nodes,) f64 in caller
 * numbering, host or device; NULL switches the term off again.  Applies to
 * every later assembly of the RSP shape on this handle (B/RS: TAL_EINVAL). */
int tal_set_pressure_host(tal_handle *h, const double *p, void *stream);
int tal_set_pressure_device(tal_handle *h, const double *d_p, void *stream);

/* tal_run for any code shape (TAL_VARIANT_*) */
int tal_run_variant(tal_handle *h, const tal_params *p, int variant, int scatter,
                    void *stream, int64_t *kernel_launches);
/* CUDA graph of one assembly step (zeroing + kernels + merge) on the
 * internal buffers, captured with the current parameters, variant, scatter
 * and pressure setting; replay with tal_graph_launch on any stream.
 * Re-capture after changing any of
 * them (also after attaching peers); the mesh upload destroys the graph.  With
 * peers attached the graph holds the whole fused step (flag epochs live on the
 * device). */
int tal_graph_capture(tal_handle *h, const tal_params *p, int variant, int scatter);
int tal_graph_launch(tal_handle *h, void *stream, int64_t *kernel_launches);
int tal_graph_destroy(tal_handle *h);
/* Optional SUPG stabilisation of the convective residual (extension, no
 * reference counterpart; tal_element.cuh supg_add): every later RSP-shape
 * assembly on this handle adds
 *   r_a[i] -= int tau (rho u.grad N_a)(rho u.grad u_i),
 *   tau = 1 / (c1 (mu + rho nu_t) / h^2 + c2 rho |u_mean| / h), h = cbrt(6 vol).
 * enable = 0 switches it off.  Needs the symmetric Gauss table; not with
 * scatter 'sequential', the B/RS shapes or the fused multi-GPU path
 * (TAL_EINVAL).  A captured graph (tal_graph_capture) is dropped. */
int tal_set_stabilization(tal_handle *h, int enable, double c1, double c2);
/* One assembly straight from and to the caller's device arrays d_u, d_rhs
 * ((N,3) AoS doubles in the caller's node numbering), no internal layout
 * conversion: the private kernel gathers u from d_u and writes the sums to
 * d_rhs (scatter 'private' / 'private-atomic', symmetric rule, no pressure /
 * SUPG / peers); otherwise the composition set_velocity_device -> run ->
 * get_rhs_device.  Asynchronous on 'stream'. */
int tal_run_caller(tal_handle *h, const tal_params *p, int scatter, const double *d_u, double *d_rhs,
                   void *stream, int64_t *kernel_launches);
/* tal_get_rhs_host blocks until rhs (caller order, (N,3) AoS) is complete. */
int tal_get_rhs_host(tal_handle *h, double *rhs, void *stream);
int tal_get_rhs_device(tal_handle *h, double *d_rhs, void *stream);
int tal_synchronize(tal_handle *h, void *stream);

/* Element-subset seam, signature-for-signature the numba kernel
 * _rsp_kernels.assemble_elements (_rsp_kernels.py:20-21): assembles elements
 * ids[0..k) and ADDS (+=) into the host rhs, as the numba loop does.  The
 * mesh stays resident between calls in a small internal cache keyed by the
 * arrays' addresses and sizes; every call re-checks 64-KB block fingerprints
 * of the parts it reads (its conn rows, the coords rows they reference), so
 * a changed array is re-uploaded, never served stale.  ids = the whole mesh
 * runs the edge-star kernel, any other subset the per-element kernel; a
 * contiguous range moves only the node rows its elements reference across
 * PCIe (the reference's threaded slabs, variants.py:578-596). */
int tal_assemble_elements(int device, const double *coords, const int64_t *conn,
                          int64_t n_nodes, int64_t n_elems, const double *u,
                          double rho, double mu, double cvre,
                          const double *pmat, const int64_t *ids, int64_t k,
                          double *rhs);
/* Same signature and semantics, bitwise identical to the numba loop: every
 * node continues from its incoming rhs value through its elements in ids
 * order, element arithmetic in the reference's operation order without FMA
 * contraction (tal_strict.cuh).  Dropped into the reference's own driver
 * (variants.py:573-596, any thread count), it reproduces assemble_rsp bit for
 * bit. */
int tal_assemble_elements_strict(int device, const double *coords, const int64_t *conn,
                                 int64_t n_nodes, int64_t n_elems, const double *u,
                                 double rho, double mu, double cvre,
                                 const double *pmat, const int64_t *ids, int64_t k,
                                 double *rhs);

/* The same seam with an explicit per-mesh context (no per-call fingerprint
 * check: the caller keeps coords / conn unchanged while the context is open):
 * open once per (coords, conn), call tal_seam_assemble with the numba
 * kernel's remaining arguments, close.  Thread-safe: id checks run
 * concurrently, the GPU part of the calls is serialised; u and rhs are
 * caller-order (N,3) host arrays, rhs += result. */
typedef struct tal_seam tal_seam;
int tal_seam_open(int device, const double *coords, const int64_t *conn, int64_t n_nodes,
                  int64_t n_elems, tal_seam **out);
int tal_seam_assemble(tal_seam *ctx, const double *u, double rho, double mu, double cvre,
                      const double *pmat, const int64_t *ids, int64_t k, double *rhs);
int tal_seam_close(tal_seam *ctx);

/* ---- mesh IO and partitioning (host only) ------------ */
/* The reference's text format (mesh.py:280-371): tal_mesh_save_text writes
 * it byte for byte like save_mesh; tal_mesh_load_text parses it like
 * load_mesh (comments, blank lines, inverted elements re-oriented and
 * counted).  A format error returns TAL_EINVAL with "line N: ..." and
 * tal_last_error_line() = N (the reference's MeshFormatError.line). */
typedef struct tal_meshbuf tal_meshbuf;
int64_t tal_last_error_line(void);
int tal_mesh_load_text(const char *path, tal_meshbuf **out);
int tal_meshbuf_info(tal_meshbuf *b, int64_t *n_nodes, int64_t *n_elems, int64_t *n_reoriented);
int tal_meshbuf_copy(tal_meshbuf *b, double *coords, int64_t *conn);
int tal_meshbuf_free(tal_meshbuf *b);
int tal_mesh_save_text(const char *path, const double *coords, const int64_t *conn,
                       int64_t n_nodes, int64_t n_elems);
/* Binary "TALMESH1": 64-byte header (magic, version, sizes, content hash),
 * coords f64 (N,3), conn i64 (E,4); exact round trip, hash verified. */
int tal_mesh_save_binary(const char *path, const double *coords, const int64_t *conn,
                         int64_t n_nodes, int64_t n_elems);
int tal_mesh_probe_binary(const char *path, int64_t *n_nodes, int64_t *n_elems, int *is_binary);
int tal_mesh_load_binary(const char *path, double *coords, int64_t n_nodes, int64_t *conn,
                         int64_t n_elems);
/* Recursive coordinate bisection of n points (n,3) into 'world' parts. */
int tal_rcb_parts(const double *points, int64_t n, int world, int32_t *parts);

/* ---- multi-GPU interface (domain decomposition) ----------------------------- */
/* Gather rhs of internal node ids list[0..n) into a packed buffer d_out
 * (n*3 doubles, component-interleaved) / add a packed buffer into rhs. */
int tal_halo_pack(tal_handle *h, const int32_t *d_list, int64_t n, double *d_out, void *stream);
int tal_halo_accumulate(tal_handle *h, const int32_t *d_list, int64_t n, const double *d_in, void *stream);
/* caller node id -> internal node id (host arrays) */
int tal_map_nodes(tal_handle *h, const int64_t *caller_ids, int64_t n, int32_t *internal_ids);

/* ---- fused interface sum over peer memory (domain decomposition) ---------- */
/* With up to two neighbours attached, tal_run(scatter=private-atomic) REDs the
 * partial sums of the attached interface nodes into the local RHS AND directly
 * into the neighbour's RHS (NVLink peer memory), ordered across ranks by
 * device-side flag words: zero -> signal/wait -> assemble -> signal/wait.
 * The neighbour's RHS must be sized/renumbered as that neighbour's handle
 * says: pass its INTERNAL ids (tal_map_nodes on the neighbour) for my caller
 * ids my_ids[0..n).  In-process neighbours: tal_peer_local + tal_peer_attach;
 * other processes: tal_peer_export (64-B cudaIpcMemHandle_t each) + tal_peer_open. */
int tal_peer_local(tal_handle *h, double **rx, unsigned long long **flags, int64_t *n_nodes);
int tal_peer_export(tal_handle *h, void *rhs_handle, int64_t *rhs_offset, void *flags_handle);
int tal_peer_attach(tal_handle *h, int slot, double *peer_rx, int64_t peer_n_nodes,
                    unsigned long long *peer_flags, const int64_t *my_ids,
                    const int32_t *peer_ids, int64_t n);
int tal_peer_open(tal_handle *h, int slot, const void *rhs_handle, int64_t rhs_offset,
                  const void *flags_handle, int64_t peer_n_nodes, const int64_t *my_ids,
                  const int32_t *peer_ids, int64_t n);
int tal_peer_detach(tal_handle *h);

/* ---- host-side mesh utilities (native; used by the Python Mesh type) ------- */
/* Kuhn 6-tet split of a box (mesh.py:145-184). coords (N,3), conn (E,4). */
int tal_box_mesh(int64_t nx, int64_t ny, int64_t nz, double ex, double ey,
                 double ez, double *coords, int64_t *conn);
/* signed volumes det/6 (mesh.py:110-123); min_out may be NULL */
int tal_signed_volumes(const double *coords, const int64_t *conn, int64_t n_elems,
                       double *vols);
/* greedy lowest-free colouring in element order (mesh.py:235-257) */
int tal_color_elements(const int64_t *conn, int64_t n_nodes, int64_t n_elems,
                       int64_t *colors, int64_t *n_colors);
/* 1 if no two elements sharing a node share a colour (mesh.py:260-267) */
int tal_check_coloring(const int64_t *conn, const int64_t *colors, int64_t n_nodes,
                       int64_t n_elems, int *valid);
/* node permutation perm[new] = old by the given TAL_RENUMBER_* */
int tal_renumber_nodes(const double *coords, const int64_t *conn, int64_t n_nodes,
                       int64_t n_elems, int method, int64_t *perm);

/* edge-star patch decomposition used by the private scatter (host utility,
 * for inspection/tests).  Two-call protocol: with nodes_out == NULL only the
 * sizes are returned.  Patch g = off[g]..off[g+1] into nodes: a, b, r_0..r_m-1;
 * its tets are (a, b, r_i, r_i+1), i < m (closed[g]) or i < m-1 (open). */
int tal_build_patches(const int64_t *conn, int64_t n_nodes, int64_t n_elems, int mode,
                      int64_t *n_patches, int64_t *n_patch_nodes, int32_t *off_out,
                      int32_t *nodes_out, uint8_t *closed_out);

/* ---- measurement ------------------------------------------------------------ */
/* When enabled, tal_run records a CUDA event pair around the dominant
 * assembly kernel of every call (on the launching stream, inside the real
 * step).  tal_profile_read waits for and returns the per-call durations (ms)
 * recorded since the last read, oldest first (at most 'cap', ring of 4096). */
int tal_profile(tal_handle *h, int enable);
int tal_profile_read(tal_handle *h, double *ms_out, int64_t cap, int64_t *n_out);
/* Sustained FP64 FMA throughput of 'device' (TFLOP/s, 2 flop per DFMA),
 * timed with CUDA events over 'ms_target' milliseconds of work. */
int tal_fp64_peak(int device, double ms_target, double *tflops, double *sm_clock_mhz);

#ifdef __cplusplus
}
#endif
#endif /* TAL_B200_H */
