// tal_capi.cu -- the C-ABI (include/tal_b200.h) over the sm_100a kernels.
//
// Replaces the reference seam _rsp_kernels.assemble_elements
// (_rsp_kernels.py:20-21) and the kernel loop of variants.assemble_rsp
// (variants.py:572-615).  See DESIGN.md for the data layout.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/tal_b200.h"
#include "tal_kernels.cuh"
#include "tal_strict.cuh"
#include <mutex>
#include <memory>
#include <atomic>
#include "tal_prep.hpp"
#include "tal_meshio.hpp"
#include "tal_par.hpp"
#include "tal_shapes.cuh"

using namespace tal;

static_assert(SLOTS == PATCH_SLOTS && BLOB_LEVELS == CHUNK_LEVELS, "blob layout mismatch host/device");

namespace {

thread_local std::string g_err;
thread_local int64_t g_err_line = 0;

int fail(int code, const std::string &msg)
{
    g_err = msg;
    g_err_line = 0;
    return code;
}

#define TAL_CK(call)                                                                        \
    do {                                                                                    \
        cudaError_t _e = (call);                                                            \
        if (_e != cudaSuccess)                                                              \
            return fail(TAL_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e));     \
    } while (0)

#define TAL_CK_LAUNCH()                                                                     \
    do {                                                                                    \
        cudaError_t _e = cudaGetLastError();                                                \
        if (_e != cudaSuccess)                                                              \
            return fail(TAL_ECUDA, std::string("kernel launch: ") + cudaGetErrorString(_e)); \
    } while (0)

template <class T>
int dev_upload(T **dst, const T *src, size_t count)
{
    *dst = nullptr;
    if (count == 0)
        return TAL_OK;
    TAL_CK(cudaMalloc((void **)dst, count * sizeof(T)));
    TAL_CK(cudaMemcpy(*dst, src, count * sizeof(T), cudaMemcpyHostToDevice));
    return TAL_OK;
}

unsigned grid_for(int64_t n, int threads) { return (unsigned)((n + threads - 1) / threads); }

}  // namespace

struct tal_handle {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev[6] = {};
    // pipelined host round trip (tal_assemble_async): ASYNC_SLOTS fields in
    // flight on two copy streams.  Three slots let the H2D of field n+1, the
    // assembly of n and the D2H of n-1 run concurrently: the period is then
    // max(h2d, d2h) instead of (h2d + compute + d2h) / 2 with two slots.
#ifndef TAL_ASYNC_SLOTS
#define TAL_ASYNC_SLOTS 3
#endif
    static constexpr int ASYNC_SLOTS = TAL_ASYNC_SLOTS;
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_h2d[ASYNC_SLOTS] = {}, ev_comp[ASYNC_SLOTS] = {}, ev_d2h[ASYNC_SLOTS] = {};
    double *astage_u[ASYNC_SLOTS] = {}, *astage_r[ASYNC_SLOTS] = {};
    int64_t async_next = 0;  // next ticket
    int64_t N = 0, E = 0;
    int64_t n_interior = 0;  // internal ids [0, n_interior) are chunk-interior (HostLayout)
    bool has_mesh = false;
    // node data (internal order): records x y z ux uy uz (6*N) then rx ry rz (3*N)
    double *nodebuf = nullptr;
    double *staging = nullptr;  // 3*N doubles (AoS in/out)
    int32_t *perm = nullptr, *iperm = nullptr;
    std::vector<int32_t> h_iperm;  // caller -> internal (host)
    int4 *conn = nullptr;          // element order of the chunking
    std::vector<int32_t> h_eperm;  // conn row -> caller element id (empty: identity)
    // reference-order scatter (built on first use): node -> incident conn rows
    int64_t *d_seq_off = nullptr;  // N+1
    int32_t *d_seq_ent = nullptr;  // 4E: row << 2 | corner, ascending caller element id
    double *d_seq_dlt = nullptr;   // E: Vreman filter width cbrt(6 vol) per conn row (host libm)
    double *d_seq_rows = nullptr;  // 12 E: strict element rows (two-pass sequential scatter)
    // colouring
    int4 *conn_col = nullptr;
    std::vector<int64_t> col_off;
    // private scatter
    Chunking ch;
    uint8_t *d_blobs = nullptr;
    int32_t *d_blob_off = nullptr;
    int32_t *d_bnd_nodes = nullptr, *d_bnd_off = nullptr, *d_bnd_pos = nullptr;
    // tal_run_caller: chunk blobs with caller node ids, caller-order coordinates
    uint8_t *d_blobs_cl = nullptr;
    double *d_xc = nullptr;
    int64_t blob_bytes = 0;
    double *d_partial = nullptr;  // 3 * n_chunk_nodes
    int priv_cfg = 1;
    int priv_grid_ext[4] = {0, 0, 0, 0};  // persistent grid per (pressure, SUPG) instance
    bool has_st = false;                  // SUPG stabilisation (tal_set_stabilization)
    double st_c1 = 4.0, st_c2 = 2.0;
    // optional nodal pressure (internal order) for the pressure-gradient term
    double *d_press = nullptr;
    bool has_press = false;
    // fused interface sum with up to two neighbours (domain decomposition)
    struct Peer {
        double *rx = nullptr;              // neighbour's RHS x (y, z follow at +n, +2n)
        int64_t n = 0;                     // neighbour's node count
        unsigned long long *flags = nullptr;  // neighbour's flag words
        void *ipc_rhs = nullptr, *ipc_flags = nullptr;  // IPC mappings to close
    } peers[2];
    unsigned long long *d_flags = nullptr;  // own flag words (8): [0] zeroed, [1] done
    int32_t *d_pidx = nullptr;              // per chunk-node entry: slot<<30 | remote id
    std::vector<int32_t> h_pidx;
    std::vector<uint8_t> external;  // internal-id mask of nodes completed by peers
    tal_mesh_info info = {};
    tal_timings last = {};
    // dominant-kernel event ring (tal_profile)
    static constexpr int PROF_RING = 4096;
    bool prof_on = false;
    std::vector<cudaEvent_t> prof_ev;  // 2 per slot
    // one captured assembly step (tal_graph_capture / tal_graph_launch)
    cudaGraphExec_t gexec = nullptr;
    int64_t g_launches = 0;
    void free_graph()
    {
        if (gexec)
            cudaGraphExecDestroy(gexec);
        gexec = nullptr;
        g_launches = 0;
    }
    int64_t prof_head = 0, prof_count = 0;

    double *REC() const { return nodebuf; }
    double *RX() const { return nodebuf + 6 * N; }
    double *RY() const { return nodebuf + 7 * N; }
    double *RZ() const { return nodebuf + 8 * N; }

    int n_peers() const { return (peers[0].rx ? 1 : 0) + (peers[1].rx ? 1 : 0); }

    void free_peers()
    {
        free_graph();  // a captured step may hold the peer launches
        for (auto &p : peers) {
            if (p.ipc_rhs)
                cudaIpcCloseMemHandle(p.ipc_rhs);
            if (p.ipc_flags)
                cudaIpcCloseMemHandle(p.ipc_flags);
            p = Peer();
        }
        if (d_pidx)
            cudaFree(d_pidx);
        d_pidx = nullptr;
        h_pidx.clear();
        if (d_flags)
            cudaMemset(d_flags, 0, 8 * sizeof(unsigned long long));
    }

    void free_mesh()
    {
        free_graph();
        free_peers();
        void *ptrs[] = {nodebuf, staging, perm, iperm, conn, conn_col, d_blobs, d_blob_off,
                        d_bnd_nodes, d_bnd_off, d_bnd_pos, d_partial, d_press, d_seq_off, d_seq_ent, d_seq_dlt, d_seq_rows,
                        d_blobs_cl, d_xc};
        for (void *p : ptrs)
            if (p)
                cudaFree(p);
        nodebuf = staging = d_partial = d_press = nullptr;
        d_seq_off = nullptr;
        d_seq_ent = nullptr;
        d_seq_dlt = nullptr;
        d_seq_rows = nullptr;
        h_eperm.clear();
        has_press = false;
        for (int s = 0; s < ASYNC_SLOTS; ++s) {
            if (astage_u[s])
                cudaFree(astage_u[s]);
            if (astage_r[s])
                cudaFree(astage_r[s]);
            astage_u[s] = astage_r[s] = nullptr;
        }
        async_next = 0;
        perm = iperm = d_blob_off = d_bnd_nodes = d_bnd_off = d_bnd_pos = nullptr;
        d_blobs_cl = nullptr;
        d_xc = nullptr;
        blob_bytes = 0;
        conn = conn_col = nullptr;
        d_blobs = nullptr;
        col_off.clear();
        h_iperm.clear();
        ch = Chunking();
        n_interior = 0;
        std::fill(priv_grid_ext, priv_grid_ext + 4, 0);
        has_mesh = false;
        info = tal_mesh_info{};
    }
};

namespace {

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev)
    {
        cudaGetDevice(&prev);
        cudaSetDevice(dev);
    }
    ~DeviceGuard()
    {
        if (prev >= 0)
            cudaSetDevice(prev);
    }
};

// RHS zeroing before RED accumulation (cudaMemsetAsync: a streaming-store
// zero kernel measured 1.8 us slower per step)
cudaError_t zero_rhs(tal_handle *h, cudaStream_t s, bool tail_only = false)
{
    const int64_t n = 3 * h->N;
    if (!n)
        return cudaSuccess;
    if (tail_only && h->n_interior > 0) {  // interior nodes are plain-stored by their chunk
        const int64_t t = h->N - h->n_interior;
        cudaError_t e = cudaSuccess;
        // the three component tails as one 2-D memset (rows N doubles apart):
        // one graph node instead of three, step 0.2720 -> 0.2696 ms at 128^3
        if (t > 0)
            e = cudaMemset2DAsync(h->RX() + h->n_interior, sizeof(double) * h->N, 0, sizeof(double) * t, 3, s);
        return e;
    }
    return cudaMemsetAsync(h->RX(), 0, sizeof(double) * n, s);
}

bool make_consts(const tal_params *p, ElemConsts &kc, bool &sym)
{
    kc.rho = p->rho;
    kc.mu = p->mu;
    kc.cvre = p->c_vreman;
    kc.rc = p->rho * p->c_vreman;
    for (int i = 0; i < 16; ++i)
        kc.pm[i] = p->pmat[i];
    double pd = 0.0, po = 0.0;
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b)
            (a == b ? pd : po) += p->pmat[4 * a + b];
    pd /= 4.0;
    po /= 12.0;
    sym = true;
    for (int a = 0; a < 4; ++a)
        for (int b = 0; b < 4; ++b) {
            const double ref = (a == b) ? pd : po;
            if (std::fabs(p->pmat[4 * a + b] - ref) > 1e-14 * std::max(std::fabs(ref), 1e-300))
                sym = false;
        }
    kc.a_po = -p->rho * po / 24.0;
    kc.a_q = -p->rho * (pd - po) / 24.0;
    kc.a_4 = 4.0 * kc.a_po + kc.a_q;
    kc.rc6 = -kc.rc / 6.0;
    kc.mu6 = -p->mu / 6.0;
    kc.st_po = po;
    kc.st_dq = pd - po;
    kc.st_c1 = 4.0;
    kc.st_c2 = 2.0;
    return std::isfinite(p->rho) && std::isfinite(p->mu) && std::isfinite(p->c_vreman);
}

int check_params(const tal_params *p)
{
    if (!p)
        return fail(TAL_EINVAL, "params is NULL");
    // PhysParams.__post_init__ (kernel.py:41-49)
    if (!(p->rho > 0.0))
        return fail(TAL_EINVAL, "rho must be positive, got " + std::to_string(p->rho));
    if (p->mu < 0.0)
        return fail(TAL_EINVAL, "mu must be non-negative, got " + std::to_string(p->mu));
    if (p->c_vreman < 0.0)
        return fail(TAL_EINVAL, "c_vreman must be non-negative, got " + std::to_string(p->c_vreman));
    for (int i = 0; i < 16; ++i)
        if (!std::isfinite(p->pmat[i]))
            return fail(TAL_EINVAL, "pmat contains non-finite entries");
    return TAL_OK;
}

template <int CFG, bool ORDERED>
const void *private_fn(bool peer, bool pr, bool st, bool cl = false)
{
    if (cl)  // caller layout: the plain step only (no peers, pressure, SUPG)
        return (const void *)k_assemble_private<CFG, ORDERED, false, false, false, true>;
    if (peer)  // the fused multi-GPU path: no SUPG instance (host-checked)
        return pr ? (const void *)k_assemble_private<CFG, ORDERED, true, true>
                  : (const void *)k_assemble_private<CFG, ORDERED, true>;
    return st ? (pr ? (const void *)k_assemble_private<CFG, ORDERED, false, true, true>
                    : (const void *)k_assemble_private<CFG, ORDERED, false, false, true>)
              : (pr ? (const void *)k_assemble_private<CFG, ORDERED, false, true>
                    : (const void *)k_assemble_private<CFG, ORDERED>);
}

template <int CFG>
cudaError_t launch_private_cfg(bool ordered, bool st, unsigned grid, cudaStream_t s, PrivArgs pa,
                               const double *nodes, RhsSoA rhs, ElemConsts kc, PeerArgs peer)
{
    const bool pr = pa.press != nullptr;
    const bool cl = pa.rhs_caller != nullptr;
    const size_t sm = pr ? PrivLayoutOf<CFG, true>::TOTAL : PrivLayoutOf<CFG>::TOTAL;
    constexpr int T = PrivCfg<CFG>::THREADS;
    void *args[] = {(void *)&pa, (void *)&nodes, (void *)&rhs, (void *)&kc, (void *)&peer};
    const bool peer_on = peer.pidx != nullptr && !ordered;
    const void *fn =
        ordered ? private_fn<CFG, true>(false, pr, st, cl) : private_fn<CFG, false>(peer_on, pr, st, cl);
    // plain launch of a persistent grid (occupancy x SMs); no grid-wide barrier
    // is used, so CTAs that cannot be resident yet simply start later
    return cudaLaunchKernel(fn, dim3(grid), dim3(T), args, sm, s);
}

cudaError_t launch_private(int cfg, bool ordered, bool st, unsigned grid, cudaStream_t s, const PrivArgs &pa,
                           const double *nodes, RhsSoA rhs, const ElemConsts &kc, const PeerArgs &peer)
{
    return cfg == 0   ? launch_private_cfg<0>(ordered, st, grid, s, pa, nodes, rhs, kc, peer)
           : cfg == 1 ? launch_private_cfg<1>(ordered, st, grid, s, pa, nodes, rhs, kc, peer)
                      : launch_private_cfg<2>(ordered, st, grid, s, pa, nodes, rhs, kc, peer);
}

struct ProfMark {
    tal_handle *h;
    cudaStream_t s;
    int64_t slot = -1;
    void begin()
    {
        if (!h->prof_on)
            return;
        slot = (h->prof_head + h->prof_count) % tal_handle::PROF_RING;
        if (h->prof_count == tal_handle::PROF_RING)  // overwrite the oldest
            h->prof_head = (h->prof_head + 1) % tal_handle::PROF_RING;
        else
            ++h->prof_count;
        cudaEventRecord(h->prof_ev[2 * slot], s);
    }
    void end()
    {
        if (slot >= 0)
            cudaEventRecord(h->prof_ev[2 * slot + 1], s);
    }
};

// Vreman filter width delta = cbrt(6 vol) of one element as the reference
// computes it (_rsp_kernels.py:45-62: edges, cofactor row 1, det, vol, numba's
// np.cbrt = libm pow(x, 1/3)); host code, baseline x86-64 (no FMA contraction
// possible).  xyz: node coordinates with 'stride' doubles per node.
template <class Id>
double filter_width(const double *xyz, int stride, const Id *nodes4)
{
    const double *x0 = xyz + stride * (int64_t)nodes4[0];
    double ed[4][3];
    for (int b = 1; b < 4; ++b)
        for (int c = 0; c < 3; ++c)
            ed[b][c] = xyz[stride * (int64_t)nodes4[b] + c] - x0[c];
    const double c0 = ed[2][1] * ed[3][2] - ed[2][2] * ed[3][1];
    const double c1 = ed[2][2] * ed[3][0] - ed[2][0] * ed[3][2];
    const double c2 = ed[2][0] * ed[3][1] - ed[2][1] * ed[3][0];
    const double det = ed[1][0] * c0 + ed[1][1] * c1 + ed[1][2] * c2;
    const double x = 6.0 * (std::fabs(det) / 6.0);
    return std::isnan(x) ? x : std::pow(x, 1.0 / 3.0);  // x >= 0: the sign-symmetric branch is moot
}

// two-pass reference-order scatter (rows once, then ordered sums); the
// single-pass form evaluates every element once per node.  TAL_SEQ_TWO_PASS=0
// selects the single pass.
bool seq_two_pass()
{
    static const bool on = [] {
        const char *e = std::getenv("TAL_SEQ_TWO_PASS");
        return !e || std::atoi(e) != 0;
    }();
    return on;
}

// node -> (conn row, corner) lists in ascending caller element id, for the
// reference-order scatter; built on the host from the device connectivity
int build_sequential(tal_handle *h)
{
    const int64_t N = h->N, E = h->E;
    if (4 * E > INT32_MAX)
        return fail(TAL_EINVAL, "scatter 'sequential' supports up to 2^29 elements");
    std::vector<int32_t> cord((size_t)(4 * E));
    if (E)
        TAL_CK(cudaMemcpy(cord.data(), h->conn, sizeof(int32_t) * 4 * E, cudaMemcpyDeviceToHost));
    std::vector<int32_t> row((size_t)E);  // caller element id -> conn row
    for (int64_t e = 0; e < E; ++e)
        row[h->h_eperm.empty() ? e : h->h_eperm[e]] = (int32_t)e;
    std::vector<int64_t> off((size_t)N + 1, 0);
    for (int64_t i = 0; i < 4 * E; ++i)
        off[cord[i] + 1]++;
    for (int64_t v = 0; v < N; ++v)
        off[v + 1] += off[v];
    std::vector<int64_t> fill(off.begin(), off.end() - 1);
    std::vector<int32_t> ent((size_t)(4 * E));
    for (int64_t eo = 0; eo < E; ++eo) {
        const int32_t r = row[eo];
        for (int a = 0; a < 4; ++a)
            ent[fill[cord[4 * (int64_t)r + a]]++] = r << 2 | a;
    }
    // filter width per element, _rsp_kernels.py:45-62 in the reference's
    // operation order (baseline x86-64 code: no FMA contraction possible) and
    // the reference's libm pow -- see tal_strict.cuh for why on the host
    std::vector<double> rec((size_t)(6 * N));
    if (N)
        TAL_CK(cudaMemcpy(rec.data(), h->REC(), sizeof(double) * 6 * N, cudaMemcpyDeviceToHost));
    std::vector<double> dlt((size_t)E);
    for (int64_t e = 0; e < E; ++e)
        dlt[e] = filter_width(rec.data(), 6, &cord[4 * e]);
    if (int rc = dev_upload(&h->d_seq_off, off.data(), off.size()))
        return rc;
    if (!E)
        return TAL_OK;
    if (int rc = dev_upload(&h->d_seq_dlt, dlt.data(), dlt.size()))
        return rc;
    if (seq_two_pass() && cudaMalloc((void **)&h->d_seq_rows, sizeof(double) * 12 * (size_t)E) != cudaSuccess) {
        cudaGetLastError();  // not enough memory for the row buffer: single-pass form
        h->d_seq_rows = nullptr;
    }
    return dev_upload(&h->d_seq_ent, ent.data(), ent.size());
}

int launch_run(tal_handle *h, const tal_params *p, int scatter, cudaStream_t s, int64_t *launches)
{
    ProfMark pm{h, s};
    ElemConsts kc;
    bool sym;
    if (!make_consts(p, kc, sym))
        return fail(TAL_EINVAL, "non-finite physical parameters");
    const double *nodes = h->REC();
    RhsSoA rhs{h->RX(), h->RY(), h->RZ()};
    int64_t nl = 0;
    const int64_t N = h->N, E = h->E;
    const bool st = h->has_st;
    if (st) {
        if (!sym)
            return fail(TAL_EINVAL, "the SUPG stabilisation needs the symmetric Gauss table (pmat = P^T P)");
        if (h->n_peers())
            return fail(TAL_EINVAL, "the SUPG stabilisation is not available on the fused multi-GPU path");
        kc.st_c1 = h->st_c1;
        kc.st_c2 = h->st_c2;
    }
    // the fused interface sum lives in the private-atomic kernel's phase C
    // (and its signal/wait kernels): any other path would drop this rank's
    // interface sums and leave the neighbours waiting
    if (h->n_peers() && (scatter != TAL_SCATTER_PRIVATE_ATOMIC || !sym))
        return fail(TAL_EINVAL, "peers are attached: only scatter='private-atomic' with the symmetric "
                                "Gauss table performs the fused interface sum");
    switch (scatter) {
    case TAL_SCATTER_ATOMIC: {
        if (N) {
            TAL_CK(zero_rhs(h, s));
        }
        if (E) {
            pm.begin();
            const double *pr = h->has_press ? h->d_press : nullptr;
            const unsigned g = grid_for(E, 256);
            if (sym && st)
                pr ? k_assemble_atomic<true, true, true><<<g, 256, 0, s>>>(h->conn, 0, E, nodes, rhs, kc, pr)
                   : k_assemble_atomic<true, false, true><<<g, 256, 0, s>>>(h->conn, 0, E, nodes, rhs, kc, nullptr);
            else if (sym)
                pr ? k_assemble_atomic<true, true><<<g, 256, 0, s>>>(h->conn, 0, E, nodes, rhs, kc, pr)
                   : k_assemble_atomic<true><<<g, 256, 0, s>>>(h->conn, 0, E, nodes, rhs, kc, nullptr);
            else
                pr ? k_assemble_atomic<false, true><<<g, 256, 0, s>>>(h->conn, 0, E, nodes, rhs, kc, pr)
                   : k_assemble_atomic<false><<<g, 256, 0, s>>>(h->conn, 0, E, nodes, rhs, kc, nullptr);
            pm.end();
            TAL_CK_LAUNCH();
            ++nl;
        }
        break;
    }
    case TAL_SCATTER_COLORED: {
        if (!h->conn_col && E)
            return fail(TAL_ESTATE, "mesh was uploaded without a colouring (build_colors=0, colors=NULL)");
        if (N) {
            TAL_CK(zero_rhs(h, s));
        }
        pm.begin();  // colour launches together form the dominant work
        for (size_t c = 0; c + 1 < h->col_off.size(); ++c) {
            const int64_t b = h->col_off[c], e = h->col_off[c + 1];
            if (e <= b)
                continue;
            const double *pr = h->has_press ? h->d_press : nullptr;
            const unsigned g = grid_for(e - b, 256);
            if (sym && st)
                pr ? k_assemble_colored<true, true, true><<<g, 256, 0, s>>>(h->conn_col, b, e, nodes, rhs, kc, pr)
                   : k_assemble_colored<true, false, true><<<g, 256, 0, s>>>(h->conn_col, b, e, nodes, rhs, kc,
                                                                             nullptr);
            else if (sym)
                pr ? k_assemble_colored<true, true><<<g, 256, 0, s>>>(h->conn_col, b, e, nodes, rhs, kc, pr)
                   : k_assemble_colored<true><<<g, 256, 0, s>>>(h->conn_col, b, e, nodes, rhs, kc, nullptr);
            else
                pr ? k_assemble_colored<false, true><<<g, 256, 0, s>>>(h->conn_col, b, e, nodes, rhs, kc, pr)
                   : k_assemble_colored<false><<<g, 256, 0, s>>>(h->conn_col, b, e, nodes, rhs, kc, nullptr);
            TAL_CK_LAUNCH();
            ++nl;
        }
        pm.end();
        break;
    }
    case TAL_SCATTER_PRIVATE:
    case TAL_SCATTER_PRIVATE_ATOMIC: {
        // patches permute tet corners: only valid for the symmetric rule.  A
        // general table runs the per-element atomic kernel -- for
        // 'private-atomic' (already order-free) only: 'private' promises a
        // bitwise reproducible sum, which the atomic kernel cannot keep
        if (!sym && scatter == TAL_SCATTER_PRIVATE)
            return fail(TAL_EINVAL, "scatter='private' needs the symmetric Gauss table (pmat = P^T P of "
                                    "quadrature_tet4); use 'colored' (reproducible) or 'atomic'");
        if (!sym)
            return launch_run(h, p, TAL_SCATTER_ATOMIC, s, launches);
        const bool ordered = scatter == TAL_SCATTER_PRIVATE;
        PrivArgs pa{h->d_blobs, h->d_blob_off, (int)h->info.n_chunks, nullptr,
                    h->has_press ? h->d_press : nullptr};
        PeerArgs peer{};
        const int np = h->n_peers();
        if (np && ordered)
            return fail(TAL_EINVAL, "the fused interface sum needs scatter='private-atomic'");
        if (np) {
            peer.pidx = h->d_pidx;
            for (int sl = 0; sl < 2; ++sl)
                if (h->peers[sl].rx) {
                    peer.rx[sl] = h->peers[sl].rx;
                    peer.ry[sl] = h->peers[sl].rx + h->peers[sl].n;
                    peer.rz[sl] = h->peers[sl].rx + 2 * h->peers[sl].n;
                }
        }
        if (ordered && h->d_partial) {
            pa.part = h->d_partial;
        }
        // shared nodes receive FP64 REDs: zero the RHS first (a separate pass:
        // zeroing inside the kernel, by thread or TMA bulk stores, measured
        // ~45 us slower -- DESIGN.md)
        if (!ordered && N) {
            TAL_CK(zero_rhs(h, s, true));
        }
        if (np) {  // every neighbour has zeroed before anyone REDs into it
            k_peer_signal<<<1, 1, 0, s>>>(h->peers[0].flags, h->peers[1].flags, 0, h->d_flags + 2);
            k_peer_wait<<<1, 1, 0, s>>>(h->d_flags, 0, np);
            TAL_CK_LAUNCH();
            nl += 2;
        }
        if (h->info.n_chunks) {
            const int ext = (pa.press ? 1 : 0) | (st ? 2 : 0);
            const unsigned grid = (unsigned)std::min<int64_t>(h->priv_grid_ext[ext], h->info.n_chunks);
            pm.begin();
            const cudaError_t le = launch_private(h->priv_cfg, ordered, st, grid, s, pa, nodes, rhs, kc, peer);
            pm.end();
            if (le != cudaSuccess)
                return fail(TAL_ECUDA, std::string("private kernel launch: ") + cudaGetErrorString(le));
            ++nl;
        }
        if (np) {  // every neighbour's REDs into this RHS have landed
            k_peer_signal<<<1, 1, 0, s>>>(h->peers[0].flags, h->peers[1].flags, 1, nullptr);
            k_peer_wait<<<1, 1, 0, s>>>(h->d_flags, 1, np);
            TAL_CK_LAUNCH();
            nl += 2;
        }
        const int64_t nb = (int64_t)h->ch.bnd_nodes.size();
        if (ordered && nb) {
            k_merge_partials<<<grid_for(nb, 256), 256, 0, s>>>(h->d_bnd_nodes, h->d_bnd_off, h->d_bnd_pos,
                                                              nb, pa.part, rhs);
            TAL_CK_LAUNCH();
            ++nl;
        }
        break;
    }
    case TAL_SCATTER_SEQUENTIAL: {
        if (h->has_press || st)
            return fail(TAL_EINVAL, "scatter 'sequential' reproduces the reference operator, which has no "
                                    "pressure or stabilisation term; switch them off first");
        if (N && !h->d_seq_off)
            if (int rc = build_sequential(h))
                return rc;
        if (N) {
            pm.begin();
            if (h->d_seq_rows) {
                if (E)
                    k_strict_rows<<<grid_for(E, 128), 128, 0, s>>>(E, h->conn, nodes, h->d_seq_dlt,
                                                                  h->d_seq_rows, kc);
                k_sum_rows_ordered<<<grid_for(N, 256), 256, 0, s>>>(h->d_seq_off, h->d_seq_ent, N,
                                                                    h->d_seq_rows, rhs.rx, rhs.ry, rhs.rz);
                nl += E ? 1 : 0;
            } else {
                k_assemble_sequential<<<grid_for(N, 128), 128, 0, s>>>(h->d_seq_off, h->d_seq_ent, N, h->conn,
                                                                      nodes, h->d_seq_dlt, rhs.rx, rhs.ry,
                                                                      rhs.rz, kc, false);
            }
            pm.end();
            TAL_CK_LAUNCH();
            ++nl;
        }
        break;
    }
    default:
        return fail(TAL_EINVAL, "unknown scatter mode " + std::to_string(scatter));
    }
    if (launches)
        *launches = nl;
    return TAL_OK;
}

// B / RS code shapes (tal_shapes.cuh): one thread per element over the
// chunk-ordered connectivity (REDs) or colour by colour (plain stores)
ShapeConsts shape_consts(const tal_params *p)
{
    ShapeConsts sc{};
    sc.rho = p->rho;
    sc.mu = p->mu;
    sc.cvre = p->c_vreman;
    sc.nn = 4;
    sc.nd = 3;
    sc.ng = 4;
    // quadrature_tet4 (kernel.py:71-86): same IEEE operations as the reference
    const double qa = (5.0 + 3.0 * std::sqrt(5.0)) / 20.0, qb = (5.0 - std::sqrt(5.0)) / 20.0;
    static const double ref_grads[4][3] = {{-1.0, -1.0, -1.0}, {1.0, 0.0, 0.0}, {0.0, 1.0, 0.0}, {0.0, 0.0, 1.0}};
    for (int g = 0; g < 4; ++g) {
        sc.wts[g] = 0.25;
        for (int a = 0; a < 4; ++a) {
            sc.npts[g][a] = (a == g) ? qa : qb;
            for (int k = 0; k < 3; ++k)
                sc.dshape[g][a][k] = ref_grads[a][k];
        }
    }
    return sc;
}

int launch_shape(tal_handle *h, const tal_params *p, int variant, int scatter, cudaStream_t s,
                 int64_t *launches)
{
    ProfMark pm{h, s};
    ElemConsts kc;
    bool sym;
    if (!make_consts(p, kc, sym))
        return fail(TAL_EINVAL, "non-finite physical parameters");
    const ShapeConsts sc = shape_consts(p);
    const double *nodes = h->REC();
    RhsSoA rhs{h->RX(), h->RY(), h->RZ()};
    const int64_t N = h->N, E = h->E;
    const bool colored = scatter == TAL_SCATTER_PRIVATE || scatter == TAL_SCATTER_COLORED;
    if (!colored && scatter != TAL_SCATTER_ATOMIC && scatter != TAL_SCATTER_PRIVATE_ATOMIC)
        return fail(TAL_EINVAL, "unknown scatter mode " + std::to_string(scatter));
    if (colored && !h->conn_col && E)
        return fail(TAL_ESTATE, "colour-by-colour scatter needs a colouring (build_colors=1 or colors)");
    int64_t nl = 0;
    if (N) {
        TAL_CK(zero_rhs(h, s));
    }
    auto one = [&](const int4 *conn, int64_t b, int64_t e) -> int {
        const unsigned grid = grid_for(e - b, 256);
        if (variant == TAL_VARIANT_B) {
            if (colored)
                k_assemble_baseline<true><<<grid, 256, 0, s>>>(conn, b, e, nodes, rhs, sc);
            else
                k_assemble_baseline<false><<<grid, 256, 0, s>>>(conn, b, e, nodes, rhs, sc);
        } else if (variant == TAL_VARIANT_P) {
            if (colored)
                k_assemble_baseline<true, true><<<grid, 256, 0, s>>>(conn, b, e, nodes, rhs, sc);
            else
                k_assemble_baseline<false, true><<<grid, 256, 0, s>>>(conn, b, e, nodes, rhs, sc);
        } else {
            if (colored)
                k_assemble_rs<true><<<grid, 256, 0, s>>>(conn, b, e, nodes, rhs, sc);
            else
                k_assemble_rs<false><<<grid, 256, 0, s>>>(conn, b, e, nodes, rhs, sc);
        }
        TAL_CK_LAUNCH();
        ++nl;
        return TAL_OK;
    };
    pm.begin();
    if (colored) {
        for (size_t c = 0; c + 1 < h->col_off.size(); ++c) {
            const int64_t b = h->col_off[c], e = h->col_off[c + 1];
            if (e > b)
                if (int rc = one(h->conn_col, b, e))
                    return rc;
        }
    } else if (E) {
        if (int rc = one(h->conn, 0, E))
            return rc;
    }
    pm.end();
    if (launches)
        *launches = nl;
    return TAL_OK;
}

// caller ids of the chunk-node entries (gather order, rank order), built on
// first use from the host chunk tables and the node permutation
int build_caller_ids(tal_handle *h)
{
    if (h->d_blobs_cl || h->ch.gather_nodes.empty())
        return TAL_OK;
    const int64_t n = (int64_t)h->ch.gather_nodes.size();
    std::vector<int32_t> perm;
    if (!h->h_iperm.empty()) {
        perm.resize((size_t)h->N);
        for (int64_t c = 0; c < h->N; ++c)
            perm[h->h_iperm[c]] = (int32_t)c;
    }
    std::vector<int32_t> cg((size_t)n), cc((size_t)n);
    parallel_for(n, [&](int64_t i0, int64_t i1, int) {
        for (int64_t i = i0; i < i1; ++i) {
            const int32_t g = h->ch.gather_nodes[i], c = h->ch.cnodes[i] & 0x7fffffff;
            cg[i] = perm.empty() ? g : perm[g];
            cc[i] = perm.empty() ? c : perm[c];
        }
    });
    int32_t *d_cg = nullptr, *d_cc = nullptr;
    int rc = dev_upload(&d_cg, cg.data(), cg.size());
    if (!rc)
        rc = dev_upload(&d_cc, cc.data(), cc.size());
    cudaError_t e = cudaSuccess;
    if (!rc && ((e = cudaMalloc((void **)&h->d_blobs_cl, (size_t)h->blob_bytes)) != cudaSuccess ||
                (e = cudaMalloc((void **)&h->d_xc, sizeof(double) * 3 * h->N)) != cudaSuccess ||
                (e = cudaMemcpyAsync(h->d_blobs_cl, h->d_blobs, (size_t)h->blob_bytes, cudaMemcpyDeviceToDevice,
                                     h->stream)) != cudaSuccess))
        rc = fail(TAL_ECUDA, std::string("caller-layout tables: ") + cudaGetErrorString(e));
    if (!rc) {
        const unsigned nc = (unsigned)h->info.n_chunks;
        if (h->priv_cfg == 0)
            k_cl_blobs<0><<<nc, PrivCfg<0>::THREADS, 0, h->stream>>>(h->d_blobs_cl, h->d_blob_off, d_cg, d_cc);
        else if (h->priv_cfg == 1)
            k_cl_blobs<1><<<nc, PrivCfg<1>::THREADS, 0, h->stream>>>(h->d_blobs_cl, h->d_blob_off, d_cg, d_cc);
        else
            k_cl_blobs<2><<<nc, PrivCfg<2>::THREADS, 0, h->stream>>>(h->d_blobs_cl, h->d_blob_off, d_cg, d_cc);
        k_caller_coords<<<grid_for(h->N, 256), 256, 0, h->stream>>>(h->REC(), h->perm, h->N, h->d_xc);
        if ((e = cudaGetLastError()) != cudaSuccess || (e = cudaStreamSynchronize(h->stream)) != cudaSuccess)
            rc = fail(TAL_ECUDA, std::string("caller-layout tables: ") + cudaGetErrorString(e));
    }
    if (d_cg)
        cudaFree(d_cg);
    if (d_cc)
        cudaFree(d_cc);
    return rc;
}

// One assembly from and to the caller's device arrays: the fused caller-layout
// private kernel when it applies (symmetric rule, private / private-atomic,
// no pressure / SUPG / peers), else the composition set_velocity_device ->
// run -> get_rhs_device.
int launch_caller(tal_handle *h, const tal_params *p, int scatter, const double *d_u, double *d_rhs,
                  cudaStream_t s, int64_t *launches)
{
    ElemConsts kc;
    bool sym;
    if (!make_consts(p, kc, sym))
        return fail(TAL_EINVAL, "non-finite physical parameters");
    const bool fused = sym && !h->has_press && !h->has_st && !h->n_peers() && h->info.n_chunks > 0 &&
                       (scatter == TAL_SCATTER_PRIVATE || scatter == TAL_SCATTER_PRIVATE_ATOMIC);
    if (!fused) {
        if (h->N) {
            k_pack_velocity<<<grid_for(h->N, 256), 256, 0, s>>>(d_u, h->perm, h->N, h->REC());
            TAL_CK_LAUNCH();
        }
        int64_t nl = 0;
        if (int rc = launch_run(h, p, scatter, s, &nl))
            return rc;
        if (h->N) {
            k_unpack_aos<<<grid_for(h->N, 256), 256, 0, s>>>(h->RX(), h->RY(), h->RZ(), h->iperm, h->N, d_rhs);
            TAL_CK_LAUNCH();
        }
        if (launches)
            *launches = nl + (h->N ? 2 : 0);
        return TAL_OK;
    }
    if (int rc = build_caller_ids(h))
        return rc;
    const bool ordered = scatter == TAL_SCATTER_PRIVATE;
    ProfMark pm{h, s};
    int64_t nl = 0;
    if (!ordered)  // shared nodes are REDed into it: zero the caller's rhs first
        TAL_CK(cudaMemsetAsync(d_rhs, 0, sizeof(double) * 3 * h->N, s));
    PrivArgs pa{h->d_blobs_cl, h->d_blob_off, (int)h->info.n_chunks, ordered ? h->d_partial : nullptr, nullptr,
                h->d_xc, d_u, d_rhs};
    RhsSoA rhs{h->RX(), h->RY(), h->RZ()};
    const unsigned grid = (unsigned)std::min<int64_t>(h->priv_grid_ext[0], h->info.n_chunks);
    pm.begin();
    const cudaError_t le = launch_private(h->priv_cfg, ordered, false, grid, s, pa, h->REC(), rhs, kc, PeerArgs{});
    pm.end();
    if (le != cudaSuccess)
        return fail(TAL_ECUDA, std::string("private kernel launch: ") + cudaGetErrorString(le));
    ++nl;
    const int64_t nb = (int64_t)h->ch.bnd_nodes.size();
    if (ordered && nb) {
        k_merge_partials<<<grid_for(nb, 256), 256, 0, s>>>(h->d_bnd_nodes, h->d_bnd_off, h->d_bnd_pos, nb,
                                                          h->d_partial, rhs, d_rhs, h->perm);
        TAL_CK_LAUNCH();
        ++nl;
    }
    if (launches)
        *launches = nl;
    return TAL_OK;
}

int launch_any(tal_handle *h, const tal_params *p, int variant, int scatter, cudaStream_t s, int64_t *launches)
{
    if (variant == TAL_VARIANT_RSP)
        return launch_run(h, p, scatter, s, launches);
    const bool shape = variant == TAL_VARIANT_B || variant == TAL_VARIANT_RS || variant == TAL_VARIANT_P;
    if ((h->has_press || h->has_st) && shape)
        return fail(TAL_EINVAL, "the pressure-gradient and SUPG terms are implemented for the RSP shape only");
    if (shape)
        return launch_shape(h, p, variant, scatter, s, launches);
    return fail(TAL_EINVAL, "unknown variant " + std::to_string(variant));
}

template <int CFG>
int set_attrs_cfg(int device, int grid_ext[4])
{
    constexpr int sm = PrivLayoutOf<CFG>::TOTAL, sm_pr = PrivLayoutOf<CFG, true>::TOTAL;
    int n_sm = 0;
    TAL_CK(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, device));
    for (int ext = 0; ext < 4; ++ext) {
        const bool pr = ext & 1, st = ext & 2;
        const int bytes = pr ? sm_pr : sm;
        const void *fns[] = {private_fn<CFG, true>(false, pr, st), private_fn<CFG, false>(false, pr, st),
                             private_fn<CFG, false>(true, pr, false), private_fn<CFG, true>(false, pr, st, true),
                             private_fn<CFG, false>(false, pr, st, true)};
        for (const void *f : fns)
            TAL_CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
        int per_sm = 0;
        TAL_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fns[1], PrivCfg<CFG>::THREADS, bytes));
        grid_ext[ext] = std::max(1, per_sm) * n_sm;
    }
    return TAL_OK;
}

int set_kernel_attrs(int device, int cfg, int grid_ext[4])
{
    return cfg == 0   ? set_attrs_cfg<0>(device, grid_ext)
           : cfg == 1 ? set_attrs_cfg<1>(device, grid_ext)
                      : set_attrs_cfg<2>(device, grid_ext);
}

// cta_patches -> CTA configuration (PrivCfg in tal_kernels.cuh)
int cfg_for(int cta_patches)
{
    return cta_patches <= PrivCfg<0>::THREADS ? 0 : cta_patches <= PrivCfg<1>::THREADS ? 1 : 2;
}
template <class F>
int by_cfg(int cfg, F f)
{
    return cfg == 0 ? f(PrivCfg<0>{}) : cfg == 1 ? f(PrivCfg<1>{}) : f(PrivCfg<2>{});
}
int cfg_threads(int cfg) { return by_cfg(cfg, [](auto c) { return decltype(c)::THREADS; }); }
int cfg_max_nodes(int cfg) { return by_cfg(cfg, [](auto c) { return decltype(c)::NM; }); }
int cfg_max_contrib(int cfg) { return by_cfg(cfg, [](auto c) { return decltype(c)::NC; }); }

// Host half of a mesh upload: renumbering, element order, patches, CTA
// chunks (tal_prep.hpp).  Shared by tal_upload_mesh_ex and tal_plan_layout.
struct HostLayout {
    std::vector<int32_t> perm, iperm, eperm, cord;
    std::vector<double> xin;
    Patches patches;
    Chunking ch;
    int cfg = 1;
    int64_t n_interior = 0;  // internal ids [0, n_interior): chunk-interior nodes (shared_tail)
};

// Renumber so that the chunk-interior nodes come first, in chunk / slot
// order, and the shared (and isolated) nodes form the tail [n_interior, N):
// scatter 'private-atomic' then zeroes only the tail (interior nodes are
// plain-stored by their one chunk), and a chunk's interior records are one
// contiguous block for the gather.  TAL_SHARED_TAIL=0 disables it.
void shared_tail_renumber(int64_t n_nodes, HostLayout &L)
{
    static const bool on = [] {
        const char *e = std::getenv("TAL_SHARED_TAIL");
        return !e || std::atoi(e) != 0;
    }();
    if (!on || !n_nodes)
        return;
    std::vector<uint8_t> interior((size_t)n_nodes, 0);
    for (int32_t raw : L.ch.cnodes)
        if (raw < 0)
            interior[raw & 0x7fffffff] = 1;
    std::vector<int32_t> nid((size_t)n_nodes, -1);
    int32_t next = 0;
    for (int32_t v : L.ch.gather_nodes)
        if (interior[v] && nid[v] < 0)
            nid[v] = next++;
    L.n_interior = next;
    for (int64_t v = 0; v < n_nodes; ++v)
        if (nid[v] < 0)
            nid[v] = next++;
    const bool had = !L.perm.empty();
    std::vector<int32_t> perm((size_t)n_nodes), iperm((size_t)n_nodes);
    std::vector<double> xin((size_t)(3 * n_nodes));
    parallel_for(n_nodes, [&](int64_t v0, int64_t v1, int) {  // nid is a permutation: disjoint writes
        for (int64_t v = v0; v < v1; ++v) {
            const int32_t caller = had ? L.perm[v] : (int32_t)v;
            perm[nid[v]] = caller;
            iperm[caller] = nid[v];
            for (int c = 0; c < 3; ++c)
                xin[3 * (int64_t)nid[v] + c] = L.xin[3 * v + c];
        }
    });
    L.perm.swap(perm);
    L.iperm.swap(iperm);
    L.xin.swap(xin);
    auto remap = [&](std::vector<int32_t> &a) {
        parallel_for((int64_t)a.size(), [&](int64_t i0, int64_t i1, int) {
            for (int64_t i = i0; i < i1; ++i)
                a[i] = nid[a[i]];
        });
    };
    remap(L.cord);
    remap(L.patches.nodes);
    remap(L.ch.gather_nodes);
    remap(L.ch.bnd_nodes);
    parallel_for((int64_t)L.ch.cnodes.size(), [&](int64_t i0, int64_t i1, int) {
        for (int64_t i = i0; i < i1; ++i) {
            const int32_t x = L.ch.cnodes[i];
            L.ch.cnodes[i] = (int32_t)(((uint32_t)x & 0x80000000u) | (uint32_t)nid[x & 0x7fffffff]);
        }
    });
}

int host_layout(const double *coords, const int64_t *conn, int64_t n_nodes, int64_t n_elems,
                const tal_mesh_opts &opts, const int64_t *external, int64_t n_external, HostLayout &L)
{
    static const bool times = std::getenv("TAL_PREP_TIMES") != nullptr;  // phase timings to stderr
    auto tick = std::chrono::steady_clock::now();
    auto lap = [&](const char *what) {
        const auto now = std::chrono::steady_clock::now();
        if (times)
            std::fprintf(stderr, "[tal prep] %-14s %8.3f s\n", what,
                         std::chrono::duration<double>(now - tick).count());
        tick = now;
    };
    // node renumbering: perm[new] = old
    if (opts.renumber == TAL_RENUMBER_RCM)
        renumber_rcm(conn, n_nodes, n_elems, L.perm);
    else if (opts.renumber == TAL_RENUMBER_SFC)
        renumber_sfc(coords, n_nodes, L.perm);
    else if (opts.renumber != TAL_RENUMBER_NONE)
        return fail(TAL_EINVAL, "unknown renumber method");
    lap("renumber");
    const bool renum = !L.perm.empty();
    if (renum) {
        L.iperm.resize((size_t)n_nodes);
        parallel_for(n_nodes, [&](int64_t i0, int64_t i1, int) {
            for (int64_t i = i0; i < i1; ++i)
                L.iperm[L.perm[i]] = (int32_t)i;
        });
    }
    L.xin.resize((size_t)(3 * n_nodes));  // internal AoS coords
    parallel_for(n_nodes, [&](int64_t i0, int64_t i1, int) {
        for (int64_t i = i0; i < i1; ++i) {
            const int64_t s = renum ? L.perm[i] : i;
            for (int c = 0; c < 3; ++c)
                L.xin[3 * i + c] = coords[3 * s + c];
        }
    });
    std::vector<int32_t> cin((size_t)(4 * n_elems));
    parallel_for(4 * n_elems, [&](int64_t i0, int64_t i1, int) {
        for (int64_t i = i0; i < i1; ++i)
            cin[i] = renum ? L.iperm[conn[i]] : (int32_t)conn[i];
    });
    lap("relabel");
    // element order
    element_order(opts.element_order, cin.data(), L.xin.data(), n_nodes, n_elems, L.eperm);
    lap("element order");
    L.cord.resize((size_t)(4 * n_elems));
    parallel_for(n_elems, [&](int64_t e0, int64_t e1, int) {
        for (int64_t e = e0; e < e1; ++e)
            for (int a = 0; a < 4; ++a)
                L.cord[4 * e + a] = cin[4 * (int64_t)L.eperm[e] + a];
    });
    // chunks
    std::string err;
    const int cfg = cfg_for(opts.cta_patches);
    if (opts.cta_patches < 1 || opts.cta_patches > cfg_threads(2) || opts.chunk_nodes < 16 ||
        opts.chunk_nodes > cfg_max_nodes(cfg) || (opts.patch_mode != 0 && opts.patch_mode != 1))
        return fail(TAL_EINVAL, "cta_patches must be in [1," + std::to_string(cfg_threads(2)) +
                                    "], chunk_nodes in [16," + std::to_string(cfg_max_nodes(cfg)) +
                                    "], patch_mode 0|1");
    L.cfg = cfg;
    lap("reorder");
    build_patches(L.cord.data(), n_nodes, n_elems, opts.patch_mode, L.patches);
#if TAL_ORIENT
    orient_patches(L.patches, L.xin.data());
#endif
    lap("patches");
    std::vector<uint8_t> ext;
    if (n_external) {
        ext.assign((size_t)n_nodes, 0);
        for (int64_t i = 0; i < n_external; ++i)
            ext[renum ? L.iperm[external[i]] : external[i]] = 1;
    }
    if (!build_chunks(L.patches, n_nodes, opts.cta_patches, opts.chunk_nodes, cfg_max_contrib(cfg),
                      ext.empty() ? nullptr : ext.data(), L.ch, err))
        return fail(TAL_EINVAL, err);
    lap("chunks");
    if (opts.renumber != TAL_RENUMBER_NONE)  // 'none' keeps the caller's numbering
        shared_tail_renumber(n_nodes, L);
    lap("tail renumber");
    return TAL_OK;
}

}  // namespace

// No C++ exception may cross the C ABI: every entry
// point's body runs inside this guard (allocation failures -> TAL_ENOMEM,
// anything else -> TAL_EINTERNAL with the message kept for tal_last_error).
#define TAL_GUARD_BEGIN try {
#define TAL_GUARD_END                                                           \
    }                                                                           \
    catch (const std::bad_alloc &) { return fail(TAL_ENOMEM, "host allocation failed"); } \
    catch (const std::exception &ex) { return fail(TAL_EINTERNAL, ex.what()); } \
    catch (...) { return fail(TAL_EINTERNAL, "unknown C++ exception"); }

extern "C" {

const char *tal_last_error(void) { return g_err.c_str(); }
int64_t tal_last_error_line(void) { return g_err_line; }

// ---- mesh IO / partitioning (tal_meshio.cpp) ---------------------------------
struct tal_meshbuf {
    MeshText m;
};

int tal_mesh_load_text(const char *path, tal_meshbuf **out)
{
    TAL_GUARD_BEGIN
    if (!path || !out)
        return fail(TAL_EINVAL, "NULL argument");
    *out = nullptr;
    std::unique_ptr<tal_meshbuf> b(new tal_meshbuf());
    std::string err;
    int64_t line = 0;
    if (!load_mesh_text(path, b->m, err, line)) {
        const int rc = fail(TAL_EINVAL, line > 0 ? "line " + std::to_string(line) + ": " + err : err);
        g_err_line = line;
        return rc;
    }
    *out = b.release();
    return TAL_OK;
    TAL_GUARD_END
}

int tal_meshbuf_info(tal_meshbuf *b, int64_t *n_nodes, int64_t *n_elems, int64_t *n_reoriented)
{
    TAL_GUARD_BEGIN
    if (!b || !n_nodes || !n_elems || !n_reoriented)
        return fail(TAL_EINVAL, "NULL argument");
    *n_nodes = b->m.n_nodes, *n_elems = b->m.n_elems, *n_reoriented = b->m.n_reoriented;
    return TAL_OK;
    TAL_GUARD_END
}

int tal_meshbuf_copy(tal_meshbuf *b, double *coords, int64_t *conn)
{
    TAL_GUARD_BEGIN
    if (!b || (b->m.n_nodes && !coords) || (b->m.n_elems && !conn))
        return fail(TAL_EINVAL, "NULL argument");
    std::memcpy(coords, b->m.coords.data(), sizeof(double) * b->m.coords.size());
    std::memcpy(conn, b->m.conn.data(), sizeof(int64_t) * b->m.conn.size());
    return TAL_OK;
    TAL_GUARD_END
}

int tal_meshbuf_free(tal_meshbuf *b)
{
    delete b;
    return TAL_OK;
}

int tal_mesh_save_text(const char *path, const double *coords, const int64_t *conn, int64_t n_nodes,
                       int64_t n_elems)
{
    TAL_GUARD_BEGIN
    if (!path || n_nodes < 0 || n_elems < 0 || (n_nodes && !coords) || (n_elems && !conn))
        return fail(TAL_EINVAL, "bad arguments");
    std::string err;
    if (!save_mesh_text(path, coords, conn, n_nodes, n_elems, err))
        return fail(TAL_EIO, err);
    return TAL_OK;
    TAL_GUARD_END
}

int tal_mesh_save_binary(const char *path, const double *coords, const int64_t *conn, int64_t n_nodes,
                         int64_t n_elems)
{
    TAL_GUARD_BEGIN
    if (!path || n_nodes < 0 || n_elems < 0 || (n_nodes && !coords) || (n_elems && !conn))
        return fail(TAL_EINVAL, "bad arguments");
    std::string err;
    if (!save_mesh_binary(path, coords, conn, n_nodes, n_elems, err))
        return fail(TAL_EIO, err);
    return TAL_OK;
    TAL_GUARD_END
}

int tal_mesh_probe_binary(const char *path, int64_t *n_nodes, int64_t *n_elems, int *is_binary)
{
    TAL_GUARD_BEGIN
    if (!path || !n_nodes || !n_elems || !is_binary)
        return fail(TAL_EINVAL, "NULL argument");
    const int r = probe_mesh_binary(path, n_nodes, n_elems);
    if (r < 0)
        return fail(TAL_EIO, std::string("cannot open ") + path);
    *is_binary = r;
    return TAL_OK;
    TAL_GUARD_END
}

int tal_mesh_load_binary(const char *path, double *coords, int64_t n_nodes, int64_t *conn, int64_t n_elems)
{
    TAL_GUARD_BEGIN
    if (!path || n_nodes < 0 || n_elems < 0 || (n_nodes && !coords) || (n_elems && !conn))
        return fail(TAL_EINVAL, "bad arguments");
    std::string err;
    if (!load_mesh_binary(path, coords, n_nodes, conn, n_elems, err))
        return fail(TAL_EINVAL, err);
    return TAL_OK;
    TAL_GUARD_END
}

int tal_rcb_parts(const double *points, int64_t n, int world, int32_t *parts)
{
    TAL_GUARD_BEGIN
    if (n < 0 || world < 1 || (n && (!points || !parts)))
        return fail(TAL_EINVAL, "bad arguments (world must be >= 1)");
    rcb_parts(points, n, world, parts);
    return TAL_OK;
    TAL_GUARD_END
}
int tal_abi_version(void) { return TAL_ABI_VERSION; }

int tal_device_count(int *count)
{
    TAL_GUARD_BEGIN
    if (!count)
        return fail(TAL_EINVAL, "count is NULL");
    *count = 0;
    cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) {
        *count = 0;
        return fail(TAL_ECUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
    }
    return TAL_OK;
    TAL_GUARD_END
}

int tal_create(int device, tal_handle **out)
{
    TAL_GUARD_BEGIN
    if (!out)
        return fail(TAL_EINVAL, "out is NULL");
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return fail(TAL_ECUDA, std::string("no CUDA device available (") + cudaGetErrorString(e) +
                                   "); the assembly has no CPU fallback");
    if (device < 0 || device >= n)
        return fail(TAL_EINVAL, "device index out of range");
    cudaDeviceProp prop;
    TAL_CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
        return fail(TAL_ECUDA, std::string("device ") + prop.name + " is not sm_100-class");
    DeviceGuard g(device);
    tal_handle *h = new tal_handle();
    h->device = device;
    if (cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete h;
        return fail(TAL_ECUDA, "cudaStreamCreate failed");
    }
    for (auto &ev : h->ev)
        cudaEventCreate(&ev);
    if (cudaMalloc((void **)&h->d_flags, 8 * sizeof(unsigned long long)) != cudaSuccess ||
        cudaMemset(h->d_flags, 0, 8 * sizeof(unsigned long long)) != cudaSuccess) {
        delete h;
        return fail(TAL_ECUDA, "flag allocation failed");
    }
    cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking);
    for (int s = 0; s < tal_handle::ASYNC_SLOTS; ++s) {
        cudaEventCreateWithFlags(&h->ev_h2d[s], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&h->ev_comp[s], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&h->ev_d2h[s], cudaEventDisableTiming);
    }
    *out = h;
    return TAL_OK;
    TAL_GUARD_END
}

int tal_destroy(tal_handle *h)
{
    TAL_GUARD_BEGIN
    if (!h)
        return TAL_OK;
    DeviceGuard g(h->device);
    cudaStreamSynchronize(h->stream);
    cudaStreamSynchronize(h->s_h2d);
    cudaStreamSynchronize(h->s_d2h);
    h->free_mesh();
    for (auto &ev : h->ev)
        cudaEventDestroy(ev);
    for (int s = 0; s < tal_handle::ASYNC_SLOTS; ++s) {
        cudaEventDestroy(h->ev_h2d[s]);
        cudaEventDestroy(h->ev_comp[s]);
        cudaEventDestroy(h->ev_d2h[s]);
    }
    cudaStreamDestroy(h->s_h2d);
    cudaStreamDestroy(h->s_d2h);
    if (h->d_flags)
        cudaFree(h->d_flags);
    for (auto &ev : h->prof_ev)
        cudaEventDestroy(ev);
    cudaStreamDestroy(h->stream);
    delete h;
    return TAL_OK;
    TAL_GUARD_END
}

int tal_host_alloc(int64_t bytes, void **out)
{
    TAL_GUARD_BEGIN
    if (!out || bytes < 0)
        return fail(TAL_EINVAL, "bad arguments");
    TAL_CK(cudaMallocHost(out, (size_t)std::max<int64_t>(bytes, 1)));
    return TAL_OK;
    TAL_GUARD_END
}

int tal_host_register(void *p, int64_t bytes)
{
    TAL_GUARD_BEGIN
    if (!p || bytes <= 0)
        return fail(TAL_EINVAL, "bad arguments");
    TAL_CK(cudaHostRegister(p, (size_t)bytes, cudaHostRegisterDefault));
    return TAL_OK;
    TAL_GUARD_END
}

int tal_host_unregister(void *p)
{
    TAL_GUARD_BEGIN
    if (p)
        TAL_CK(cudaHostUnregister(p));
    return TAL_OK;
    TAL_GUARD_END
}

int tal_host_free(void *p)
{
    TAL_GUARD_BEGIN
    if (p)
        TAL_CK(cudaFreeHost(p));
    return TAL_OK;
    TAL_GUARD_END
}

int tal_default_mesh_opts(tal_mesh_opts *o)
{
    TAL_GUARD_BEGIN
    if (!o)
        return fail(TAL_EINVAL, "NULL");
    o->renumber = TAL_RENUMBER_RCM;
    o->element_order = TAL_EORDER_SFC;
    o->cta_patches = 128;
    o->patch_mode = 1;
    o->chunk_nodes = 256;
    o->validate = 1;
    o->build_colors = 0;
    return TAL_OK;
    TAL_GUARD_END
}

int tal_upload_mesh(tal_handle *h, const double *coords, const int64_t *conn, int64_t n_nodes,
                    int64_t n_elems, const int64_t *colors, const tal_mesh_opts *opts_in)
{
    TAL_GUARD_BEGIN
    return tal_upload_mesh_ex(h, coords, conn, n_nodes, n_elems, colors, opts_in, nullptr, 0);
    TAL_GUARD_END
}

int tal_upload_mesh_ex(tal_handle *h, const double *coords, const int64_t *conn, int64_t n_nodes,
                       int64_t n_elems, const int64_t *colors, const tal_mesh_opts *opts_in,
                       const int64_t *external, int64_t n_external)
{
    TAL_GUARD_BEGIN
    if (!h)
        return fail(TAL_EINVAL, "handle is NULL");
    if (n_external < 0 || (n_external && !external))
        return fail(TAL_EINVAL, "bad external node list");
    for (int64_t i = 0; i < n_external; ++i)
        if (external[i] < 0 || external[i] >= n_nodes)
            return fail(TAL_EINVAL, "external node id out of range [0, n_nodes)");
    if (n_nodes < 0 || n_elems < 0)
        return fail(TAL_EINVAL, "negative sizes");
    if (n_nodes >= (int64_t)1 << 31 || n_elems >= (int64_t)1 << 31)
        return fail(TAL_EINVAL, "meshes are limited to 2^31-1 nodes/elements per device");
    if ((n_nodes && !coords) || (n_elems && !conn))
        return fail(TAL_EINVAL, "NULL mesh arrays");
    tal_mesh_opts opts;
    tal_default_mesh_opts(&opts);
    if (opts_in)
        opts = *opts_in;
    const auto t0 = std::chrono::steady_clock::now();
    // validation (Mesh.__post_init__, mesh.py:50-75)
    {
        std::atomic<bool> bad{false};
        parallel_for(4 * n_elems, [&](int64_t i0, int64_t i1, int) {
            for (int64_t i = i0; i < i1; ++i)
                if (conn[i] < 0 || conn[i] >= n_nodes) {
                    bad = true;
                    return;
                }
        });
        if (bad)
            return fail(TAL_EINVAL, "connectivity index out of range [0, n_nodes)");
    }
    if (opts.validate && n_elems) {
        std::vector<double> vols((size_t)n_elems);
        signed_volumes(coords, conn, n_elems, vols.data());
        for (int64_t e = 0; e < n_elems; ++e)
            if (!(vols[e] > 0.0)) {
                char buf[128];
                snprintf(buf, sizeof buf, "element %lld has non-positive signed volume %g",
                         (long long)e, vols[e]);
                return fail(TAL_EINVAL, buf);
            }
    }
    if (colors) {  // colour ids index per-colour tables below: bound them first
        for (int64_t e = 0; e < n_elems; ++e)
            if (colors[e] < 0 || colors[e] >= std::max<int64_t>(n_elems, 1))
                return fail(TAL_EINVAL, "colour ids must lie in [0, n_elems)");
        if (!check_coloring(conn, colors, n_nodes, n_elems))
            return fail(TAL_EINVAL, "coloring invalid: elements sharing a node share a color");
    }

    DeviceGuard g(h->device);
    cudaStreamSynchronize(h->stream);
    h->free_mesh();
    h->N = n_nodes;
    h->E = n_elems;

    HostLayout L;
    if (int rc = host_layout(coords, conn, n_nodes, n_elems, opts, external, n_external, L))
        return rc;
    const int cfg = L.cfg;
    h->priv_cfg = cfg;
    h->n_interior = L.n_interior;
    h->ch = std::move(L.ch);
    std::vector<int32_t> &perm = L.perm, &iperm = L.iperm, &eperm = L.eperm, &cord = L.cord;
    std::vector<double> &xin = L.xin;
    const bool renum = !perm.empty();
    Patches &patches = L.patches;
    h->info.n_patches = patches.n_patches();
    std::vector<uint8_t> blobs;
    std::vector<int32_t> blob_off;
    pack_blobs(h->ch, cfg_threads(cfg), blobs, blob_off);
    // colouring (caller's or greedy on the internal order), colour-sorted copy
    std::vector<int64_t> col;
    int64_t ncol = 0;
    if (colors) {
        col.resize((size_t)n_elems);
        for (int64_t e = 0; e < n_elems; ++e)
            col[e] = colors[eperm[e]];
        for (int64_t c : col)
            ncol = std::max(ncol, c + 1);
    } else if (opts.build_colors) {
        std::vector<int64_t> c64((size_t)(4 * n_elems));
        for (int64_t i = 0; i < 4 * n_elems; ++i)
            c64[i] = cord[i];
        col.resize((size_t)n_elems);
        ncol = color_elements(c64.data(), n_nodes, n_elems, col.data());
        if (ncol < 0)
            return fail(TAL_EINVAL, "greedy colouring needs more than 256 colours");
    }
    std::vector<int32_t> ccol;
    if (!col.empty()) {
        h->col_off.assign((size_t)ncol + 1, 0);
        for (int64_t c : col)
            h->col_off[c + 1]++;
        for (int64_t c = 0; c < ncol; ++c)
            h->col_off[c + 1] += h->col_off[c];
        std::vector<int64_t> fill(h->col_off.begin(), h->col_off.end() - 1);
        ccol.resize((size_t)(4 * n_elems));
        for (int64_t e = 0; e < n_elems; ++e) {
            const int64_t d = fill[col[e]]++;
            for (int a = 0; a < 4; ++a)
                ccol[4 * d + a] = cord[4 * e + a];
        }
    }
    const auto t1 = std::chrono::steady_clock::now();

    // ---- device upload ----
    int rc;
    size_t bytes = 0;
    TAL_CK(cudaMalloc((void **)&h->nodebuf, sizeof(double) * 9 * std::max<int64_t>(n_nodes, 1)));
    TAL_CK(cudaMalloc((void **)&h->staging, sizeof(double) * 3 * std::max<int64_t>(n_nodes, 1)));
    bytes += sizeof(double) * 12 * n_nodes;
    TAL_CK(cudaMemset(h->nodebuf, 0, sizeof(double) * 9 * std::max<int64_t>(n_nodes, 1)));
    {
        std::vector<double> rec((size_t)(6 * n_nodes), 0.0);  // x y z (u = 0 until set)
        for (int64_t i = 0; i < n_nodes; ++i)
            for (int c = 0; c < 3; ++c)
                rec[6 * i + c] = xin[3 * i + c];
        if (n_nodes)
            TAL_CK(cudaMemcpy(h->nodebuf, rec.data(), sizeof(double) * 6 * n_nodes, cudaMemcpyHostToDevice));
    }
    if (renum) {
        if ((rc = dev_upload(&h->perm, perm.data(), perm.size())))
            return rc;
        if ((rc = dev_upload(&h->iperm, iperm.data(), iperm.size())))
            return rc;
        bytes += 8 * n_nodes;
        h->h_iperm.swap(iperm);
    }
    if ((rc = dev_upload(&h->conn, (const int4 *)cord.data(), (size_t)n_elems)))
        return rc;
    bytes += 16 * n_elems;
    if (!ccol.empty()) {
        if ((rc = dev_upload(&h->conn_col, (const int4 *)ccol.data(), (size_t)n_elems)))
            return rc;
        bytes += 16 * n_elems;
    }
    const Chunking &C = h->ch;
    if ((rc = dev_upload(&h->d_blobs, blobs.data(), blobs.size())))
        return rc;
    h->blob_bytes = (int64_t)blobs.size();
    if ((rc = dev_upload(&h->d_blob_off, blob_off.data(), blob_off.size())))
        return rc;
    if ((rc = dev_upload(&h->d_bnd_nodes, C.bnd_nodes.data(), C.bnd_nodes.size())))
        return rc;
    if ((rc = dev_upload(&h->d_bnd_off, C.bnd_off.data(), C.bnd_off.size())))
        return rc;
    if ((rc = dev_upload(&h->d_bnd_pos, C.bnd_pos.data(), C.bnd_pos.size())))
        return rc;
    if (!C.cnodes.empty())
        TAL_CK(cudaMalloc((void **)&h->d_partial, sizeof(double) * 3 * C.cnodes.size()));
    bytes += blobs.size() + blob_off.size() * 4 + C.cnodes.size() * 24 +
             (C.bnd_nodes.size() + C.bnd_off.size() + C.bnd_pos.size()) * 4;
    if ((rc = set_kernel_attrs(h->device, h->priv_cfg, h->priv_grid_ext)))
        return rc;
    TAL_CK(cudaDeviceSynchronize());

    h->h_eperm.swap(eperm);
    h->has_mesh = true;
    h->info.n_nodes = n_nodes;
    h->info.n_elems = n_elems;
    h->info.n_colors = col.empty() ? 0 : ncol;
    h->info.n_chunks = (int64_t)C.chunks.size() / 5;
    h->info.n_chunk_nodes = (int64_t)C.cnodes.size();
    h->info.n_shared_nodes = C.n_shared;
    h->info.device_bytes = (int64_t)bytes;
    h->info.prep_seconds = std::chrono::duration<double>(t1 - t0).count();
    return TAL_OK;
    TAL_GUARD_END
}

int tal_layout_bank_stats(int64_t out[6])
{
    TAL_GUARD_BEGIN
    if (!out)
        return fail(TAL_EINVAL, "out is NULL");
    bank_stats(out, out + 1, out + 2);
    pos_stats(out + 3, out + 4, out + 5);
    return TAL_OK;
    TAL_GUARD_END
}

int tal_plan_blobs(const double *coords, const int64_t *conn, int64_t n_nodes, int64_t n_elems,
                   const tal_mesh_opts *opts_in, int64_t sizes[4], uint8_t *blobs, int32_t *blob_off,
                   int32_t *perm)
{
    TAL_GUARD_BEGIN
    if (!sizes || n_nodes < 0 || n_elems < 0 || (n_nodes && !coords) || (n_elems && !conn))
        return fail(TAL_EINVAL, "bad arguments");
    if (n_nodes >= (int64_t)1 << 31 || n_elems >= (int64_t)1 << 31)
        return fail(TAL_EINVAL, "meshes are limited to 2^31-1 nodes/elements per device");
    for (int64_t i = 0; i < 4 * n_elems; ++i)
        if (conn[i] < 0 || conn[i] >= n_nodes)
            return fail(TAL_EINVAL, "connectivity index out of range [0, n_nodes)");
    tal_mesh_opts opts;
    tal_default_mesh_opts(&opts);
    if (opts_in)
        opts = *opts_in;
    HostLayout L;
    if (int rc = host_layout(coords, conn, n_nodes, n_elems, opts, nullptr, 0, L))
        return rc;
    std::vector<uint8_t> b;
    std::vector<int32_t> off;
    const int T = cfg_threads(L.cfg);
    pack_blobs(L.ch, T, b, off);
    sizes[0] = (int64_t)b.size();
    sizes[1] = (int64_t)off.size();
    sizes[2] = T;
    sizes[3] = L.perm.empty() ? 0 : n_nodes;
    if (blobs)
        std::memcpy(blobs, b.data(), b.size());
    if (blob_off)
        std::memcpy(blob_off, off.data(), 4 * off.size());
    if (perm && !L.perm.empty())
        std::memcpy(perm, L.perm.data(), 4 * L.perm.size());
    return TAL_OK;
    TAL_GUARD_END
}

int tal_plan_layout(const double *coords, const int64_t *conn, int64_t n_nodes, int64_t n_elems,
                    const tal_mesh_opts *opts_in, tal_mesh_info *out)
{
    TAL_GUARD_BEGIN
    if (!out || n_nodes < 0 || n_elems < 0 || (n_nodes && !coords) || (n_elems && !conn))
        return fail(TAL_EINVAL, "bad arguments");
    if (n_nodes >= (int64_t)1 << 31 || n_elems >= (int64_t)1 << 31)
        return fail(TAL_EINVAL, "meshes are limited to 2^31-1 nodes/elements per device");
    for (int64_t i = 0; i < 4 * n_elems; ++i)
        if (conn[i] < 0 || conn[i] >= n_nodes)
            return fail(TAL_EINVAL, "connectivity index out of range [0, n_nodes)");
    tal_mesh_opts opts;
    tal_default_mesh_opts(&opts);
    if (opts_in)
        opts = *opts_in;
    const auto t0 = std::chrono::steady_clock::now();
    HostLayout L;
    if (int rc = host_layout(coords, conn, n_nodes, n_elems, opts, nullptr, 0, L))
        return rc;
    *out = tal_mesh_info{};
    out->n_nodes = n_nodes;
    out->n_elems = n_elems;
    out->n_patches = L.patches.n_patches();
    out->n_chunks = (int64_t)L.ch.chunks.size() / 5;
    out->n_chunk_nodes = (int64_t)L.ch.cnodes.size();
    out->n_shared_nodes = L.ch.n_shared;
    out->prep_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return TAL_OK;
    TAL_GUARD_END
}

int tal_mesh_info_get(tal_handle *h, tal_mesh_info *out)
{
    TAL_GUARD_BEGIN
    if (!h || !out)
        return fail(TAL_EINVAL, "NULL argument");
    if (!h->has_mesh)
        return fail(TAL_ESTATE, "no mesh uploaded");
    *out = h->info;
    return TAL_OK;
    TAL_GUARD_END
}

int tal_buffers_get(tal_handle *h, tal_buffers *out)
{
    TAL_GUARD_BEGIN
    if (!h || !out)
        return fail(TAL_EINVAL, "NULL argument");
    if (!h->has_mesh)
        return fail(TAL_ESTATE, "no mesh uploaded");
    out->ux = h->REC() + 3;
    out->uy = h->REC() + 4;
    out->uz = h->REC() + 5;
    out->u_stride = 6;
    out->rx = h->RX();
    out->ry = h->RY();
    out->rz = h->RZ();
    out->perm = h->perm;
    out->iperm = h->iperm;
    return TAL_OK;
    TAL_GUARD_END
}

int tal_set_velocity_device(tal_handle *h, const double *d_u, void *stream)
{
    TAL_GUARD_BEGIN
    if (!h || (!d_u && h->N))
        return fail(TAL_EINVAL, "NULL argument");
    if (!h->has_mesh)
        return fail(TAL_ESTATE, "no mesh uploaded");
    DeviceGuard g(h->device);
    cudaStream_t s = stream ? (cudaStream_t)stream : h->stream;
    if (h->N) {
        k_pack_velocity<<<grid_for(h->N, 256), 256, 0, s>>>(d_u, h->perm, h->N, h->REC());
        TAL_CK_LAUNCH();
    }
    return TAL_OK;
    TAL_GUARD_END
}

int tal_set_pressure_device(tal_handle *h, const double *d_p, void *stream)
{
    TAL_GUARD_BEGIN
    if (!h)
        return fail(TAL_EINVAL, "handle is NULL");
    if (!h->has_mesh)
        return fail(TAL_ESTATE, "no mesh uploaded");
    DeviceGuard g(h->device);
    if (!d_p) {
        h->has_press = false;
        return TAL_OK;
    }
    cudaStream_t s = stream ? (cudaStream_t)stream : h->stream;
    if (!h->d_press)
        TAL_CK(cudaMalloc((void **)&h->d_press, sizeof(double) * std::max<int64_t>(h->N, 1)));
    if (h->N) {
        k_pack_scalar<<<grid_for(h->N, 256), 256, 0, s>>>(d_p, h->perm, h->N, h->d_press);
        TAL_CK_LAUNCH();
    }
    h->has_press = true;
    return TAL_OK;
    TAL_GUARD_END
}

int tal_set_stabilization(tal_handle *h, int enable, double c1, double c2)
{
    TAL_GUARD_BEGIN
    if (!h)
        return fail(TAL_EINVAL, "handle is NULL");
    if (enable && !(c1 > 0.0 && std::isfinite(c1) && c2 >= 0.0 && std::isfinite(c2)))
        return fail(TAL_EINVAL, "SUPG constants need c1 > 0 and c2 >= 0 (finite)");
    h->has_st = enable != 0;
    if (enable)
        h->st_c1 = c1, h->st_c2 = c2;
    if (h->gexec) {  // a captured step no longer matches the handle state: capture again
        cudaGraphExecDestroy(h->gexec);
        h->gexec = nullptr;
    }
    return TAL_OK;
    TAL_GUARD_END
}

int tal_set_pressure_host(tal_handle *h, const double *p, void *stream)
{
    TAL_GUARD_BEGIN
    if (!h)
        return fail(TAL_EINVAL, "handle is NULL");
    if (!h->has_mesh)
        return fail(TAL_ESTATE, "no mesh uploaded");
    if (!p)
        return tal_set_pressure_device(h, nullptr, stream);
    DeviceGuard g(h->device);
    cudaStream_t s = stream ? (cudaStream_t)stream : h->stream;
    // the staging buffer (3N doubles) is free between calls on this stream
    if (h->N)
        TAL_CK(cudaMemcpyAsync(h->staging, p, sizeof(double) * h->N, cudaMemcpyHostToDevice, s));
    int rc = tal_set_pressure_device(h, h->staging, s);
    if (rc == TAL_OK)
        TAL_CK(cudaStreamSynchronize(s));  // staging is reused by the next host call
    return rc;
    TAL_GUARD_END
}

int tal_set_velocity_host(tal_handle *h, const double *u, void *stream)
{
    TAL_GUARD_BEGIN
    if (!h || (!u && h->N))
        return fail(TAL_EINVAL, "NULL argument");
    if (!h->has_mesh)
        return fail(TAL_ESTATE, "no mesh uploaded");
    DeviceGuard g(h->device);
    cudaStream_t s = stream ? (cudaStream_t)stream : h->stream;
    if (h->N)
        TAL_CK(cudaMemcpyAsync(h->staging, u, sizeof(double) * 3 * h->N, cudaMemcpyHostToDevice, s));
    return tal_set_velocity_device(h, h->staging, s);
    TAL_GUARD_END
}

int tal_run(tal_handle *h, const tal_params *p, int scatter, void *stream, int64_t *kernel_launches)
{
    TAL_GUARD_BEGIN
    if (!h)
        return fail(TAL_EINVAL, "handle is NULL");
    if (!h->has_mesh)
        return fail(TAL_ESTATE, "no mesh uploaded");
    int rc = check_params(p);
    if (rc)
        return rc;
    DeviceGuard g(h->device);
    return launch_run(h, p, scatter, stream ? (cudaStream_t)stream : h->stream, kernel_launches);
    TAL_GUARD_END
}

int tal_run_variant(tal_handle *h, const tal_params *p, int variant, int scatter, void *stream,
                    int64_t *kernel_launches)
{
    TAL_GUARD_BEGIN
    if (!h)
        return fail(TAL_EINVAL, "handle is NULL");
    if (!h->has_mesh)
        return fail(TAL_ESTATE, "no mesh uploaded");
    int rc = check_params(p);
    if (rc)
        return rc;
    DeviceGuard g(h->device);
    return launch_any(h, p, variant, scatter, stream ? (cudaStream_t)stream : h->stream, kernel_launches);
    TAL_GUARD_END
}

int tal_graph_capture(tal_handle *h, const tal_params *p, int variant, int scatter)
{
    TAL_GUARD_BEGIN
    if (!h)
        return fail(TAL_EINVAL, "handle is NULL");
    if (!h->has_mesh)
        return fail(TAL_ESTATE, "no mesh uploaded");
    int rc = check_params(p);
    if (rc)
        return rc;
    DeviceGuard g(h->device);
    h->free_graph();
    TAL_CK(cudaStreamSynchronize(h->stream));
    // lazily built tables (allocation + copies) cannot happen inside a capture
    if (scatter == TAL_SCATTER_SEQUENTIAL && h->N && !h->d_seq_off)
        if ((rc = build_sequential(h)))
            return rc;
    TAL_CK(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    const bool prof = h->prof_on;
    h->prof_on = false;  // the profile event ring is per call, not per replay
    int64_t nl = 0;
    rc = launch_any(h, p, variant, scatter, h->stream, &nl);
    h->prof_on = prof;
    cudaGraph_t graph = nullptr;
    const cudaError_t ce = cudaStreamEndCapture(h->stream, &graph);
    if (rc == TAL_OK && ce != cudaSuccess)
        rc = fail(TAL_ECUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(ce));
    if (rc == TAL_OK) {
        const cudaError_t ie = cudaGraphInstantiate(&h->gexec, graph, 0);
        if (ie != cudaSuccess) {
            h->gexec = nullptr;
            rc = fail(TAL_ECUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ie));
        }
    }
    if (graph)
        cudaGraphDestroy(graph);
    cudaGetLastError();
    h->g_launches = rc == TAL_OK ? nl : 0;
    return rc;
    TAL_GUARD_END
}

int tal_graph_launch(tal_handle *h, void *stream, int64_t *kernel_launches)
{
    TAL_GUARD_BEGIN
    if (!h)
        return fail(TAL_EINVAL, "handle is NULL");
    if (!h->gexec)
        return fail(TAL_ESTATE, "no captured graph (tal_graph_capture)");
    DeviceGuard g(h->device);
    TAL_CK(cudaGraphLaunch(h->gexec, stream ? (cudaStream_t)stream : h->stream));
    if (kernel_launches)
        *kernel_launches = h->g_launches;
    return TAL_OK;
    TAL_GUARD_END
}

int tal_graph_destroy(tal_handle *h)
{
    TAL_GUARD_BEGIN
    if (!h)
        return fail(TAL_EINVAL, "handle is NULL");
    DeviceGuard g(h->device);
    h->free_graph();
    return TAL_OK;
    TAL_GUARD_END
}

int tal_run_caller(tal_handle *h, const tal_params *p, int scatter, const double *d_u, double *d_rhs, void *stream,
                   int64_t *kernel_launches)
{
    TAL_GUARD_BEGIN
    if (!h || ((!d_u || !d_rhs) && h->N))
        return fail(TAL_EINVAL, "NULL argument");
    if (!h->has_mesh)
        return fail(TAL_ESTATE, "no mesh uploaded");
    if (int rc = check_params(p))
        return rc;
    DeviceGuard g(h->device);
    int64_t nl = 0;
    const int rc = launch_caller(h, p, scatter, d_u, d_rhs, stream ? (cudaStream_t)stream : h->stream, &nl);
    if (kernel_launches)
        *kernel_launches = nl;
    return rc;
    TAL_GUARD_END
}

int tal_get_rhs_device(tal_handle *h, double *d_rhs, void *stream)
{
    TAL_GUARD_BEGIN
    if (!h || (!d_rhs && h->N))
        return fail(TAL_EINVAL, "NULL argument");
    if (!h->has_mesh)
        return fail(TAL_ESTATE, "no mesh uploaded");
    DeviceGuard g(h->device);
    cudaStream_t s = stream ? (cudaStream_t)stream : h->stream;
    if (h->N) {
        k_unpack_aos<<<grid_for(h->N, 256), 256, 0, s>>>(h->RX(), h->RY(), h->RZ(), h->iperm, h->N, d_rhs);
        TAL_CK_LAUNCH();
    }
    return TAL_OK;
    TAL_GUARD_END
}

int tal_get_rhs_host(tal_handle *h, double *rhs, void *stream)
{
    TAL_GUARD_BEGIN
    if (!h || (!rhs && h->N))
        return fail(TAL_EINVAL, "NULL argument");
    if (!h->has_mesh)
        return fail(TAL_ESTATE, "no mesh uploaded");
    DeviceGuard g(h->device);
    cudaStream_t s = stream ? (cudaStream_t)stream : h->stream;
    int rc = tal_get_rhs_device(h, h->staging, s);
    if (rc)
        return rc;
    if (h->N)
        TAL_CK(cudaMemcpyAsync(rhs, h->staging, sizeof(double) * 3 * h->N, cudaMemcpyDeviceToHost, s));
    // blocking: rhs is complete on return, even if it is page-locked (the
    // copy would otherwise still be in flight), and the shared staging
    // buffer is free for the next host call on any stream
    TAL_CK(cudaStreamSynchronize(s));
    return TAL_OK;
    TAL_GUARD_END
}

int tal_synchronize(tal_handle *h, void *stream)
{
    TAL_GUARD_BEGIN
    if (!h)
        return fail(TAL_EINVAL, "handle is NULL");
    DeviceGuard g(h->device);
    TAL_CK(cudaStreamSynchronize(stream ? (cudaStream_t)stream : h->stream));
    return TAL_OK;
    TAL_GUARD_END
}

int tal_assemble_async(tal_handle *h, const double *u, const tal_params *p, double *rhs, int scatter,
                       int64_t *ticket)
{
    TAL_GUARD_BEGIN
    if (!h || !ticket)
        return fail(TAL_EINVAL, "NULL argument");
    if (!h->has_mesh)
        return fail(TAL_ESTATE, "no mesh uploaded");
    if (h->N && (!u || !rhs))
        return fail(TAL_EINVAL, "NULL field arrays");
    int rc = check_params(p);
    if (rc)
        return rc;
    DeviceGuard g(h->device);
    constexpr int NS = tal_handle::ASYNC_SLOTS;
    const int64_t n = h->async_next;
    const int s = (int)(n % NS);
    const size_t nb = sizeof(double) * 3 * (size_t)h->N;
    if (nb && !h->astage_u[s]) {
        TAL_CK(cudaMalloc((void **)&h->astage_u[s], nb));
        TAL_CK(cudaMalloc((void **)&h->astage_r[s], nb));
    }
    // slot s was last used by ticket n-NS: its device staging must be free
    if (n >= NS)
        TAL_CK(cudaEventSynchronize(h->ev_d2h[s]));
    if (n >= NS)
        TAL_CK(cudaStreamWaitEvent(h->s_h2d, h->ev_comp[s], 0));  // staging_u[s] consumed
    if (nb)
        TAL_CK(cudaMemcpyAsync(h->astage_u[s], u, nb, cudaMemcpyHostToDevice, h->s_h2d));
    TAL_CK(cudaEventRecord(h->ev_h2d[s], h->s_h2d));
    TAL_CK(cudaStreamWaitEvent(h->stream, h->ev_h2d[s], 0));
    if ((rc = tal_set_velocity_device(h, h->astage_u[s], h->stream)))
        return rc;
    if ((rc = launch_run(h, p, scatter, h->stream, nullptr)))
        return rc;
    if (n >= NS)
        TAL_CK(cudaStreamWaitEvent(h->stream, h->ev_d2h[s], 0));  // staging_r[s] drained
    if ((rc = tal_get_rhs_device(h, h->astage_r[s], h->stream)))
        return rc;
    TAL_CK(cudaEventRecord(h->ev_comp[s], h->stream));
    TAL_CK(cudaStreamWaitEvent(h->s_d2h, h->ev_comp[s], 0));
    if (nb)
        TAL_CK(cudaMemcpyAsync(rhs, h->astage_r[s], nb, cudaMemcpyDeviceToHost, h->s_d2h));
    TAL_CK(cudaEventRecord(h->ev_d2h[s], h->s_d2h));
    *ticket = n;
    h->async_next = n + 1;
    return TAL_OK;
    TAL_GUARD_END
}

int tal_wait(tal_handle *h, int64_t ticket)
{
    TAL_GUARD_BEGIN
    if (!h)
        return fail(TAL_EINVAL, "handle is NULL");
    if (ticket < 0 || ticket >= h->async_next)
        return fail(TAL_EINVAL, "unknown ticket");
    if (ticket < h->async_next - tal_handle::ASYNC_SLOTS)
        return TAL_OK;  // its slot was reused, so it completed already
    DeviceGuard g(h->device);
    TAL_CK(cudaEventSynchronize(h->ev_d2h[ticket % tal_handle::ASYNC_SLOTS]));
    return TAL_OK;
    TAL_GUARD_END
}

int tal_assemble(tal_handle *h, const double *u, const tal_params *p, double *rhs, int scatter,
                 tal_timings *t)
{
    TAL_GUARD_BEGIN
    return tal_assemble_variant(h, u, p, rhs, TAL_VARIANT_RSP, scatter, t);
    TAL_GUARD_END
}

int tal_assemble_variant(tal_handle *h, const double *u, const tal_params *p, double *rhs, int variant,
                         int scatter, tal_timings *t)
{
    TAL_GUARD_BEGIN
    if (!h)
        return fail(TAL_EINVAL, "handle is NULL");
    if (!h->has_mesh)
        return fail(TAL_ESTATE, "no mesh uploaded");
    if (h->N && (!u || !rhs))
        return fail(TAL_EINVAL, "NULL field arrays");
    int rc = check_params(p);
    if (rc)
        return rc;
    DeviceGuard g(h->device);
    cudaStream_t s = h->stream;
    const size_t nb = sizeof(double) * 3 * (size_t)h->N;
    int64_t nl = 0;
    TAL_CK(cudaEventRecord(h->ev[0], s));
    if (nb)
        TAL_CK(cudaMemcpyAsync(h->staging, u, nb, cudaMemcpyHostToDevice, s));
    TAL_CK(cudaEventRecord(h->ev[1], s));
    if ((rc = tal_set_velocity_device(h, h->staging, s)))
        return rc;
    nl += h->N ? 1 : 0;
    TAL_CK(cudaEventRecord(h->ev[2], s));
    int64_t nrun = 0;
    if ((rc = launch_any(h, p, variant, scatter, s, &nrun)))
        return rc;
    nl += nrun;
    TAL_CK(cudaEventRecord(h->ev[3], s));
    if ((rc = tal_get_rhs_device(h, h->staging, s)))
        return rc;
    nl += h->N ? 1 : 0;
    TAL_CK(cudaEventRecord(h->ev[4], s));
    if (nb)
        TAL_CK(cudaMemcpyAsync(rhs, h->staging, nb, cudaMemcpyDeviceToHost, s));
    TAL_CK(cudaEventRecord(h->ev[5], s));
    TAL_CK(cudaEventSynchronize(h->ev[5]));
    float ms[5];
    for (int i = 0; i < 5; ++i)
        TAL_CK(cudaEventElapsedTime(&ms[i], h->ev[i], h->ev[i + 1]));
    tal_timings tt;
    tt.h2d_ms = ms[0];
    tt.pack_ms = ms[1];
    tt.kernel_ms = ms[2];
    tt.unpack_ms = ms[3];
    tt.d2h_ms = ms[4];
    float tot = 0.f;
    TAL_CK(cudaEventElapsedTime(&tot, h->ev[0], h->ev[5]));
    tt.total_ms = tot;
    tt.kernel_launches = nl;
    h->last = tt;
    if (t)
        *t = tt;
    return TAL_OK;
    TAL_GUARD_END
}

namespace {
// the strict numba seam (_rsp_kernels.py:20-164), tal_strict.cuh: each node
// continues from its incoming rhs value through its elements in ids order
// with the reference's operation order -- bitwise the numba loop.  Transient
// upload (a parity/debug path; the fast seam is tal_seam_* below).
int seam_impl(int device, const double *coords, const int64_t *conn, int64_t n_nodes, int64_t n_elems,
              const double *u, double rho, double mu, double cvre, const double *pmat, const int64_t *ids,
              int64_t k, double *rhs)
{
    if (n_nodes < 0 || n_elems < 0 || k < 0)
        return fail(TAL_EINVAL, "negative sizes");
    if (k == 0 || n_nodes == 0)
        return TAL_OK;
    if (!coords || !conn || !u || !pmat || !ids || !rhs)
        return fail(TAL_EINVAL, "NULL arrays");
    if (n_nodes >= (int64_t)1 << 31)
        return fail(TAL_EINVAL, "too many nodes");
    std::vector<int32_t> sub((size_t)(4 * k));
    for (int64_t t = 0; t < k; ++t) {
        if (ids[t] < 0 || ids[t] >= n_elems)
            return fail(TAL_EINVAL, "element id out of range");
        for (int a = 0; a < 4; ++a) {
            const int64_t v = conn[4 * ids[t] + a];
            if (v < 0 || v >= n_nodes)
                return fail(TAL_EINVAL, "connectivity index out of range [0, n_nodes)");
            sub[4 * t + a] = (int32_t)v;
        }
    }
    tal_params p;
    p.rho = rho;
    p.mu = mu;
    p.c_vreman = cvre;
    std::memcpy(p.pmat, pmat, sizeof p.pmat);
    int rc = check_params(&p);
    if (rc)
        return rc;
    ElemConsts kc;
    bool sym;
    make_consts(&p, kc, sym);
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        return fail(TAL_ECUDA, "no CUDA device available; the assembly has no CPU fallback");
    if (device < 0 || device >= n)
        return fail(TAL_EINVAL, "device index out of range");
    DeviceGuard g(device);
    std::vector<double> soa((size_t)(6 * n_nodes));
    for (int64_t i = 0; i < n_nodes; ++i)
        for (int c = 0; c < 3; ++c) {
            soa[6 * i + c] = coords[3 * i + c];  // node records x y z ux uy uz
            soa[6 * i + 3 + c] = u[3 * i + c];
        }
    // strict: incoming rhs as SoA start values; node -> (entry t, corner) in
    // ids order; filter width per entry from the host libm (tal_strict.cuh)
    std::vector<double> rin, dlt;
    std::vector<int64_t> off;
    std::vector<int32_t> ent;
    {
        if (4 * k > INT32_MAX)
            return fail(TAL_EINVAL, "strict seam supports up to 2^29 element ids per call");
        rin.resize((size_t)(3 * n_nodes));
        for (int64_t i = 0; i < n_nodes; ++i)
            for (int c = 0; c < 3; ++c)
                rin[c * n_nodes + i] = rhs[3 * i + c];
        off.assign((size_t)n_nodes + 1, 0);
        for (int64_t i = 0; i < 4 * k; ++i)
            off[sub[i] + 1]++;
        for (int64_t v = 0; v < n_nodes; ++v)
            off[v + 1] += off[v];
        std::vector<int64_t> fill(off.begin(), off.end() - 1);
        ent.resize((size_t)(4 * k));
        dlt.resize((size_t)k);
        for (int64_t t = 0; t < k; ++t) {
            for (int a = 0; a < 4; ++a)
                ent[fill[sub[4 * t + a]]++] = (int32_t)(t << 2 | a);
            dlt[t] = filter_width(coords, 3, &sub[4 * t]);
        }
    }
    double *buf = nullptr, *ddlt = nullptr;
    int4 *dconn = nullptr;
    int64_t *doff = nullptr;
    int32_t *dent = nullptr;
    TAL_CK(cudaMalloc((void **)&buf, sizeof(double) * 9 * n_nodes));
    rc = TAL_OK;
    do {
        cudaError_t e;
        if ((e = cudaMalloc((void **)&dconn, sizeof(int4) * k)) != cudaSuccess ||
            (e = cudaMemcpy(buf, soa.data(), sizeof(double) * 6 * n_nodes, cudaMemcpyHostToDevice)) !=
                cudaSuccess ||
            (e = cudaMemcpy(buf + 6 * n_nodes, rin.data(), sizeof(double) * 3 * n_nodes,
                            cudaMemcpyHostToDevice)) != cudaSuccess ||
            (e = cudaMemcpy(dconn, sub.data(), sizeof(int4) * k, cudaMemcpyHostToDevice)) != cudaSuccess) {
            rc = fail(TAL_ECUDA, std::string("assemble_elements upload: ") + cudaGetErrorString(e));
            break;
        }
        if (((e = cudaMalloc((void **)&doff, sizeof(int64_t) * off.size())) != cudaSuccess ||
                       (e = cudaMalloc((void **)&dent, sizeof(int32_t) * ent.size())) != cudaSuccess ||
                       (e = cudaMalloc((void **)&ddlt, sizeof(double) * dlt.size())) != cudaSuccess ||
                       (e = cudaMemcpy(doff, off.data(), sizeof(int64_t) * off.size(),
                                       cudaMemcpyHostToDevice)) != cudaSuccess ||
                       (e = cudaMemcpy(dent, ent.data(), sizeof(int32_t) * ent.size(),
                                       cudaMemcpyHostToDevice)) != cudaSuccess ||
                       (e = cudaMemcpy(ddlt, dlt.data(), sizeof(double) * dlt.size(),
                                       cudaMemcpyHostToDevice)) != cudaSuccess)) {
            rc = fail(TAL_ECUDA, std::string("assemble_elements upload: ") + cudaGetErrorString(e));
            break;
        }
        const double *nodes = buf;
        RhsSoA r{buf + 6 * n_nodes, buf + 7 * n_nodes, buf + 8 * n_nodes};
        k_assemble_sequential<<<grid_for(n_nodes, 128), 128>>>(doff, dent, n_nodes, dconn, nodes, ddlt,
                                                               r.rx, r.ry, r.rz, kc, true);
        if ((e = cudaGetLastError()) != cudaSuccess || (e = cudaDeviceSynchronize()) != cudaSuccess) {
            rc = fail(TAL_ECUDA, std::string("assemble_elements kernel: ") + cudaGetErrorString(e));
            break;
        }
        if ((e = cudaMemcpy(soa.data(), buf + 6 * n_nodes, sizeof(double) * 3 * n_nodes,
                            cudaMemcpyDeviceToHost)) != cudaSuccess) {
            rc = fail(TAL_ECUDA, std::string("assemble_elements download: ") + cudaGetErrorString(e));
            break;
        }
        for (int64_t i = 0; i < n_nodes; ++i)
            for (int c = 0; c < 3; ++c)
                rhs[3 * i + c] = soa[c * n_nodes + i];  // accumulated on the device
    } while (0);
    void *tmp[] = {buf, dconn, doff, dent, ddlt};
    for (void *q : tmp)
        if (q)
            cudaFree(q);
    return rc;
}
}  // namespace

// ---------------------------------------------------------------------------
// The fast numba seam: a per-mesh context (resident mesh on the device in the
// caller's own layout, per-block content fingerprints, pinned staging) so a
// call costs the velocity rows it reads, one kernel and the RHS rows it
// writes.  'ids' = the whole mesh in order (the reference's one-thread
// driver, variants.py:573-576): the private edge-star kernel in caller layout
// (launch_caller); a contiguous range (its threaded slabs, :578-596) or any
// other list: the per-element kernel on the caller-layout arrays.  Only the
// node rows the call's elements reference, [nmin, nmax], cross PCIe and are
// added into the caller's rhs, so T threaded slab calls move ~1/T of the
// arrays each instead of all of them.  The GPU part of the calls on one
// context is serialised (the reference calls the seam from a thread pool);
// id validation and fingerprint checks run outside that lock.
// ---------------------------------------------------------------------------
namespace {
constexpr int64_t SEAM_BLOCK = 1 << 16;  // fingerprint block, bytes
constexpr int64_t SEAM_EBLK = SEAM_BLOCK / 32;  // elements per conn block

// order-fixed 64-bit fingerprint of one block: four independent lanes (the
// multiply chains overlap, so this runs at memory speed)
uint64_t block_hash(const uint8_t *q, int64_t n, uint64_t seed)
{
    uint64_t h[4] = {seed ^ 0x9e3779b97f4a7c15ull, seed ^ 0xc2b2ae3d27d4eb4full, seed ^ 0x165667b19e3779f9ull,
                     seed ^ 0x27d4eb2f165667c5ull};
    int64_t i = 0;
    for (; i + 32 <= n; i += 32) {
        uint64_t w[4];
        std::memcpy(w, q + i, 32);
        for (int l = 0; l < 4; ++l) {
            h[l] = (h[l] ^ w[l]) * 0xff51afd7ed558ccdull;
            h[l] ^= h[l] >> 29;
        }
    }
    for (; i < n; ++i)
        h[0] = (h[0] ^ q[i]) * 0xc4ceb9fe1a85ec53ull;
    uint64_t x = (uint64_t)n;
    for (int l = 0; l < 4; ++l)
        x = (x ^ h[l]) * 0x100000001b3ull + 0x9e3779b97f4a7c15ull;
    return x ^ (x >> 31);
}

int64_t n_blocks(int64_t bytes) { return (bytes + SEAM_BLOCK - 1) / SEAM_BLOCK; }

void hash_blocks(const void *p, int64_t bytes, int64_t b0, int64_t b1, uint64_t *out)
{
    parallel_items(b1 - b0, [&](int64_t i, int) {
        const int64_t b = b0 + i, o = b * SEAM_BLOCK;
        out[i] = block_hash((const uint8_t *)p + o, std::min(SEAM_BLOCK, bytes - o), (uint64_t)b);
    }, 4);
}

// do blocks [b0, b1) of p still hash to ref[b0 .. b1)?
bool blocks_match(const void *p, int64_t bytes, int64_t b0, int64_t b1, const std::vector<uint64_t> &ref)
{
    if (b1 <= b0)
        return true;
    std::vector<uint64_t> h((size_t)(b1 - b0));
    hash_blocks(p, bytes, b0, b1, h.data());
    return std::equal(h.begin(), h.end(), ref.begin() + b0);
}
}  // namespace

struct tal_seam {
    tal_handle *h = nullptr;  // resident mesh (renumbered, edge-star chunks)
    int4 *conn_c = nullptr;   // caller element order, caller node ids
    double *xc = nullptr;     // caller-order coords, u staging, rhs accumulator (N,3)
    double *uc = nullptr, *rc = nullptr;
    int32_t *d_ids = nullptr;
    int64_t ids_cap = 0;
    double *pin_u = nullptr, *pin_r = nullptr;
    int64_t N = 0, E = 0;
    std::vector<uint64_t> hx, hc;     // per-block fingerprints of coords / conn at open
    std::vector<int32_t> bmin, bmax;  // per conn block (SEAM_EBLK elements): node id range
    std::mutex mu;
};

namespace {
void seam_free(tal_seam *c)
{
    if (!c)
        return;
    if (c->h) {
        DeviceGuard g(c->h->device);
        for (void *q : {(void *)c->conn_c, (void *)c->xc, (void *)c->uc, (void *)c->rc, (void *)c->d_ids})
            if (q)
                cudaFree(q);
        if (c->pin_u)
            cudaFreeHost(c->pin_u);
        if (c->pin_r)
            cudaFreeHost(c->pin_r);
        tal_destroy(c->h);
    }
    delete c;
}

int seam_open_impl(int device, const double *coords, const int64_t *conn, int64_t n_nodes, int64_t n_elems,
                   tal_seam **out)
{
    *out = nullptr;
    if (n_nodes < 0 || n_elems < 0 || (n_nodes && !coords) || (n_elems && !conn))
        return fail(TAL_EINVAL, "bad mesh arguments");
    if (n_nodes >= (int64_t)1 << 31 || n_elems >= (int64_t)1 << 31)
        return fail(TAL_EINVAL, "too many nodes / elements");
    std::unique_ptr<tal_seam, void (*)(tal_seam *)> c(new tal_seam(), seam_free);
    c->N = n_nodes, c->E = n_elems;
    // connectivity range check + per-block node ranges (one pass), fingerprints
    const int64_t nbe = (n_elems + SEAM_EBLK - 1) / SEAM_EBLK;
    c->bmin.assign((size_t)nbe, INT32_MAX);
    c->bmax.assign((size_t)nbe, -1);
    std::atomic<bool> bad{false};
    parallel_items(nbe, [&](int64_t b, int) {
        int64_t lo = INT64_MAX, hi = -1;
        for (int64_t i = 4 * b * SEAM_EBLK, e = std::min(4 * n_elems, 4 * (b + 1) * SEAM_EBLK); i < e; ++i) {
            const int64_t v = conn[i];
            lo = std::min(lo, v), hi = std::max(hi, v);
        }
        if (lo < 0 || hi >= n_nodes)
            bad = true;
        else
            c->bmin[b] = (int32_t)lo, c->bmax[b] = (int32_t)hi;
    }, 4);
    if (bad)
        return fail(TAL_EINVAL, "connectivity index out of range [0, n_nodes)");
    const int64_t xb = sizeof(double) * 3 * n_nodes, cb = sizeof(int64_t) * 4 * n_elems;
    c->hx.resize((size_t)n_blocks(xb));
    c->hc.resize((size_t)n_blocks(cb));
    hash_blocks(coords, xb, 0, n_blocks(xb), c->hx.data());
    hash_blocks(conn, cb, 0, n_blocks(cb), c->hc.data());
    if (int rc = tal_create(device, &c->h))
        return rc;
    tal_mesh_opts o;
    tal_default_mesh_opts(&o);
    o.validate = 0;  // the numba seam takes any mesh (no orientation check)
    if (int rc = tal_upload_mesh_ex(c->h, coords, conn, n_nodes, n_elems, nullptr, &o, nullptr, 0))
        return rc;
    DeviceGuard g(device);
    const size_t nb = sizeof(double) * 3 * (size_t)std::max<int64_t>(n_nodes, 1);
    TAL_CK(cudaMallocHost((void **)&c->pin_u, nb));
    TAL_CK(cudaMallocHost((void **)&c->pin_r, nb));
    TAL_CK(cudaMalloc((void **)&c->xc, nb));
    TAL_CK(cudaMalloc((void **)&c->uc, nb));
    TAL_CK(cudaMalloc((void **)&c->rc, nb));
    if (n_nodes)
        TAL_CK(cudaMemcpy(c->xc, coords, sizeof(double) * 3 * n_nodes, cudaMemcpyHostToDevice));
    if (n_elems) {
        std::vector<int4> cc((size_t)n_elems);
        parallel_for(n_elems, [&](int64_t e0, int64_t e1, int) {
            for (int64_t e = e0; e < e1; ++e)
                cc[e] = make_int4((int)conn[4 * e], (int)conn[4 * e + 1], (int)conn[4 * e + 2],
                                  (int)conn[4 * e + 3]);
        });
        TAL_CK(cudaMalloc((void **)&c->conn_c, sizeof(int4) * n_elems));
        TAL_CK(cudaMemcpy(c->conn_c, cc.data(), sizeof(int4) * n_elems, cudaMemcpyHostToDevice));
    }
    *out = c.release();
    return TAL_OK;
}

// The elements of one call: validated ids, contiguous or not, node row range.
struct SeamCall {
    bool whole = false, range = false;
    int64_t a0 = 0, k = 0, nmin = 0, nmax = -1;
    std::vector<int32_t> i32;  // list calls: the ids as int32
};

int seam_plan(const tal_seam *c, const int64_t *ids, int64_t k, SeamCall &sc)
{
    const int64_t E = c->E, a0 = ids[0];
    std::atomic<bool> bad{false}, seq{true};
    parallel_for(k, [&](int64_t t0, int64_t t1, int) {
        for (int64_t t = t0; t < t1; ++t) {
            if (ids[t] < 0 || ids[t] >= E) {
                bad = true;
                return;
            }
            if (ids[t] != a0 + t)
                seq = false;
        }
    });
    if (bad)
        return fail(TAL_EINVAL, "element id out of range");
    sc.a0 = a0, sc.k = k;
    sc.range = seq;
    sc.whole = seq && a0 == 0 && k == E;
    if (seq) {  // node rows from the per-block ranges (conservative at the ends)
        int64_t lo = INT64_MAX, hi = -1;
        for (int64_t b = a0 / SEAM_EBLK; b <= (a0 + k - 1) / SEAM_EBLK; ++b)
            lo = std::min<int64_t>(lo, c->bmin[b]), hi = std::max<int64_t>(hi, c->bmax[b]);
        sc.nmin = lo, sc.nmax = hi;
        return TAL_OK;
    }
    // a list (e.g. one colour class of the coloured driver) spans the mesh:
    // all node rows
    sc.i32.resize((size_t)k);
    parallel_for(k, [&](int64_t t0, int64_t t1, int) {
        for (int64_t t = t0; t < t1; ++t)
            sc.i32[t] = (int32_t)ids[t];
    });
    sc.nmin = 0, sc.nmax = c->N - 1;
    return TAL_OK;
}

// do the mesh arrays still hold what the context was built from, wherever this
// call reads them (its conn rows, the coords rows [nmin, nmax])?
bool seam_fresh(const tal_seam *c, const double *coords, const int64_t *conn, const SeamCall &sc)
{
    const int64_t xb = sizeof(double) * 3 * c->N, cb = sizeof(int64_t) * 4 * c->E;
    if (sc.range) {
        if (!blocks_match(conn, cb, sc.a0 * 32 / SEAM_BLOCK, ((sc.a0 + sc.k) * 32 - 1) / SEAM_BLOCK + 1, c->hc))
            return false;
    } else if (!blocks_match(conn, cb, 0, n_blocks(cb), c->hc)) {
        return false;
    }
    return blocks_match(coords, xb, sc.nmin * 24 / SEAM_BLOCK, ((sc.nmax + 1) * 24 - 1) / SEAM_BLOCK + 1, c->hx);
}

int seam_assemble_impl(tal_seam *c, const double *u, double rho, double mu, double cvre, const double *pmat,
                       const SeamCall &sc, double *rhs)
{
    tal_params p;
    p.rho = rho, p.mu = mu, p.c_vreman = cvre;
    std::memcpy(p.pmat, pmat, sizeof p.pmat);
    if (int rc = check_params(&p))
        return rc;
    ElemConsts kc;
    bool sym;
    make_consts(&p, kc, sym);
    std::lock_guard<std::mutex> lk(c->mu);
    tal_handle *h = c->h;
    DeviceGuard g(h->device);
    cudaStream_t s = h->stream;
    const int64_t r0 = 3 * sc.nmin, n3 = 3 * (sc.nmax - sc.nmin + 1);  // the call's rows, in doubles
    constexpr int64_t PIECE = 1 << 19;                                  // doubles
    cudaPointerAttributes pa_u{};
    const bool u_locked = cudaPointerGetAttributes(&pa_u, u) == cudaSuccess && pa_u.type == cudaMemoryTypeHost;
    cudaGetLastError();
    if (u_locked)  // page-locked (cudaHostRegister / pinned): one DMA
        TAL_CK(cudaMemcpyAsync(c->uc + r0, u + r0, sizeof(double) * n3, cudaMemcpyHostToDevice, s));
    // pageable u -> pinned -> device in 4 MB pieces: the host copy of piece
    // i+1 overlaps the DMA of piece i
    for (int64_t i0 = 0; i0 < n3 && !u_locked; i0 += PIECE) {
        const int64_t i1 = std::min(n3, i0 + PIECE);
        parallel_for(i1 - i0, [&](int64_t a, int64_t b, int) {
            std::memcpy(c->pin_u + r0 + i0 + a, u + r0 + i0 + a, sizeof(double) * (b - a));
        }, 1 << 15);
        TAL_CK(cudaMemcpyAsync(c->uc + r0 + i0, c->pin_u + r0 + i0, sizeof(double) * (i1 - i0),
                               cudaMemcpyHostToDevice, s));
    }
    if (sc.whole) {  // the resident edge-star kernel, caller layout in and out
        int64_t nl = 0;
        if (int rc = launch_caller(h, &p, TAL_SCATTER_PRIVATE_ATOMIC, c->uc, c->rc, s, &nl))
            return rc;
    } else {
        TAL_CK(cudaMemsetAsync(c->rc + r0, 0, sizeof(double) * n3, s));
        const int32_t *d_ids = nullptr;
        if (!sc.range) {
            if (sc.k > c->ids_cap) {
                if (c->d_ids)
                    cudaFree(c->d_ids);
                c->d_ids = nullptr;
                c->ids_cap = 0;
                TAL_CK(cudaMalloc((void **)&c->d_ids, sizeof(int32_t) * sc.k));
                c->ids_cap = sc.k;
            }
            TAL_CK(cudaMemcpyAsync(c->d_ids, sc.i32.data(), sizeof(int32_t) * sc.k, cudaMemcpyHostToDevice, s));
            d_ids = c->d_ids;
        }
        if (sym)
            k_assemble_atomic_caller<true><<<grid_for(sc.k, 256), 256, 0, s>>>(c->conn_c, d_ids, sc.a0, sc.k, c->xc,
                                                                              c->uc, c->rc, kc);
        else
            k_assemble_atomic_caller<false><<<grid_for(sc.k, 256), 256, 0, s>>>(c->conn_c, d_ids, sc.a0, sc.k, c->xc,
                                                                               c->uc, c->rc, kc);
        TAL_CK_LAUNCH();
    }
    // device -> pinned in pieces; piece i is added into rhs while piece i+1 copies
    const int64_t np_ = (n3 + PIECE - 1) / PIECE;
    std::vector<cudaEvent_t> ev((size_t)np_);
    for (auto &e : ev)
        TAL_CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    int rc = TAL_OK;
    for (int64_t q = 0; q < np_; ++q) {
        const int64_t i0 = r0 + q * PIECE, i1 = std::min(r0 + n3, i0 + PIECE);
        if (cudaMemcpyAsync(c->pin_r + i0, c->rc + i0, sizeof(double) * (i1 - i0), cudaMemcpyDeviceToHost, s) !=
                cudaSuccess ||
            cudaEventRecord(ev[q], s) != cudaSuccess) {
            rc = fail(TAL_ECUDA, "seam D2H");
            break;
        }
    }
    for (int64_t q = 0; q < np_ && rc == TAL_OK; ++q) {
        if (cudaEventSynchronize(ev[q]) != cudaSuccess) {
            rc = fail(TAL_ECUDA, "seam D2H sync");
            break;
        }
        const int64_t i0 = r0 + q * PIECE, i1 = std::min(r0 + n3, i0 + PIECE);
        parallel_for(i1 - i0, [&](int64_t a, int64_t b, int) {
            for (int64_t i = i0 + a; i < i0 + b; ++i)
                rhs[i] += c->pin_r[i];
        }, 1 << 15);
    }
    cudaStreamSynchronize(s);
    for (auto &e : ev)
        cudaEventDestroy(e);
    return rc;
}

int seam_call(tal_seam *c, const double *u, double rho, double mu, double cvre,
              const double *pmat, const int64_t *ids, int64_t k, double *rhs)
{
    if (!c || !c->h)
        return fail(TAL_EINVAL, "seam context is NULL");
    if (k < 0)
        return fail(TAL_EINVAL, "negative sizes");
    if (k == 0 || c->N == 0)
        return TAL_OK;
    if (!u || !pmat || !ids || !rhs)
        return fail(TAL_EINVAL, "NULL arrays");
    SeamCall sc;
    if (int rc = seam_plan(c, ids, k, sc))
        return rc;
    return seam_assemble_impl(c, u, rho, mu, cvre, pmat, sc, rhs);
}

// stateless entry: a small cache of contexts keyed by the mesh arrays'
// addresses and sizes; every call re-checks the fingerprints of the blocks it
// reads (its conn rows, its coords rows), so a changed array is never served
// stale -- the context is rebuilt instead
struct SeamKey {
    int device;
    const void *coords, *conn;
    int64_t N, E;
    bool operator==(const SeamKey &o) const
    {
        return device == o.device && coords == o.coords && conn == o.conn && N == o.N && E == o.E;
    }
};
std::mutex g_seam_mu;
std::vector<std::pair<SeamKey, std::shared_ptr<tal_seam>>> g_seams;  // most recent last, at most 2

std::shared_ptr<tal_seam> seam_lookup(const SeamKey &key, const tal_seam *stale, int &rc)
{
    std::lock_guard<std::mutex> lk(g_seam_mu);
    for (size_t i = 0; i < g_seams.size(); ++i)
        if (g_seams[i].first == key) {
            if (g_seams[i].second.get() == stale) {  // rebuild from the current contents
                g_seams.erase(g_seams.begin() + i);
                break;
            }
            auto c = g_seams[i].second;
            std::rotate(g_seams.begin() + i, g_seams.begin() + i + 1, g_seams.end());
            return c;
        }
    tal_seam *raw = nullptr;
    rc = seam_open_impl(key.device, (const double *)key.coords, (const int64_t *)key.conn, key.N, key.E, &raw);
    if (rc)
        return nullptr;
    std::shared_ptr<tal_seam> c(raw, seam_free);
    g_seams.push_back({key, c});
    if (g_seams.size() > 2)
        g_seams.erase(g_seams.begin());  // freed when its last in-flight call ends
    return c;
}
}  // namespace

int tal_seam_open(int device, const double *coords, const int64_t *conn, int64_t n_nodes, int64_t n_elems,
                  tal_seam **out)
{
    TAL_GUARD_BEGIN
    if (!out)
        return fail(TAL_EINVAL, "out is NULL");
    return seam_open_impl(device, coords, conn, n_nodes, n_elems, out);
    TAL_GUARD_END
}

int tal_seam_assemble(tal_seam *ctx, const double *u, double rho, double mu, double cvre, const double *pmat,
                      const int64_t *ids, int64_t k, double *rhs)
{
    TAL_GUARD_BEGIN
    // the mesh is the caller's contract here (unchanged since tal_seam_open)
    return seam_call(ctx, u, rho, mu, cvre, pmat, ids, k, rhs);
    TAL_GUARD_END
}

int tal_seam_close(tal_seam *ctx)
{
    TAL_GUARD_BEGIN
    seam_free(ctx);
    return TAL_OK;
    TAL_GUARD_END
}

int tal_assemble_elements(int device, const double *coords, const int64_t *conn, int64_t n_nodes,
                          int64_t n_elems, const double *u, double rho, double mu, double cvre,
                          const double *pmat, const int64_t *ids, int64_t k, double *rhs)
{
    TAL_GUARD_BEGIN
    if (n_nodes < 0 || n_elems < 0 || k < 0)
        return fail(TAL_EINVAL, "negative sizes");
    if (k == 0 || n_nodes == 0)
        return TAL_OK;
    if (!coords || !conn || !u || !pmat || !ids || !rhs)
        return fail(TAL_EINVAL, "NULL arrays");
    if (n_nodes >= (int64_t)1 << 31 || n_elems >= (int64_t)1 << 31)
        return fail(TAL_EINVAL, "too many nodes / elements");
    const SeamKey key{device, coords, conn, n_nodes, n_elems};
    const tal_seam *stale = nullptr;
    for (int attempt = 0; attempt < 2; ++attempt) {
        int rc = TAL_OK;
        std::shared_ptr<tal_seam> c = seam_lookup(key, stale, rc);
        if (!c)
            return rc;
        SeamCall sc;
        if ((rc = seam_plan(c.get(), ids, k, sc)))
            return rc;
        if (!seam_fresh(c.get(), coords, conn, sc)) {
            stale = c.get();  // the mesh changed under this key: rebuild once
            continue;
        }
        return seam_assemble_impl(c.get(), u, rho, mu, cvre, pmat, sc, rhs);
    }
    return fail(TAL_ESTATE, "mesh arrays changed while assembling");
    TAL_GUARD_END
}

int tal_assemble_elements_strict(int device, const double *coords, const int64_t *conn, int64_t n_nodes,
                                 int64_t n_elems, const double *u, double rho, double mu, double cvre,
                                 const double *pmat, const int64_t *ids, int64_t k, double *rhs)
{
    TAL_GUARD_BEGIN
    return seam_impl(device, coords, conn, n_nodes, n_elems, u, rho, mu, cvre, pmat, ids, k, rhs);
    TAL_GUARD_END
}

int tal_halo_pack(tal_handle *h, const int32_t *d_list, int64_t n, double *d_out, void *stream)
{
    TAL_GUARD_BEGIN
    if (!h || n < 0 || (n && (!d_list || !d_out)))
        return fail(TAL_EINVAL, "bad arguments");
    if (!h->has_mesh)
        return fail(TAL_ESTATE, "no mesh uploaded");
    if (!n)
        return TAL_OK;
    DeviceGuard g(h->device);
    cudaStream_t s = stream ? (cudaStream_t)stream : h->stream;
    k_halo_pack<<<grid_for(n, 256), 256, 0, s>>>(d_list, n, h->RX(), h->RY(), h->RZ(), d_out);
    TAL_CK_LAUNCH();
    return TAL_OK;
    TAL_GUARD_END
}

int tal_halo_accumulate(tal_handle *h, const int32_t *d_list, int64_t n, const double *d_in, void *stream)
{
    TAL_GUARD_BEGIN
    if (!h || n < 0 || (n && (!d_list || !d_in)))
        return fail(TAL_EINVAL, "bad arguments");
    if (!h->has_mesh)
        return fail(TAL_ESTATE, "no mesh uploaded");
    if (!n)
        return TAL_OK;
    DeviceGuard g(h->device);
    cudaStream_t s = stream ? (cudaStream_t)stream : h->stream;
    k_halo_accumulate<<<grid_for(n, 256), 256, 0, s>>>(d_list, n, d_in, h->RX(), h->RY(), h->RZ());
    TAL_CK_LAUNCH();
    return TAL_OK;
    TAL_GUARD_END
}

int tal_map_nodes(tal_handle *h, const int64_t *caller_ids, int64_t n, int32_t *internal_ids)
{
    TAL_GUARD_BEGIN
    if (!h || n < 0 || (n && (!caller_ids || !internal_ids)))
        return fail(TAL_EINVAL, "bad arguments");
    if (!h->has_mesh)
        return fail(TAL_ESTATE, "no mesh uploaded");
    for (int64_t i = 0; i < n; ++i) {
        const int64_t v = caller_ids[i];
        if (v < 0 || v >= h->N)
            return fail(TAL_EINVAL, "node id out of range");
        internal_ids[i] = h->h_iperm.empty() ? (int32_t)v : h->h_iperm[v];
    }
    return TAL_OK;
    TAL_GUARD_END
}

int tal_box_mesh(int64_t nx, int64_t ny, int64_t nz, double ex, double ey, double ez, double *coords,
                 int64_t *conn)
{
    TAL_GUARD_BEGIN
    if (nx < 1 || ny < 1 || nz < 1)
        return fail(TAL_EINVAL, "box dimensions must be positive");
    if (!(ex > 0.0 && ey > 0.0 && ez > 0.0))
        return fail(TAL_EINVAL, "extents must be 3 positive lengths");
    if (!coords || !conn)
        return fail(TAL_EINVAL, "NULL output arrays");
    box_mesh(nx, ny, nz, ex, ey, ez, coords, conn);
    return TAL_OK;
    TAL_GUARD_END
}

int tal_signed_volumes(const double *coords, const int64_t *conn, int64_t n_elems, double *vols)
{
    TAL_GUARD_BEGIN
    if (n_elems < 0 || (n_elems && (!coords || !conn || !vols)))
        return fail(TAL_EINVAL, "bad arguments");
    signed_volumes(coords, conn, n_elems, vols);
    return TAL_OK;
    TAL_GUARD_END
}

int tal_color_elements(const int64_t *conn, int64_t n_nodes, int64_t n_elems, int64_t *colors,
                       int64_t *n_colors)
{
    TAL_GUARD_BEGIN
    if (n_elems < 0 || n_nodes < 0 || (n_elems && (!conn || !colors)) || !n_colors)
        return fail(TAL_EINVAL, "bad arguments");
    const int64_t nc = color_elements(conn, n_nodes, n_elems, colors);
    if (nc < 0)
        return fail(TAL_EINVAL, "greedy colouring needs more than 256 colours");
    *n_colors = nc;
    return TAL_OK;
    TAL_GUARD_END
}

int tal_check_coloring(const int64_t *conn, const int64_t *colors, int64_t n_nodes, int64_t n_elems,
                       int *valid)
{
    TAL_GUARD_BEGIN
    if (!valid || n_elems < 0 || (n_elems && (!conn || !colors)))
        return fail(TAL_EINVAL, "bad arguments");
    *valid = check_coloring(conn, colors, n_nodes, n_elems) ? 1 : 0;
    return TAL_OK;
    TAL_GUARD_END
}

int tal_renumber_nodes(const double *coords, const int64_t *conn, int64_t n_nodes, int64_t n_elems,
                       int method, int64_t *perm_out)
{
    TAL_GUARD_BEGIN
    if (n_nodes < 0 || n_elems < 0 || !perm_out)
        return fail(TAL_EINVAL, "bad arguments");
    std::vector<int32_t> perm;
    if (method == TAL_RENUMBER_RCM)
        renumber_rcm(conn, n_nodes, n_elems, perm);
    else if (method == TAL_RENUMBER_SFC)
        renumber_sfc(coords, n_nodes, perm);
    else if (method == TAL_RENUMBER_NONE) {
        for (int64_t i = 0; i < n_nodes; ++i)
            perm_out[i] = i;
        return TAL_OK;
    } else
        return fail(TAL_EINVAL, "unknown renumber method");
    for (int64_t i = 0; i < n_nodes; ++i)
        perm_out[i] = perm[i];
    return TAL_OK;
    TAL_GUARD_END
}

int tal_build_patches(const int64_t *conn, int64_t n_nodes, int64_t n_elems, int mode,
                      int64_t *n_patches, int64_t *n_patch_nodes, int32_t *off_out, int32_t *nodes_out,
                      uint8_t *closed_out)
{
    TAL_GUARD_BEGIN
    if (n_nodes < 0 || n_elems < 0 || (n_elems && !conn) || !n_patches || !n_patch_nodes ||
        (mode != 0 && mode != 1))
        return fail(TAL_EINVAL, "bad arguments");
    if (n_nodes >= (int64_t)1 << 31 || n_elems >= (int64_t)1 << 31)
        return fail(TAL_EINVAL, "too large");
    std::vector<int32_t> c32((size_t)(4 * n_elems));
    for (int64_t i = 0; i < 4 * n_elems; ++i) {
        if (conn[i] < 0 || conn[i] >= n_nodes)
            return fail(TAL_EINVAL, "connectivity index out of range [0, n_nodes)");
        c32[i] = (int32_t)conn[i];
    }
    Patches p;
    build_patches(c32.data(), n_nodes, n_elems, mode, p);
    *n_patches = p.n_patches();
    *n_patch_nodes = (int64_t)p.nodes.size();
    if (nodes_out && off_out && closed_out) {
        std::memcpy(off_out, p.off.data(), sizeof(int32_t) * p.off.size());
        std::memcpy(nodes_out, p.nodes.data(), sizeof(int32_t) * p.nodes.size());
        std::memcpy(closed_out, p.closed.data(), p.closed.size());
    }
    return TAL_OK;
    TAL_GUARD_END
}

int tal_peer_local(tal_handle *h, double **rx, unsigned long long **flags, int64_t *n_nodes)
{
    TAL_GUARD_BEGIN
    if (!h || !rx || !flags || !n_nodes)
        return fail(TAL_EINVAL, "NULL argument");
    if (!h->has_mesh)
        return fail(TAL_ESTATE, "no mesh uploaded");
    *rx = h->RX();
    *flags = h->d_flags;
    *n_nodes = h->N;
    return TAL_OK;
    TAL_GUARD_END
}

int tal_peer_export(tal_handle *h, void *rhs_handle, int64_t *rhs_offset, void *flags_handle)
{
    TAL_GUARD_BEGIN
    if (!h || !rhs_handle || !rhs_offset || !flags_handle)
        return fail(TAL_EINVAL, "NULL argument");
    if (!h->has_mesh)
        return fail(TAL_ESTATE, "no mesh uploaded");
    DeviceGuard g(h->device);
    TAL_CK(cudaIpcGetMemHandle((cudaIpcMemHandle_t *)rhs_handle, h->nodebuf));
    TAL_CK(cudaIpcGetMemHandle((cudaIpcMemHandle_t *)flags_handle, h->d_flags));
    *rhs_offset = (int64_t)((char *)h->RX() - (char *)h->nodebuf);
    return TAL_OK;
    TAL_GUARD_END
}

int tal_peer_attach(tal_handle *h, int slot, double *peer_rx, int64_t peer_n_nodes,
                    unsigned long long *peer_flags, const int64_t *my_ids, const int32_t *peer_ids,
                    int64_t n)
{
    TAL_GUARD_BEGIN
    if (h)
        h->free_graph();  // captured without this neighbour
    if (!h || slot < 0 || slot > 1 || !peer_rx || !peer_flags || peer_n_nodes <= 0 || n < 0 ||
        (n && (!my_ids || !peer_ids)))
        return fail(TAL_EINVAL, "bad arguments");
    if (!h->has_mesh)
        return fail(TAL_ESTATE, "no mesh uploaded");
    DeviceGuard g(h->device);
    // caller id -> internal id -> every chunk-node entry of that node
    std::vector<int32_t> remote((size_t)h->N, -1);
    for (int64_t i = 0; i < n; ++i) {
        if (my_ids[i] < 0 || my_ids[i] >= h->N || peer_ids[i] < 0 || peer_ids[i] >= peer_n_nodes ||
            peer_ids[i] >= (1 << 30))
            return fail(TAL_EINVAL, "peer node id out of range");
        const int64_t v = h->h_iperm.empty() ? my_ids[i] : h->h_iperm[my_ids[i]];
        remote[v] = peer_ids[i];
    }
    const auto &cn = h->ch.cnodes;
    if (h->h_pidx.size() != cn.size())
        h->h_pidx.assign(cn.size(), -1);
    for (size_t q = 0; q < cn.size(); ++q) {
        const uint32_t raw = (uint32_t)cn[q];
        const int32_t r = remote[raw & 0x7fffffffu];
        if (r < 0)
            continue;
        if (raw & 0x80000000u)
            return fail(TAL_EINVAL, "peer node was not declared external at upload");
        h->h_pidx[q] = (int32_t)(((uint32_t)slot << 30) | (uint32_t)r);
    }
    if (!h->d_pidx && !cn.empty())
        TAL_CK(cudaMalloc((void **)&h->d_pidx, sizeof(int32_t) * cn.size()));
    if (!cn.empty())
        TAL_CK(cudaMemcpy(h->d_pidx, h->h_pidx.data(), sizeof(int32_t) * cn.size(), cudaMemcpyHostToDevice));
    h->peers[slot].rx = peer_rx;
    h->peers[slot].n = peer_n_nodes;
    h->peers[slot].flags = peer_flags;
    return TAL_OK;
    TAL_GUARD_END
}

int tal_peer_open(tal_handle *h, int slot, const void *rhs_handle, int64_t rhs_offset,
                  const void *flags_handle, int64_t peer_n_nodes, const int64_t *my_ids,
                  const int32_t *peer_ids, int64_t n)
{
    TAL_GUARD_BEGIN
    if (!h || slot < 0 || slot > 1 || !rhs_handle || !flags_handle)
        return fail(TAL_EINVAL, "bad arguments");
    DeviceGuard g(h->device);
    void *rb = nullptr, *fb = nullptr;
    cudaIpcMemHandle_t hr, hf;
    std::memcpy(&hr, rhs_handle, sizeof hr);
    std::memcpy(&hf, flags_handle, sizeof hf);
    TAL_CK(cudaIpcOpenMemHandle(&rb, hr, cudaIpcMemLazyEnablePeerAccess));
    cudaError_t e = cudaIpcOpenMemHandle(&fb, hf, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
        cudaIpcCloseMemHandle(rb);
        return fail(TAL_ECUDA, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
    }
    int rc = tal_peer_attach(h, slot, (double *)((char *)rb + rhs_offset), peer_n_nodes,
                             (unsigned long long *)fb, my_ids, peer_ids, n);
    if (rc) {
        cudaIpcCloseMemHandle(rb);
        cudaIpcCloseMemHandle(fb);
        return rc;
    }
    h->peers[slot].ipc_rhs = rb;
    h->peers[slot].ipc_flags = fb;
    return TAL_OK;
    TAL_GUARD_END
}

int tal_peer_detach(tal_handle *h)
{
    TAL_GUARD_BEGIN
    if (!h)
        return fail(TAL_EINVAL, "handle is NULL");
    DeviceGuard g(h->device);
    cudaStreamSynchronize(h->stream);
    h->free_peers();
    return TAL_OK;
    TAL_GUARD_END
}

int tal_profile(tal_handle *h, int enable)
{
    TAL_GUARD_BEGIN
    if (!h)
        return fail(TAL_EINVAL, "handle is NULL");
    DeviceGuard g(h->device);
    if (enable && h->prof_ev.empty()) {
        h->prof_ev.resize(2 * tal_handle::PROF_RING);
        for (auto &ev : h->prof_ev)
            TAL_CK(cudaEventCreate(&ev));
    }
    h->prof_on = enable != 0;
    h->prof_head = h->prof_count = 0;
    return TAL_OK;
    TAL_GUARD_END
}

int tal_profile_read(tal_handle *h, double *ms_out, int64_t cap, int64_t *n_out)
{
    TAL_GUARD_BEGIN
    if (!h || !n_out || cap < 0 || (cap && !ms_out))
        return fail(TAL_EINVAL, "bad arguments");
    DeviceGuard g(h->device);
    int64_t n = 0;
    while (h->prof_count > 0 && n < cap) {
        const int64_t slot = h->prof_head;
        TAL_CK(cudaEventSynchronize(h->prof_ev[2 * slot + 1]));
        float ms = 0.f;
        TAL_CK(cudaEventElapsedTime(&ms, h->prof_ev[2 * slot], h->prof_ev[2 * slot + 1]));
        ms_out[n++] = ms;
        h->prof_head = (h->prof_head + 1) % tal_handle::PROF_RING;
        --h->prof_count;
    }
    *n_out = n;
    return TAL_OK;
    TAL_GUARD_END
}

int tal_fp64_peak(int device, double ms_target, double *tflops, double *sm_clock_mhz)
{
    TAL_GUARD_BEGIN
    // Burst FP64 FMA throughput: launches sized to ~ms_target (comparable to
    // one assembly), best of 20; the SM clock of the best launch is measured
    // in-kernel (clock64 cycles / globaltimer ns of block 0).
    if (!tflops)
        return fail(TAL_EINVAL, "NULL output");
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n)
        return fail(TAL_ECUDA, "no such CUDA device");
    DeviceGuard g(device);
    cudaDeviceProp prop;
    TAL_CK(cudaGetDeviceProperties(&prop, device));
    const int blocks = prop.multiProcessorCount * 8, threads = 256;
    double *out = nullptr;
    long long *clk = nullptr;
    TAL_CK(cudaMalloc((void **)&out, sizeof(double) * blocks));
    TAL_CK(cudaMalloc((void **)&clk, sizeof(long long) * 2));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int iters = 16;
    float ms = 0.f;
    k_dfma_peak<<<blocks, threads>>>(out, iters, 0.999999, 1e-7, clk);  // warm-up
    for (int rep = 0; rep < 16; ++rep) {
        cudaEventRecord(a);
        k_dfma_peak<<<blocks, threads>>>(out, iters, 0.999999, 1e-7, clk);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        if (ms >= ms_target)
            break;
        iters = (int)std::min<double>(iters * std::max(1.25, ms_target / std::max(ms, 1e-3f)), 1 << 26);
    }
    float best = 1e30f;
    long long best_clk[2] = {0, 1};
    for (int rep = 0; rep < 20; ++rep) {
        cudaEventRecord(a);
        k_dfma_peak<<<blocks, threads>>>(out, iters, 0.999999, 1e-7, clk);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) {
            best = ms;
            cudaMemcpy(best_clk, clk, sizeof best_clk, cudaMemcpyDeviceToHost);
        }
    }
    cudaError_t e = cudaGetLastError();
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    cudaFree(clk);
    if (e != cudaSuccess)
        return fail(TAL_ECUDA, std::string("fp64 probe: ") + cudaGetErrorString(e));
    const double flops = 2.0 * 16.0 * 8.0 * (double)iters * blocks * threads;
    *tflops = flops / (best * 1e-3) / 1e12;
    if (sm_clock_mhz)
        *sm_clock_mhz = best_clk[1] > 0 ? (double)best_clk[0] / (double)best_clk[1] * 1e3 : 0.0;
    return TAL_OK;
    TAL_GUARD_END
}

}  // extern "C"
