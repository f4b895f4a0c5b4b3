// tal_kernels.cuh -- sm_100a kernels of the assembly path.
//
// Device layout (per mesh handle, internal = renumbered node order):
//   nrec      : node records, 6 doubles (48 B) per node: x y z ux uy uz
//   rx,ry,rz  : assembled RHS, FP64 SoA
//   conn      : int4 per element (atomic / colored scatter)
//   blobs     : one contiguous, 16-B aligned record per CTA chunk of
//               edge-star patches (private scatter), fetched whole by one
//               TMA bulk copy (layout at k_assemble_private)
//   blob_off  : n_chunks+1 offsets in 16-B units
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "tal_element.cuh"

namespace tal {

struct RhsSoA {
    double *rx, *ry, *rz;
};

__host__ __device__ constexpr int pad16(int b) { return (b + 15) / 16 * 16; }

// ---------------------------------------------------------------------------
// PTX helpers: TMA bulk copy + mbarrier, cp.async
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p)
{
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, int count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init()
{
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async()
{
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity)
{
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "TAL_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra TAL_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void cp_async16(void *dst, const void *src)
{
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src)
{
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ int4 ldg_stream(const int4 *p)
{
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// shared-memory loads that the compiler may neither hoist nor merge (the
// ring loop re-reads the patch's a/b records instead of holding them in
// registers: TAL_RELOAD_AB)
__device__ __forceinline__ double2 lds2(uint32_t a)
{
    double2 r;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "r"(a));
    return r;
}

// one 48-B node record -> X, U (three 16-B loads; global or shared)
__device__ __forceinline__ void load_record_g(const double *__restrict__ rec, int v, double X[3],
                                              double U[3])
{
    const double2 *p = reinterpret_cast<const double2 *>(rec + 6 * (int64_t)v);
    const double2 a = __ldg(p), b = __ldg(p + 1), c = __ldg(p + 2);
    X[0] = a.x, X[1] = a.y, X[2] = b.x;
    U[0] = b.y, U[1] = c.x, U[2] = c.y;
}
__device__ __forceinline__ void load_record_s(const double *rec, int v, double X[3], double U[3])
{
    const double2 *p = reinterpret_cast<const double2 *>(rec + 6 * v);
    const double2 a = p[0], b = p[1], c = p[2];
    X[0] = a.x, X[1] = a.y, X[2] = b.x;
    U[0] = b.y, U[1] = c.x, U[2] = c.y;
}

// ---------------------------------------------------------------------------
// (1) one thread per element, 12 FP64 REDs (scatter = atomic)
// ---------------------------------------------------------------------------
template <bool SYM, bool PR = false, bool ST = false>
__global__ void __launch_bounds__(256) k_assemble_atomic(const int4 *__restrict__ conn,
                                                         int64_t e_begin, int64_t e_end,
                                                         const double *__restrict__ nrec, RhsSoA rhs,
                                                         ElemConsts kc, const double *__restrict__ press)
{
    const int64_t e = e_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= e_end)
        return;
    const int4 q = ldg_stream(conn + e);
    const int ids[4] = {q.x, q.y, q.z, q.w};
    double X[4][3], U[4][3], R[4][3], p4[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        load_record_g(nrec, ids[a], X[a], U[a]);
        if (PR)
            p4[a] = __ldg(press + ids[a]);
    }
    element_rhs<SYM, ST>(X, U, PR ? p4 : nullptr, kc, R);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        atomicAdd(rhs.rx + ids[a], R[a][0]);
        atomicAdd(rhs.ry + ids[a], R[a][1]);
        atomicAdd(rhs.rz + ids[a], R[a][2]);
    }
}

// the numba seam over a subset of elements, entirely in the caller's layout:
// conn rows e_begin + t (ids == nullptr) or ids[t], caller node ids; coords,
// u and rhs (N,3) AoS in caller numbering (rows are 8-B aligned)
template <bool SYM>
__global__ void __launch_bounds__(256) k_assemble_atomic_caller(const int4 *__restrict__ conn,
                                                                const int32_t *__restrict__ ids,
                                                                int64_t e_begin, int64_t k,
                                                                const double *__restrict__ xc,
                                                                const double *__restrict__ uc, double *rc,
                                                                ElemConsts kc)
{
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= k)
        return;
    const int4 q = __ldg(conn + (ids ? (int64_t)__ldg(ids + t) : e_begin + t));
    const int n[4] = {q.x, q.y, q.z, q.w};
    double X[4][3], U[4][3], R[4][3];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            X[a][c] = __ldg(xc + 3 * (int64_t)n[a] + c);
            U[a][c] = __ldg(uc + 3 * (int64_t)n[a] + c);
        }
    element_rhs<SYM>(X, U, nullptr, kc, R);
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            atomicAdd(rc + 3 * (int64_t)n[a] + c, R[a][c]);
}

// ---------------------------------------------------------------------------
// (2) one colour class per launch, plain read-modify-write (scatter = colored)
// ---------------------------------------------------------------------------
template <bool SYM, bool PR = false, bool ST = false>
__global__ void __launch_bounds__(256) k_assemble_colored(const int4 *__restrict__ conn,
                                                          int64_t e_begin, int64_t e_end,
                                                          const double *__restrict__ nrec, RhsSoA rhs,
                                                          ElemConsts kc, const double *__restrict__ press)
{
    const int64_t e = e_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= e_end)
        return;
    const int4 q = ldg_stream(conn + e);
    const int ids[4] = {q.x, q.y, q.z, q.w};
    double X[4][3], U[4][3], R[4][3], p4[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        load_record_g(nrec, ids[a], X[a], U[a]);
        if (PR)
            p4[a] = __ldg(press + ids[a]);
    }
    element_rhs<SYM, ST>(X, U, PR ? p4 : nullptr, kc, R);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        rhs.rx[ids[a]] += R[a][0];
        rhs.ry[ids[a]] += R[a][1];
        rhs.rz[ids[a]] += R[a][2];
    }
}

// ---------------------------------------------------------------------------
// (3) CTA-private accumulation over edge-star patches, persistent and
//     double-buffered (scatter = private / private-atomic)
//
// Work unit = one patch per thread: the ring of tets around an edge (a,b)
// (tal_prep.hpp), e.g. the 6 tets of a Kuhn cell around its main diagonal:
// 8 node records serve 6 tets and the sums for a, b and each ring node are
// accumulated in registers, so a tet costs ~1/3 of the shared-memory traffic
// of a thread-per-tet scheme (whose operand + result traffic saturates the
// 128 B/clk L1/shared data path before the FP64 pipe).
//
// Each persistent CTA walks chunks c = blockIdx.x + i*gridDim.x.  Per chunk:
//   stage : one TMA bulk copy brings the chunk blob (patch tables, node lists,
//           contribution layout) into shared memory (mbarrier completion),
//           issued at the top of the previous chunk into the buffer freed by
//           the chunk before it; cp.async gathers the chunk's node records
//           one chunk ahead (issued after phase B of the previous chunk, so
//           the blob it reads has had a whole phase B to arrive).  Two CTA
//           barriers per chunk: records ready / phase C(i-1) done, and
//           phase B done.
//   B     : thread t walks patch t's ring, computing each tet's 4x3 RHS in
//           registers; each patch node's sum is stored once, at its position
//           in the chunk's node-major contribution list;
//   C     : one chunk node per thread sums its contiguous contributions (patch
//           order); a plain store if all of the node's tets are in this
//           chunk, else one FP64 RED per component (ORDERED=false) or a
//           partial for the ordered merge (ORDERED=true, bitwise reproducible).
// Blob: int4 {n_patch, n_node, node_begin, n_contrib}
//     | u16 ids[16][T]  (patch p: {m | closed<<8, a, b, r_0..r_{m-1}}, lane-major)
//     | u16 pos[16][T]  (contribution position of the same slots)
//     | u16 lev[32]     (jagged level offsets, tal_prep.hpp)
//     | int32 gather[n_node]  node ids in chunk-local order      (pad 16)
//     | int32 cnode[n_node]   node id | bit31 interior, by rank   (pad 16)
//     | u8 run[n_node]        contributions per node, by rank     (pad 16).
// ---------------------------------------------------------------------------
template <int CFG>
struct PrivCfg;
template <>
#ifndef TAL_CFG0_MINB
#define TAL_CFG0_MINB 7
#endif
struct PrivCfg<0> {  // 64 patches / chunk
    static constexpr int THREADS = 64, NM = 144, NC = 544, MINB = TAL_CFG0_MINB;
};
#ifndef TAL_CFG1_MINB
#define TAL_CFG1_MINB 4
#endif
#ifndef TAL_RING_UNROLL
#define TAL_RING_UNROLL 1
#endif
constexpr int kRingUnroll = TAL_RING_UNROLL;
#ifndef TAL_GATHER_COOP
#define TAL_GATHER_COOP 1
#endif
#ifndef TAL_RELOAD_AB
#define TAL_RELOAD_AB 0
#endif
#ifndef TAL_ORIENT
#define TAL_ORIENT 0  // experiment: host-oriented patches (every ring tet det > 0)
#endif

template <>
struct PrivCfg<1> {  // 128 patches / chunk
    static constexpr int THREADS = 128, NM = 256, NC = 1088, MINB = TAL_CFG1_MINB;
};
template <>
struct PrivCfg<2> {  // 256 patches / chunk
    static constexpr int THREADS = 256, NM = 512, NC = 2176, MINB = 2;
};

constexpr int BLOB_LEVELS = 32;  // = CHUNK_LEVELS (tal_prep.hpp)
constexpr int SLOTS = 12;        // = PATCH_SLOTS (tal_prep.hpp)
template <int T, int NM, int NC, bool PR = false>
struct PrivLayout {
    static constexpr int TABLES = 4 * SLOTS * T;  // u16 ids[SLOTS][T], pos[SLOTS][T]
    static constexpr int BLOB = 16 + TABLES + 2 * BLOB_LEVELS + 2 * pad16(4 * NM) + pad16(NM);
    static constexpr int BLOB_AL = (BLOB + 127) / 128 * 128;
    static constexpr int MBAR = 0;
    static constexpr int BLOBS = 128;
    static constexpr int NREC = BLOBS + 2 * BLOB_AL;  // one buffer: gathered after phase B
    static constexpr int RES = NREC + NM * 48;
    static constexpr int PRS = RES + 3 * NC * 8;     // nodal pressures (PR only)
    static constexpr int TOTAL = PRS + (PR ? NM * 8 : 0);
};
template <int CFG, bool PR = false>
using PrivLayoutOf = PrivLayout<PrivCfg<CFG>::THREADS, PrivCfg<CFG>::NM, PrivCfg<CFG>::NC, PR>;

// Fused interface sum of a domain decomposition (scatter=private-atomic):
// the partial sum of an interface-plane node is REDed into the local RHS and,
// over NVLink peer memory, straight into the neighbouring rank's RHS -- the
// assembly kernel itself performs the "collective".
struct PeerArgs {
    const int32_t *__restrict__ pidx;  // per chunk-node entry: slot<<30 | remote internal id, or -1
    double *rx[2], *ry[2], *rz[2];     // neighbours' RHS (slot 0, 1)
};

struct PrivArgs {
    const uint8_t *__restrict__ blobs;
    const int32_t *__restrict__ blob_off;  // 16-B units, n_chunks+1
    int n_chunks;
    double *part;          // ordered-merge partials, AoS (x,y,z) per chunk-node entry node_begin + j
    const double *press;   // nodal pressures, internal order (PR instances)
    // caller layout (CL instances): u and rhs are the caller's (N,3) AoS
    // arrays in its own node numbering; the CL blobs hold caller node ids in
    // their gather and rank lists (k_cl_blobs), coordinates come from the
    // caller-order copy xc -- no global index loads inside the kernel
    const double *__restrict__ xc;
    const double *__restrict__ u_caller;
    double *rhs_caller;
};

// PR: with the optional pressure-gradient term (tal_element.cuh pressure_add);
// the nodal pressures are gathered next to the records (2 KB more shared
// memory per CTA: 3 CTAs/SM instead of 4).
// CL: caller layout -- velocities gathered straight from the caller's (N,3)
// array (coordinates still from the resident records) and sums written
// straight to the caller's (N,3) rhs: no pack / unpack kernels per step.
template <int CFG, bool ORDERED, bool PEER = false, bool PR = false, bool ST = false, bool CL = false>
__global__ void __launch_bounds__(PrivCfg<CFG>::THREADS,
                                  (PR || ST) ? (PrivCfg<CFG>::MINB * 3 + 3) / 4 : PrivCfg<CFG>::MINB)
    k_assemble_private(PrivArgs pa, const double *__restrict__ nrec_g, RhsSoA rhs, ElemConsts kc,
                       PeerArgs peer)
{
    constexpr int T = PrivCfg<CFG>::THREADS, NM = PrivCfg<CFG>::NM, NC = PrivCfg<CFG>::NC;
    using L = PrivLayoutOf<CFG, PR>;
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t *bar = reinterpret_cast<uint64_t *>(sm + L::MBAR);
    // node-major contribution lists: res*[coff[j] .. coff[j+1]) belong to node j
    double *resx = reinterpret_cast<double *>(sm + L::RES);
    double *resy = resx + NC, *resz = resy + NC;
    const int tid = threadIdx.x;
    const int first = blockIdx.x, stride = gridDim.x;
    const int n_my = pa.n_chunks > first ? (pa.n_chunks - first + stride - 1) / stride : 0;
    if (n_my == 0)
        return;
    auto blob = [&](int b) { return sm + L::BLOBS + b * L::BLOB_AL; };
    double *const nrec_s = reinterpret_cast<double *>(sm + L::NREC);
    double *const pres_s = reinterpret_cast<double *>(sm + L::PRS);

    auto issue = [&](int i, int b) {  // one thread: bulk-copy chunk i's blob into buffer b
        const int c = first + i * stride;
        const int o0 = __ldg(pa.blob_off + c), o1 = __ldg(pa.blob_off + c + 1);
        const uint32_t bytes = (uint32_t)(o1 - o0) * 16u;
        mbar_expect_tx(&bar[b], bytes);
        bulk_g2s(blob(b), pa.blobs + (size_t)o0 * 16, bytes, &bar[b]);
    };
    auto gather = [&](int b) {  // all threads: cp.async the chunk's node records
        const uint8_t *bl = blob(b);
        const int4 hdr = *reinterpret_cast<const int4 *>(bl);
        const int32_t *gl = reinterpret_cast<const int32_t *>(bl + 16 + L::TABLES + 2 * BLOB_LEVELS);
        double *dst = nrec_s;
        if constexpr (CL) {
            // two segments per node (lane-consecutive): the coordinates from
            // the caller-order copy (16 + 8 B when the 24-B row is 16-B aligned,
            // else 3 x 8 B) and the caller's u (3 x 8 B: its record slot at
            // +24 B is only 8-B aligned)
            for (int q = tid; q < 2 * hdr.y; q += T) {
                const int j = q >> 1;
                const int64_t g = gl[j];
                double *d = dst + 6 * j;
                if (q & 1) {
                    const double *us = pa.u_caller + 3 * g;
                    cp_async8(d + 3, us);
                    cp_async8(d + 4, us + 1);
                    cp_async8(d + 5, us + 2);
                } else {
                    const double *xs = pa.xc + 3 * g;
                    if (g & 1) {
                        cp_async8(d, xs);
                        cp_async8(d + 1, xs + 1);
                    } else {
                        cp_async16(d, xs);
                    }
                    cp_async8(d + 2, xs + 2);
                }
            }
            cp_async_commit();
            return;
        }
#if TAL_GATHER_COOP
        // 16-B segment per lane, lane-consecutive segments: a warp's copies
        // cover ~11 contiguous records (fewer L1 sectors / smem wavefronts
        // per instruction than one record per lane)
        for (int q = tid; q < 3 * hdr.y; q += T) {
            const int j = q / 3, sg = q - 3 * j;
            cp_async16(dst + 6 * j + 2 * sg, nrec_g + 6 * (int64_t)gl[j] + 2 * sg);
        }
        if (PR)
            for (int j = tid; j < hdr.y; j += T)
                cp_async8(pres_s + j, pa.press + gl[j]);
#else
        for (int j = tid; j < hdr.y; j += T) {
            const double *src = nrec_g + 6 * (int64_t)gl[j];
            cp_async16(dst + 6 * j, src);
            cp_async16(dst + 6 * j + 2, src + 2);
            cp_async16(dst + 6 * j + 4, src + 4);
            if (PR)
                cp_async8(pres_s + j, pa.press + gl[j]);
        }
#endif
        cp_async_commit();
    };

    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
        issue(0, 0);
        if (n_my > 1)
            issue(1, 1);
    }
    mbar_wait(&bar[0], 0);
    gather(0);

    for (int i = 0; i < n_my; ++i) {
        const int b = i & 1;
        cp_async_wait_all();
        __syncthreads();  // node records of chunk i visible to all; phase C(i-1) done
        // blob i+1 into the buffer chunk i-1 used: every thread has finished
        // reading it (phase C(i-1)) before the barrier above, so no third
        // barrier per chunk is needed; it lands during phase B(i)
        if (tid == 0 && i >= 1 && i + 1 < n_my) {
            fence_proxy_async();
            issue(i + 1, b ^ 1);
        }
        const uint8_t *bl = blob(b);
        const int4 hdr = *reinterpret_cast<const int4 *>(bl);  // n_patch, n_node, node_begin, n_contrib
        const uint16_t *lev = reinterpret_cast<const uint16_t *>(bl + 16 + L::TABLES);
        const uint8_t *tail = bl + 16 + L::TABLES + 2 * BLOB_LEVELS + pad16(4 * hdr.y);
        const int32_t *cn = reinterpret_cast<const int32_t *>(tail);
        const uint8_t *run = tail + pad16(4 * hdr.y);
        const double *nr = nrec_s;

        // phase B: one patch per thread (lane-major tables: slot s at [s*T + tid])
        if (tid < hdr.x) {
            const uint16_t *ids = reinterpret_cast<const uint16_t *>(bl + 16) + tid;
            const uint16_t *pos = ids + SLOTS * T;
#define ID(s) ids[(s) * T]
#define POS(s) pos[(s) * T]
            const int m = ID(0) & 0xff;
            const bool closed = (ID(0) >> 8) != 0;
            const int k = closed ? m : m - 1;
            // ring recurrences for tet t = (a, b, r_t, r_t+1):
            //   e1 = x_b - x_a, du1 = u_b - u_a (patch constants),
            //   e2(t) = e3(t-1), du2(t) = du3(t-1), c3(t) = e1 x e2(t) = -c2(t-1)
            // (carried as nc3 = -c3 = c2(t-1): tet_tail<.., NEG3> folds the sign)
#if TAL_RELOAD_AB
            // a's and b's records are re-read per tet (5 LDS.128) instead of
            // living in 18 registers
            const uint32_t ra = smem_u32(nr + 6 * ID(1)), rb = smem_u32(nr + 6 * ID(2));
            double S01[3], e1[3], du1[3], e2[3], du2[3], U2[3], nc3[3];
            {
                double Xa[3], Ua[3], Ub[3];
#else
            double Xa[3], Ua[3], Ub[3], S01[3], e1[3], du1[3], e2[3], du2[3], U2[3], nc3[3];
            {
#endif
                double Xb[3], Xr[3];
                load_record_s(nr, ID(1), Xa, Ua);
                load_record_s(nr, ID(2), Xb, Ub);
                load_record_s(nr, ID(3), Xr, U2);
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    e1[q] = Xb[q] - Xa[q];
                    du1[q] = Ub[q] - Ua[q];
                    S01[q] = Ua[q] + Ub[q];
                    e2[q] = Xr[q] - Xa[q];
                    du2[q] = U2[q] - Ua[q];
                }
                cross3(e2, e1, nc3);
            }
            // R[0], R[1] carry the running sums of a and b, R[2] enters with the
            // previous tet's contribution to r_t and leaves complete for r_t,
            // R[3] (r_t+1) becomes the next tet's carry
            double R[4][3] = {{0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}, {0.0, 0.0, 0.0}};
            double pab = 0.0, p2 = 0.0;  // pressure: p_a + p_b, p_{r_t}
            if (PR) {
                pab = pres_s[ID(1)] + pres_s[ID(2)];
                p2 = pres_s[ID(3)];
            }
#pragma unroll kRingUnroll
            for (int t = 0; t < k; ++t) {
                double X3[3], U3[3], e3[3], du3[3], c1[3], c2[3];
                const int nxt = (t + 1 == m) ? 0 : t + 1;
                load_record_s(nr, ID(3 + nxt), X3, U3);
#if TAL_RELOAD_AB
                double Xa[3], Ua[3], Ub[3];
                {
                    const double2 p0 = lds2(ra), p1 = lds2(ra + 16), p2 = lds2(ra + 32);
                    const double2 q1 = lds2(rb + 16), q2 = lds2(rb + 32);
                    Xa[0] = p0.x, Xa[1] = p0.y, Xa[2] = p1.x, Ua[0] = p1.y, Ua[1] = p2.x, Ua[2] = p2.y;
                    Ub[0] = q1.y, Ub[1] = q2.x, Ub[2] = q2.y;
                }
#endif
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    e3[q] = X3[q] - Xa[q];
                    du3[q] = U3[q] - Ua[q];
                }
                cross3(e2, e3, c1);
                cross3(e3, e1, c2);
                const double det = fma(e1[0], c1[0], fma(e1[1], c1[1], e1[2] * c1[2]));
                tet_tail<true, true, TAL_ORIENT != 0, ST>(c1, c2, nc3, det, du1, du2, du3, Ua, Ub, S01, U2, U3, kc, R);
                if (PR) {
                    const double p3 = pres_s[ID(3 + nxt)];
                    const double c3[3] = {-nc3[0], -nc3[1], -nc3[2]};
                    pressure_add(0.25 * (pab + (p2 + p3)), det, c1, c2, c3, R);
                    p2 = p3;
                }
                const int p = POS(3 + t);
                resx[p] = R[2][0];
                resy[p] = R[2][1];
                resz[p] = R[2][2];
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    R[2][q] = R[3][q];
                    R[3][q] = 0.0;
                    e2[q] = e3[q];
                    du2[q] = du3[q];
                    U2[q] = U3[q];
                    nc3[q] = c2[q];
                }
            }
            double *carry = R[2], *acc_a = R[0], *acc_b = R[1];
            // the ring node after the last tet: r_0 again (closed) or r_{m-1}
            const int pl = POS(3 + (closed ? 0 : m - 1));
            if (closed) {
                resx[pl] += carry[0];
                resy[pl] += carry[1];
                resz[pl] += carry[2];
            } else {
                resx[pl] = carry[0];
                resy[pl] = carry[1];
                resz[pl] = carry[2];
            }
            resx[POS(1)] = acc_a[0];
            resy[POS(1)] = acc_a[1];
            resz[POS(1)] = acc_a[2];
            resx[POS(2)] = acc_b[0];
            resy[POS(2)] = acc_b[1];
            resz[POS(2)] = acc_b[2];
#undef ID
#undef POS
        }
        __syncthreads();
        // records of chunk i+1 into the (single) record buffer, free now that
        // phase B(i) is done; its blob has had all of phase B(i) to land
        if (i + 1 < n_my) {
            mbar_wait(&bar[b ^ 1], ((i + 1) >> 1) & 1);
            gather(b ^ 1);
        }

        // phase C: one node per thread, nodes in rank order (contribution count
        // descending); its s-th contribution sits at lev[s] + q, so a warp
        // reads lane-contiguous addresses at every level
        for (int q = tid; q < hdr.y; q += T) {
            const int nr_ = run[q];
            double ax = 0.0, ay = 0.0, az = 0.0;
            for (int s = 0; s < nr_; ++s) {
                const int p = lev[s] + q;
                ax += resx[p];
                ay += resy[p];
                az += resz[p];
            }
            const int raw = cn[q];
            const int v = raw & 0x7fffffff;
            if constexpr (CL) {
                double *r = pa.rhs_caller + 3 * (int64_t)v;  // CL blobs: caller id
                if (raw < 0) {
                    r[0] = ax;
                    r[1] = ay;
                    r[2] = az;
                } else if (ORDERED) {
                    double *d = pa.part + 3 * (int64_t)(hdr.z + q);
                    d[0] = ax;
                    d[1] = ay;
                    d[2] = az;
                } else {
                    atomicAdd(r + 0, ax);
                    atomicAdd(r + 1, ay);
                    atomicAdd(r + 2, az);
                }
                continue;
            }
            if (raw < 0) {  // interior: the complete sum
                rhs.rx[v] = ax;
                rhs.ry[v] = ay;
                rhs.rz[v] = az;
            } else if (ORDERED) {
                double *d = pa.part + 3 * (int64_t)(hdr.z + q);
                d[0] = ax;
                d[1] = ay;
                d[2] = az;
            } else {
                atomicAdd(rhs.rx + v, ax);
                atomicAdd(rhs.ry + v, ay);
                atomicAdd(rhs.rz + v, az);
                if constexpr (PEER) {
                    const int pi = peer.pidx[hdr.z + q];
                    if (pi >= 0) {  // interface node: the neighbour's copy gets our sum too
                        const bool s1 = (pi >> 30) != 0;  // selects, not a local-memory index
                        const int r = pi & 0x3fffffff;
                        atomicAdd_system((s1 ? peer.rx[1] : peer.rx[0]) + r, ax);
                        atomicAdd_system((s1 ? peer.ry[1] : peer.ry[0]) + r, ay);
                        atomicAdd_system((s1 ? peer.rz[1] : peer.rz[0]) + r, az);
                    }
                }
            }
        }
    }
}

// caller-layout blobs (tal_run_caller): a copy of the chunk blobs whose
// gather list and rank-ordered node list hold caller node ids (cg / cc,
// indexed node_begin + j) instead of internal ones, interior bit kept
template <int CFG>
__global__ void __launch_bounds__(PrivCfg<CFG>::THREADS) k_cl_blobs(uint8_t *__restrict__ blobs,
                                                                    const int32_t *__restrict__ blob_off,
                                                                    const int32_t *__restrict__ cg,
                                                                    const int32_t *__restrict__ cc)
{
    using L = PrivLayoutOf<CFG>;
    uint8_t *bl = blobs + (size_t)blob_off[blockIdx.x] * 16;
    const int4 hdr = *reinterpret_cast<const int4 *>(bl);
    int32_t *gl = reinterpret_cast<int32_t *>(bl + 16 + L::TABLES + 2 * BLOB_LEVELS);
    int32_t *cn = reinterpret_cast<int32_t *>(bl + 16 + L::TABLES + 2 * BLOB_LEVELS + pad16(4 * hdr.y));
    for (int j = threadIdx.x; j < hdr.y; j += blockDim.x) {
        gl[j] = cg[hdr.z + j];
        cn[j] = (int32_t)((uint32_t)cc[hdr.z + j] | ((uint32_t)cn[j] & 0x80000000u));
    }
}

// caller-order coordinate copy for the caller-layout gather: xc[perm[i]] = rec[i]
__global__ void __launch_bounds__(256) k_caller_coords(const double *__restrict__ rec,
                                                       const int32_t *__restrict__ perm, int64_t n, double *xc)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const int64_t c = perm ? (int64_t)perm[i] : i;
    xc[3 * c + 0] = rec[6 * i + 0];
    xc[3 * c + 1] = rec[6 * i + 1];
    xc[3 * c + 2] = rec[6 * i + 2];
}

// ordered merge of chunk partials for nodes shared between chunks (and zero
// for nodes without elements): rhs[v] = sum over its chunks in chunk order
// (caller_out: write the caller's (N,3) rhs at perm[v] instead of the SoA)
__global__ void __launch_bounds__(256) k_merge_partials(const int32_t *__restrict__ bnd_nodes,
                                                        const int32_t *__restrict__ bnd_off,
                                                        const int32_t *__restrict__ bnd_pos,
                                                        int64_t n_bnd, const double *__restrict__ part,
                                                        RhsSoA rhs, double *caller_out = nullptr,
                                                        const int32_t *__restrict__ perm = nullptr)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n_bnd)
        return;
    double ax = 0.0, ay = 0.0, az = 0.0;
    const int p0 = bnd_off[i], p1 = bnd_off[i + 1];
    // batches of 4 partials: all position and value loads of a batch are in
    // flight together; the sum keeps the chunk order (bitwise unchanged)
    for (int p = p0; p < p1; p += 4) {
        int q[4];
        double x[4][3];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            q[k] = p + k < p1 ? __ldg(bnd_pos + p + k) : -1;
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (q[k] >= 0) {
                const double *e = part + 3 * (int64_t)q[k];  // one 24-B entry
                x[k][0] = e[0];
                x[k][1] = e[1];
                x[k][2] = e[2];
            }
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (q[k] >= 0) {
                ax += x[k][0];
                ay += x[k][1];
                az += x[k][2];
            }
    }
    const int v = bnd_nodes[i];
    if (caller_out) {
        double *r = caller_out + 3 * (int64_t)(perm ? perm[v] : v);
        r[0] = ax;
        r[1] = ay;
        r[2] = az;
        return;
    }
    rhs.rx[v] = ax;
    rhs.ry[v] = ay;
    rhs.rz[v] = az;
}

// ---------------------------------------------------------------------------
// layout conversion: caller AoS (n,3) <-> internal records / SoA (renumbered)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_pack_velocity(const double *__restrict__ aos,
                                                       const int32_t *__restrict__ perm, int64_t n,
                                                       double *nrec)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const int64_t s = perm ? (int64_t)perm[i] : i;
    nrec[6 * i + 3] = aos[3 * s + 0];
    nrec[6 * i + 4] = aos[3 * s + 1];
    nrec[6 * i + 5] = aos[3 * s + 2];
}

__global__ void __launch_bounds__(256) k_pack_scalar(const double *__restrict__ src,
                                                     const int32_t *__restrict__ perm, int64_t n,
                                                     double *dst)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n)
        dst[i] = src[perm ? (int64_t)perm[i] : i];
}

__global__ void __launch_bounds__(256) k_unpack_aos(const double *__restrict__ rx,
                                                    const double *__restrict__ ry,
                                                    const double *__restrict__ rz,
                                                    const int32_t *__restrict__ iperm, int64_t n,
                                                    double *aos)
{
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n)
        return;
    const int64_t s = iperm ? (int64_t)iperm[j] : j;
    aos[3 * j + 0] = rx[s];
    aos[3 * j + 1] = ry[s];
    aos[3 * j + 2] = rz[s];
}

// cross-rank ordering of the fused interface sum: a rank signals each
// neighbour (system-scope add on the neighbour's flag word) and waits until
// its own flag word reached epoch x n_neighbours.  The step epoch is a device
// word (own flags[2], advanced by the first signal of a step), so a step is
// free of host-side state and can be captured in a CUDA graph.
__global__ void k_peer_signal(unsigned long long *f0, unsigned long long *f1, int which,
                              unsigned long long *own_epoch)
{
    if (own_epoch)
        own_epoch[0] += 1ull;
    __threadfence_system();
    if (f0)
        atomicAdd_system(f0 + which, 1ull);
    if (f1)
        atomicAdd_system(f1 + which, 1ull);
}

// A neighbour that never signals (its process died, a mismatched step count)
// must not hang the GPU: after TAL_PEER_WAIT_NS of waiting the kernel traps,
// so the step fails with a launch error instead of spinning forever.
#ifndef TAL_PEER_WAIT_NS
#define TAL_PEER_WAIT_NS 30000000000ull  // 30 s
#endif
__global__ void k_peer_wait(const unsigned long long *flags, int which, int n_peers)
{
    const unsigned long long target = flags[2] * (unsigned long long)n_peers;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        unsigned long long v, t;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + which) : "memory");
        if (v >= target)
            break;
        __nanosleep(256);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > TAL_PEER_WAIT_NS)
            __trap();
    }
    __threadfence_system();
}

// interface-node exchange helpers (multi-GPU domain decomposition)
__global__ void k_halo_pack(const int32_t *__restrict__ list, int64_t n, const double *rx,
                            const double *ry, const double *rz, double *out)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const int v = list[i];
    out[3 * i + 0] = rx[v];
    out[3 * i + 1] = ry[v];
    out[3 * i + 2] = rz[v];
}

__global__ void k_halo_accumulate(const int32_t *__restrict__ list, int64_t n,
                                  const double *__restrict__ in, double *rx, double *ry, double *rz)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const int v = list[i];
    rx[v] += in[3 * i + 0];
    ry[v] += in[3 * i + 1];
    rz[v] += in[3 * i + 2];
}

// FP64 pipe throughput probe: 8 independent DFMA chains per thread
__global__ void __launch_bounds__(256) k_dfma_peak(double *out, int iters, double a, double b,
                                                   long long *clk)
{
    long long c0 = 0, t0 = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        c0 = clock64();
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    }
    double c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
        c[i] = (double)(threadIdx.x + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
            for (int i = 0; i < 8; ++i)
                c[i] = fma(c[i], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
        s += c[i];
    if (s == 1.2345)  // never true; keeps the chains live
        out[blockIdx.x] = s;
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // SM clock of this launch: cycles / ns
        long long t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        clk[0] = clock64() - c0;
        clk[1] = t1 - t0;
    }
}

}  // namespace tal
