// tal_strict.cuh -- reference-order ("sequential") assembly: the element
// arithmetic of the reference numba kernel operation by operation, and the
// node-centric summation of the reference's one-thread private driver, so the
// GPU result is bitwise identical to the reference's assemble_rsp output.
//
// Reference: _rsp_kernels.py:33-164 (element loop; numba compiles it without
// FMA contraction -- SURVEY.md section 8c: 246 vmulsd / 145 vaddsd / 42 vsubsd /
// 11 vdivsd, 0 vfmadd), variants.py:573-596 with n_threads=1 (one accumulator,
// elements in ascending id order, rhs starts at zero).
//
// Every product / sum / difference / quotient below is an explicit
// round-to-nearest intrinsic (__dmul_rn, __dadd_rn, __dsub_rn, __ddiv_rn,
// __dsqrt_rn) in the reference's left-to-right order, so nvcc cannot contract
// or reassociate.  The one library call of the reference, numba's np.cbrt =
// pow(6 vol, 1/3) from the host libm, is a per-element geometry constant (the
// Vreman filter width delta): glibc's pow is not correctly rounded (0.52 ulp
// bound; e.g. x = 0x1.3813813813810p-8, exact result 0.49996 ulp above the
// nearest double, returns the upper neighbour), so no device formula can match
// it bit for bit without glibc's tables.  delta is therefore computed once per
// mesh on the host, with the same IEEE operations as below and the same libm
// call as the reference (tal_capi.cu build_sequential), and read per element.
//
// This is the parity / debugging path (SURVEY.md 8c "strict" build), not the
// fast one: every element is evaluated once per node it touches (4x the
// arithmetic of the element loop) so each node can sum its contributions in
// ascending element order.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "tal_element.cuh"

namespace tal {

#define TM(a, b) __dmul_rn((a), (b))
#define TA(a, b) __dadd_rn((a), (b))
#define TS(a, b) __dsub_rn((a), (b))

// Row a (node a's three entries) of the element RHS, reference operation
// order.  X, U: the four corner coordinates / velocities in the element's own
// node order; pm: the 16 pmat values (variants.py:559).
// Rows a0 .. a1-1 (r: 3 doubles per row); the geometry / gradient / Vreman
// prefix is computed once per call.
__device__ __forceinline__ void element_rows_strict(const double X[4][3], const double U[4][3], double dlt,
                                                    double rho, double mu, double cvre, const double *pm,
                                                    int a0, int a1, double *r)
{
    double ed[4][3];  // edges x_b - x_0 (_rsp_kernels.py:45-47)
#pragma unroll
    for (int b = 1; b < 4; ++b)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            ed[b][c] = TS(X[b][c], X[0][c]);
    double cf[4][3];  // cofactor rows: e2 x e3, e3 x e1, e1 x e2 (:49-58)
#pragma unroll
    for (int b = 1; b < 4; ++b) {
        const int i1 = b == 1 ? 2 : b == 2 ? 3 : 1, i2 = b == 1 ? 3 : b == 2 ? 1 : 2;
        cf[b][0] = TS(TM(ed[i1][1], ed[i2][2]), TM(ed[i1][2], ed[i2][1]));
        cf[b][1] = TS(TM(ed[i1][2], ed[i2][0]), TM(ed[i1][0], ed[i2][2]));
        cf[b][2] = TS(TM(ed[i1][0], ed[i2][1]), TM(ed[i1][1], ed[i2][0]));
    }
    const double det = TA(TA(TM(ed[1][0], cf[1][0]), TM(ed[1][1], cf[1][1])), TM(ed[1][2], cf[1][2]));
    const double vol = __ddiv_rn(fabs(det), 6.0);  // :61; dlt = cbrt(6 vol) (:62) is an argument
    double bg[4][3];                               // shape gradients (:64-69)
#pragma unroll
    for (int b = 1; b < 4; ++b)
#pragma unroll
        for (int c = 0; c < 3; ++c)
            bg[b][c] = __ddiv_rn(cf[b][c], det);
#pragma unroll
    for (int c = 0; c < 3; ++c)
        bg[0][c] = -TA(TA(bg[1][c], bg[2][c]), bg[3][c]);
    double g[3][3];  // g[k][i] = sum_b bg_b[k] u_b[i] (:76-85)
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int i = 0; i < 3; ++i)
            g[k][i] = TA(TA(TA(TM(bg[0][k], U[0][i]), TM(bg[1][k], U[1][i])), TM(bg[2][k], U[2][i])),
                         TM(bg[3][k], U[3][i]));
    // Vreman (:87-120; kernel.py:99-143): aa, the nine minors in the reference order
    double aa = TA(TM(g[0][0], g[0][0]), TM(g[0][1], g[0][1]));
    aa = TA(aa, TM(g[0][2], g[0][2]));
#pragma unroll
    for (int k = 1; k < 3; ++k)
#pragma unroll
        for (int i = 0; i < 3; ++i)
            aa = TA(aa, TM(g[k][i], g[k][i]));
    double nut = 0.0;
    if (aa > 1e-30) {  // kernel.py:24
        double ssq = 0.0;
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            const int cp = q / 3, rp = q % 3;  // column pair outer, row pair inner
            const int m = rp == 2 ? 1 : 0, n = rp == 0 ? 1 : 2;
            const int i = cp == 2 ? 1 : 0, j = cp == 0 ? 1 : 2;
            const double d = TS(TM(g[m][i], g[n][j]), TM(g[m][j], g[n][i]));
            ssq = q == 0 ? TM(d, d) : TA(ssq, TM(d, d));
        }
        const double d2 = TM(dlt, dlt);
        const double bb = TM(TM(d2, d2), ssq);
        if (!(bb < 0.0))
            nut = TM(cvre, __dsqrt_rn(__ddiv_rn(bb, aa)));
    }
    const double vis = TA(mu, TM(rho, nut));         // :122
    const double nrv = -TM(TM(rho, vol), 0.25);      // :123
    const double nvv = -TM(vis, vol);                // :124
#pragma unroll 1
    for (int a = a0; a < a1; ++a) {  // :126-164, node a
        double m[3];
#pragma unroll
        for (int c = 0; c < 3; ++c)
            m[c] = TA(TA(TA(TM(pm[4 * a + 0], U[0][c]), TM(pm[4 * a + 1], U[1][c])), TM(pm[4 * a + 2], U[2][c])),
                      TM(pm[4 * a + 3], U[3][c]));
        double bsel[3];
#pragma unroll
        for (int c = 0; c < 3; ++c)
            bsel[c] = a == 0 ? bg[0][c] : a == 1 ? bg[1][c] : a == 2 ? bg[2][c] : bg[3][c];
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const double cv = TA(TA(TM(m[0], g[0][i]), TM(m[1], g[1][i])), TM(m[2], g[2][i]));
            const double df = TA(TA(TM(bsel[0], g[0][i]), TM(bsel[1], g[1][i])), TM(bsel[2], g[2][i]));
            r[3 * (a - a0) + i] = TA(TM(nrv, cv), TM(nvv, df));
        }
    }
}
__device__ __forceinline__ void element_row_strict(const double X[4][3], const double U[4][3], double dlt,
                                                   double rho, double mu, double cvre, const double *pm,
                                                   int a, double r[3])
{
    element_rows_strict(X, U, dlt, rho, mu, cvre, pm, a, a + 1, r);
}

#undef TM
#undef TA
#undef TS

// One thread per node v (internal numbering): its incident elements in
// ascending caller element id (CSR ent[off[v] .. off[v+1]), entry = e << 2 | a
// with e the row of 'conn' and a the node's corner), summed in that order from
// zero -- the reference's one-accumulator private loop, node by node.  With
// 'accumulate' the sums start from the incoming rx/ry/rz (the numba seam's
// rhs += semantics, tal_assemble_elements_strict).
__global__ void __launch_bounds__(128) k_assemble_sequential(const int64_t *__restrict__ off,
                                                             const int32_t *__restrict__ ent, int64_t n_nodes,
                                                             const int4 *__restrict__ conn,
                                                             const double *__restrict__ nrec,
                                                             const double *__restrict__ dlt, double *rx,
                                                             double *ry, double *rz, ElemConsts kc,
                                                             bool accumulate)
{
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n_nodes)
        return;
    double acc[3] = {0.0, 0.0, 0.0};
    if (accumulate)
        acc[0] = rx[v], acc[1] = ry[v], acc[2] = rz[v];
    for (int64_t k = off[v]; k < off[v + 1]; ++k) {
        const int32_t en = __ldg(ent + k);
        const int4 q = __ldg(conn + (en >> 2));
        const int ids[4] = {q.x, q.y, q.z, q.w};
        double X[4][3], U[4][3];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const double2 *p = reinterpret_cast<const double2 *>(nrec + 6 * (int64_t)ids[b]);
            const double2 s0 = __ldg(p), s1 = __ldg(p + 1), s2 = __ldg(p + 2);
            X[b][0] = s0.x, X[b][1] = s0.y, X[b][2] = s1.x;
            U[b][0] = s1.y, U[b][1] = s2.x, U[b][2] = s2.y;
        }
        double r[3];
        element_row_strict(X, U, __ldg(dlt + (en >> 2)), kc.rho, kc.mu, kc.cvre, kc.pm, en & 3, r);
#pragma unroll
        for (int i = 0; i < 3; ++i)
            acc[i] = __dadd_rn(acc[i], r[i]);
    }
    rx[v] = acc[0];
    ry[v] = acc[1];
    rz[v] = acc[2];
}

}  // namespace tal

namespace tal {

// Two-pass form of the reference-order scatter: every element's four strict
// rows computed once (one thread per conn row) into contrib[e][a][i] ...
__global__ void __launch_bounds__(128) k_strict_rows(int64_t n_elems, const int4 *__restrict__ conn,
                                                     const double *__restrict__ nrec,
                                                     const double *__restrict__ dlt, double *contrib,
                                                     ElemConsts kc)
{
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n_elems)
        return;
    const int4 q = __ldg(conn + e);
    const int ids[4] = {q.x, q.y, q.z, q.w};
    double X[4][3], U[4][3];
#pragma unroll
    for (int b = 0; b < 4; ++b) {
        const double2 *p = reinterpret_cast<const double2 *>(nrec + 6 * (int64_t)ids[b]);
        const double2 s0 = __ldg(p), s1 = __ldg(p + 1), s2 = __ldg(p + 2);
        X[b][0] = s0.x, X[b][1] = s0.y, X[b][2] = s1.x;
        U[b][0] = s1.y, U[b][1] = s2.x, U[b][2] = s2.y;
    }
    const double d = __ldg(dlt + e);
    element_rows_strict(X, U, d, kc.rho, kc.mu, kc.cvre, kc.pm, 0, 4, contrib + 12 * e);
}

// ... then each node sums its rows in ascending caller element id from zero.
__global__ void __launch_bounds__(256) k_sum_rows_ordered(const int64_t *__restrict__ off,
                                                          const int32_t *__restrict__ ent, int64_t n_nodes,
                                                          const double *__restrict__ contrib, double *rx,
                                                          double *ry, double *rz)
{
    const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n_nodes)
        return;
    double ax = 0.0, ay = 0.0, az = 0.0;
    for (int64_t k = off[v]; k < off[v + 1]; ++k) {
        const double *r = contrib + 3 * (int64_t)__ldg(ent + k);  // (row << 2 | corner) * 3
        ax = __dadd_rn(ax, r[0]);
        ay = __dadd_rn(ay, r[1]);
        az = __dadd_rn(az, r[2]);
    }
    rx[v] = ax;
    ry[v] = ay;
    rz[v] = az;
}

}  // namespace tal
