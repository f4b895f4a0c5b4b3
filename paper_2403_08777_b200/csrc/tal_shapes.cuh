// tal_shapes.cuh -- the paper's code-shape study on B200: the baseline (B) and
// restructured+specialised (RS) shapes of the same element operator, as
// sm_100a kernels.
//
// Both are one thread per tetrahedron with the scatter done by FP64 REDs
// (scatter=atomic) or by colour-by-colour plain read-modify-write
// (scatter=colored, bitwise reproducible).  They exist to measure what the
// restructuring, specialisation and privatisation of the RSP kernels
// (tal_kernels.cuh) buy on this hardware, with real counters (ncu): they are
// deliberately NOT optimised beyond their shape.
//
//  B  (variants.py:294-370, _chunk_baseline): generic element -- node,
//     dimension and Gauss-point trip counts are runtime values, the Jacobian,
//     its inverse (nine divisions), the Cartesian gradients, the point
//     velocity, the velocity gradient and the Vreman viscosity are recomputed
//     at every Gauss point, a dense 12x12 elemental matrix is built and
//     multiplied by the nodal unknowns, and the element vector is scattered
//     by a separate loop.  The per-element arrays live in local memory.
//  P  (study only; "P"): the B statements with literal trip
//     counts and unrolled loops (privatised arrays, no restructuring).
//  RS (variants.py:373-464, _chunk_restructured): tet4-specialised -- fixed
//     trip counts, geometry / gradient / viscosity once per element, explicit
//     4-point Gauss loop for the convective term, RHS entries computed
//     directly (no elemental matrix); everything in registers.
//
// Vreman closure as kernel.py:99-143 / variants.py:250-281 (same minor order,
// unfused products so exactly rank-1 gradients give exactly 0).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "tal_kernels.cuh"

namespace tal {

struct ShapeConsts {
    double rho, mu, cvre;
    int nn, nd, ng;         // runtime trip counts of the baseline shape (4, 3, 4)
    double npts[4][4];      // quadrature_tet4 points: N_a at Gauss point g = npts[g][a] (kernel.py:71-86)
    double wts[4];          // Gauss weights
    double dshape[4][4][3]; // reference shape gradients per point (TET4_REF_GRADS, variants.py:31-39)
};

// _chunk_eddy (variants.py:250-281) for one element
__device__ __forceinline__ double vreman_ref(const double g[3][3], double dlt, double cvre)
{
    double aa = 0.0;
#pragma unroll
    for (int q = 0; q < 9; ++q)
        aa = __dadd_rn(aa, __dmul_rn(g[q / 3][q % 3], g[q / 3][q % 3]));
    // minors d0..d8: rows (m,n) x columns (i,j) in the reference order
    const int M[9] = {0, 0, 1, 0, 0, 1, 0, 0, 1}, Nn[9] = {1, 2, 2, 1, 2, 2, 1, 2, 2};
    const int I[9] = {0, 0, 0, 0, 0, 0, 1, 1, 1}, J[9] = {1, 1, 1, 2, 2, 2, 2, 2, 2};
    double ssq = 0.0;
#pragma unroll
    for (int q = 0; q < 9; ++q) {
        const double d = __dsub_rn(__dmul_rn(g[M[q]][I[q]], g[Nn[q]][J[q]]),
                                   __dmul_rn(g[M[q]][J[q]], g[Nn[q]][I[q]]));
        ssq = __dadd_rn(ssq, __dmul_rn(d, d));
    }
    const double d2 = dlt * dlt;
    const double bb = d2 * d2 * ssq;
    if (!(aa > 1e-30))  // DENOM_EPSILON (kernel.py:24)
        return 0.0;
    return cvre * sqrt(fmax(bb, 0.0) / aa);
}

__device__ __forceinline__ void scatter_elem(const int ids[4], const double r[4][3], RhsSoA rhs, bool colored)
{
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        if (colored) {
            rhs.rx[ids[a]] += r[a][0];
            rhs.ry[ids[a]] += r[a][1];
            rhs.rz[ids[a]] += r[a][2];
        } else {
            atomicAdd(rhs.rx + ids[a], r[a][0]);
            atomicAdd(rhs.ry + ids[a], r[a][1]);
            atomicAdd(rhs.rz + ids[a], r[a][2]);
        }
    }
}

// ---------------------------------------------------------------------------
// B: generic baseline shape
// ---------------------------------------------------------------------------
template <bool COLORED, bool FIXED = false>
__global__ void __launch_bounds__(256) k_assemble_baseline(const int4 *__restrict__ conn, int64_t e_begin,
                                                           int64_t e_end, const double *__restrict__ nrec,
                                                           RhsSoA rhs, ShapeConsts sc)
{
    const int64_t e = e_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= e_end)
        return;
    // FIXED (the paper's "P" shape, study only): the same statements with
    // literal trip counts and unrolled loops, so the per-element arrays can be
    // privatised into registers (what does not fit spills)
    constexpr int UR = FIXED ? 16 : 1;
    const int nn = FIXED ? 4 : sc.nn, nd = FIXED ? 3 : sc.nd, ng = FIXED ? 4 : sc.ng;
    const int4 q = conn[e];
    const int ids[4] = {q.x, q.y, q.z, q.w};
    double xe[4][3], ue[4][3];
#pragma unroll UR
    for (int a = 0; a < nn; ++a)
#pragma unroll UR
        for (int k = 0; k < nd; ++k) {
            xe[a][k] = nrec[6 * (int64_t)ids[a] + k];
            ue[a][k] = nrec[6 * (int64_t)ids[a] + 3 + k];
        }
    double gpcar[4][4][3], gpvol[4], gpvel[4][3], gpvis[4];
#pragma unroll UR
    for (int ig = 0; ig < ng; ++ig) {
        double xjac[3][3];
#pragma unroll UR
        for (int k = 0; k < nd; ++k)
#pragma unroll UR
            for (int l = 0; l < nd; ++l) {
                double s = 0.0;
#pragma unroll UR
                for (int a = 0; a < nn; ++a)
                    s += xe[a][k] * sc.dshape[ig][a][l];
                xjac[k][l] = s;
            }
        const double t0 = xjac[1][1] * xjac[2][2] - xjac[1][2] * xjac[2][1];
        const double t1 = xjac[1][2] * xjac[2][0] - xjac[1][0] * xjac[2][2];
        const double t2 = xjac[1][0] * xjac[2][1] - xjac[1][1] * xjac[2][0];
        const double det = xjac[0][0] * t0 + xjac[0][1] * t1 + xjac[0][2] * t2;
        double xinv[3][3];
        xinv[0][0] = (xjac[1][1] * xjac[2][2] - xjac[1][2] * xjac[2][1]) / det;
        xinv[0][1] = (xjac[0][2] * xjac[2][1] - xjac[0][1] * xjac[2][2]) / det;
        xinv[0][2] = (xjac[0][1] * xjac[1][2] - xjac[0][2] * xjac[1][1]) / det;
        xinv[1][0] = (xjac[1][2] * xjac[2][0] - xjac[1][0] * xjac[2][2]) / det;
        xinv[1][1] = (xjac[0][0] * xjac[2][2] - xjac[0][2] * xjac[2][0]) / det;
        xinv[1][2] = (xjac[0][2] * xjac[1][0] - xjac[0][0] * xjac[1][2]) / det;
        xinv[2][0] = (xjac[1][0] * xjac[2][1] - xjac[1][1] * xjac[2][0]) / det;
        xinv[2][1] = (xjac[0][1] * xjac[2][0] - xjac[0][0] * xjac[2][1]) / det;
        xinv[2][2] = (xjac[0][0] * xjac[1][1] - xjac[0][1] * xjac[1][0]) / det;
#pragma unroll UR
        for (int a = 0; a < nn; ++a)
#pragma unroll UR
            for (int k = 0; k < nd; ++k) {
                double s = 0.0;
#pragma unroll UR
                for (int l = 0; l < nd; ++l)
                    s += sc.dshape[ig][a][l] * xinv[l][k];
                gpcar[ig][a][k] = s;
            }
        const double vol = fabs(det) / 6.0;
        gpvol[ig] = sc.wts[ig] * vol;
        const double dlt = cbrt(6.0 * vol);
        double gve[3][3];
#pragma unroll UR
        for (int i = 0; i < nd; ++i) {
            double s = 0.0;
#pragma unroll UR
            for (int a = 0; a < nn; ++a)
                s += sc.npts[ig][a] * ue[a][i];
            gpvel[ig][i] = s;
        }
#pragma unroll UR
        for (int k = 0; k < nd; ++k)
#pragma unroll UR
            for (int i = 0; i < nd; ++i) {
                double s = 0.0;
#pragma unroll UR
                for (int a = 0; a < nn; ++a)
                    s += gpcar[ig][a][k] * ue[a][i];
                gve[k][i] = s;
            }
        gpvis[ig] = sc.mu + sc.rho * vreman_ref(gve, dlt, sc.cvre);
    }
    // dense elemental matrix (nn*nd)^2, then elrhs = -elemat . u
    double elemat[12][12];
#pragma unroll UR
    for (int r = 0; r < nn * nd; ++r)
#pragma unroll UR
        for (int c = 0; c < nn * nd; ++c)
            elemat[r][c] = 0.0;
#pragma unroll UR
    for (int ig = 0; ig < ng; ++ig)
#pragma unroll UR
        for (int a = 0; a < nn; ++a)
#pragma unroll UR
            for (int b = 0; b < nn; ++b) {
                double cdot = 0.0, ddot = 0.0;
#pragma unroll UR
                for (int k = 0; k < nd; ++k) {
                    cdot += gpvel[ig][k] * gpcar[ig][b][k];
                    ddot += gpcar[ig][a][k] * gpcar[ig][b][k];
                }
                const double conv = sc.rho * gpvol[ig] * sc.npts[ig][a] * cdot;
                const double diff = gpvis[ig] * gpvol[ig] * ddot;
                const double s_ab = conv + diff;
#pragma unroll UR
                for (int i = 0; i < nd; ++i)
                    elemat[a * nd + i][b * nd + i] += s_ab;
            }
    double elrhs[4][3];
#pragma unroll UR
    for (int r = 0; r < nn * nd; ++r) {
        double s = 0.0;
#pragma unroll UR
        for (int c = 0; c < nn * nd; ++c)
            s += elemat[r][c] * ue[c / nd][c % nd];
        elrhs[r / nd][r % nd] = -s;
    }
    scatter_elem(ids, elrhs, rhs, COLORED);
}

// ---------------------------------------------------------------------------
// RS: restructured + specialised shape
// ---------------------------------------------------------------------------
template <bool COLORED>
__global__ void __launch_bounds__(256) k_assemble_rs(const int4 *__restrict__ conn, int64_t e_begin,
                                                     int64_t e_end, const double *__restrict__ nrec,
                                                     RhsSoA rhs, ShapeConsts sc)
{
    const int64_t e = e_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= e_end)
        return;
    const int4 q = conn[e];
    const int ids[4] = {q.x, q.y, q.z, q.w};
    double X[4][3], U[4][3];
#pragma unroll
    for (int a = 0; a < 4; ++a)
        load_record_g(nrec, ids[a], X[a], U[a]);
    double e1[3], e2[3], e3[3], c[4][3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        e1[k] = X[1][k] - X[0][k];
        e2[k] = X[2][k] - X[0][k];
        e3[k] = X[3][k] - X[0][k];
    }
    c[1][0] = e2[1] * e3[2] - e2[2] * e3[1];
    c[1][1] = e2[2] * e3[0] - e2[0] * e3[2];
    c[1][2] = e2[0] * e3[1] - e2[1] * e3[0];
    c[2][0] = e3[1] * e1[2] - e3[2] * e1[1];
    c[2][1] = e3[2] * e1[0] - e3[0] * e1[2];
    c[2][2] = e3[0] * e1[1] - e3[1] * e1[0];
    c[3][0] = e1[1] * e2[2] - e1[2] * e2[1];
    c[3][1] = e1[2] * e2[0] - e1[0] * e2[2];
    c[3][2] = e1[0] * e2[1] - e1[1] * e2[0];
    const double det = e1[0] * c[1][0] + e1[1] * c[1][1] + e1[2] * c[1][2];
    const double vol = fabs(det) / 6.0;
    const double dlt = cbrt(6.0 * vol);
    double b[4][3];
#pragma unroll
    for (int a = 1; a < 4; ++a)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            b[a][k] = c[a][k] / det;
#pragma unroll
    for (int k = 0; k < 3; ++k)
        b[0][k] = -(b[1][k] + b[2][k] + b[3][k]);
    double G[3][3];
#pragma unroll
    for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int i = 0; i < 3; ++i)
            G[k][i] = b[0][k] * U[0][i] + b[1][k] * U[1][i] + b[2][k] * U[2][i] + b[3][k] * U[3][i];
    const double vis = sc.mu + sc.rho * vreman_ref(G, dlt, sc.cvre);
    const double rv = (0.25 * sc.rho) * vol;
    const double vv = vis * vol;
    double cv[4][3];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        double ug[3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
            ug[i] = sc.npts[g][0] * U[0][i] + sc.npts[g][1] * U[1][i] + sc.npts[g][2] * U[2][i] +
                    sc.npts[g][3] * U[3][i];
#pragma unroll
        for (int i = 0; i < 3; ++i)
            cv[g][i] = ug[0] * G[0][i] + ug[1] * G[1][i] + ug[2] * G[2][i];
    }
    double r[4][3];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int i = 0; i < 3; ++i)
            r[a][i] = -rv * (sc.npts[0][a] * cv[0][i] + sc.npts[1][a] * cv[1][i] + sc.npts[2][a] * cv[2][i] +
                             sc.npts[3][a] * cv[3][i]) -
                      vv * (b[a][0] * G[0][i] + b[a][1] * G[1][i] + b[a][2] * G[2][i]);
    scatter_elem(ids, r, rhs, COLORED);
}

}  // namespace tal
