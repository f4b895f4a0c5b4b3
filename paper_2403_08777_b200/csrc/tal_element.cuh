// tal_element.cuh -- per-element momentum RHS of a linear tetrahedron, in
// registers, specialised for 4 nodes and the folded 4-point Gauss rule.
//
// Operator (reference: _rsp_kernels.py:33-164, kernel.py:146-170):
//   r_a[i] = -rho * int N_a (u.grad) u_i  -  (mu + rho nu_t) int gradN_a . grad u_i
// with nu_t the Vreman closure (kernel.py:99-143) on the constant element
// gradient and filter width delta = cbrt(6 vol) = cbrt(|det|).
//
// B200 restructuring (same mathematics, fewer and shorter FP64 dependency
// chains; parity is judged at 1e-12 of the max-norm, not bitwise):
//  * Shape gradients are never divided out.  With cofactor rows c_b
//    (b=1..3, c_0 = -sum) and D = det:  G = Gh / D,
//        Gh[k][i] = sum_{b=1..3} c_b[k] (u_b[i] - u_0[i]).
//  * One cube-root reciprocal r3 = |D|^(-1/3) gives both the Vreman factor
//    and 1/|D| = r3^3 (no separate division).
//  * Vreman in unscaled quantities: aa = |G|^2, ssq = sum of the nine squared
//    2x2 minors of G (the reference's Cauchy-Binet form), so
//        nu_t = c sqrt(delta^4 ssq / aa) = c r3 sqrt(ssqh / aah)
//             = c r3 ssqh rsqrt(ssqh aah)
//    (delta^2 / |D| = r3); the quiescent guard aa <= 1e-30 (kernel.py:24) is
//    aah (1/|D|)^2 <= 1e-30.  Rank-1 gradients keep ssqh == 0 exactly.
//  * pmat = P^T P of the symmetric rule: one diagonal value pd, one
//    off-diagonal po, so the moments are m_a = po S + (pd - po) u_a, S = sum u.
//  * Both terms share Gh:  r_a[i] = sum_k w_a[k] Gh[k][i],
//        w_a = A (po S + (pd-po) u_a) + B c_a,
//        A = nrv / D = -rho sgn(D) / 24,  B = nvv / D^2 = -vis / (6 |D|),
//    and w_0 = (4 A po + A (pd-po)) S - (w_1 + w_2 + w_3) since sum_a c_a = 0.
//  * Special functions: MUFU seeds + one third-order correction each
//    (rcbrt_fast, rsqrt_fast), branch-free in the normal range.
// ~185 FP64 instructions per tet inside an edge-star ring (FMA = 1) against
// the reference ledger's 448 flop (variants.py:207-217).
#pragma once
#include <cuda_runtime.h>


namespace tal {

struct ElemConsts {
    double rho, mu, cvre;
    double rc;    // rho * c_vreman
    double a_po;  // -rho * po / 24
    double a_q;   // -rho * (pd - po) / 24
    double a_4;   // 4 a_po + a_q
    double rc6;   // -rho * c_vreman / 6
    double mu6;   // -mu / 6
    double pm[16];  // full pmat (general kernel only)
    // SUPG stabilisation (ST instances; tal_set_stabilization):
    // tau = 1 / (st_c1 vis / h^2 + st_c2 rho |u_mean| / h), h = cbrt(|D|);
    // the symmetric table's off-diagonal po and pd - po for the Gauss-point
    // velocity second moments
    double st_c1, st_c2, st_po, st_dq;
};

__device__ __forceinline__ void cross3(const double a[3], const double b[3], double c[3])
{
    c[0] = fma(a[1], b[2], -a[2] * b[1]);
    c[1] = fma(a[2], b[0], -a[0] * b[2]);
    c[2] = fma(a[0], b[1], -a[1] * b[0]);
}

// |x|^(-1/3) for normal positive x: exponent split x = m 2^(3k), m in [1,8),
// single-precision MUFU seed (lg2/ex2, ~1e-6), one third-order correction
// y <- y (1 + e/3 + 2e^2/9 + 14e^3/81), e = 1 - m y^3 (error ~e^4 << 1 ulp).
// Branch-free; 8 FP64 instructions.
__device__ __forceinline__ double rcbrt_fast(double x)
{
    const int hi = __double2hiint(x), lo = __double2loint(x);
    const int ex = ((hi >> 20) & 0x7ff) - 1023;
    const int k = (ex + 1200) / 3 - 400;  // floor(ex / 3)
    const double m = __hiloint2double(hi - ((3 * k) << 20), lo);
    float l;
    const float mf = __double2float_rn(m);
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(l) : "f"(mf));
    float y0;
    const float a = l * (-1.0f / 3.0f);
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y0) : "f"(a));
    double y = (double)y0;
    const double e = fma(-m, (y * y) * y, 1.0);
    const double p = fma(e, fma(e, 14.0 / 81.0, 2.0 / 9.0), 1.0 / 3.0);
    y = fma(y * e, p, y);
    // y in (0.5, 1]: scale by 2^-k in the exponent field (INT pipe, no DMUL)
    return __hiloint2double(__double2hiint(y) - (k << 20), __double2loint(y));
}

// t^(-1/2) for normal positive t: MUFU.RSQ64H seed + one third-order
// correction y <- y (1 + e/2 + 3e^2/8 + 5e^3/16), e = 1 - t y^2.
__device__ __forceinline__ double rsqrt_fast(double t)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(t));
    const double e = fma(-t, y * y, 1.0);
    const double p = fma(e, fma(e, 5.0 / 16.0, 3.0 / 8.0), 0.5);
    return fma(y * e, p, y);
}

// normal (not zero/subnormal/inf/nan) test on the exponent field: INT pipe only
__device__ __forceinline__ bool is_normal_pos(double x)
{
    const unsigned e = ((unsigned)__double2hiint(x) >> 20) & 0x7ffu;
    return e - 1u < 2046u;
}

// |x| on the INT pipe (fabs compiles to a DADD)
__device__ __forceinline__ double abs_bits(double x)
{
    return __hiloint2double(__double2hiint(x) & 0x7fffffff, __double2loint(x));
}

// x with the sign of s flipped into it (x * sgn(s) for s != 0), integer ops only
__device__ __forceinline__ double mul_sign(double x, double s)
{
    return __longlong_as_double(__double_as_longlong(x) ^
                                (__double_as_longlong(s) & (long long)0x8000000000000000ULL));
}

// Optional P1 pressure-gradient term (absent from the
// reference operator, so its parity is pinned only by this repo's own oracle):
//   r_a[i] += int p dN_a/dx_i dV = vol * pbar * c_a[i] / D = sgn(D) pbar / 6 c_a[i]
// (weak form of -grad p without the boundary term; pbar = mean nodal pressure,
// exact for P1 p).  c_0 = -(c_1 + c_2 + c_3).  15 FP64 instructions.
__device__ __forceinline__ void pressure_add(double pbar, double det, const double c1[3],
                                             const double c2[3], const double c3[3], double R[4][3])
{
    const double P = mul_sign(pbar * (1.0 / 6.0), det);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        R[1][i] = fma(P, c1[i], R[1][i]);
        R[2][i] = fma(P, c2[i], R[2][i]);
        R[3][i] = fma(P, c3[i], R[3][i]);
        R[0][i] = fma(-P, (c1[i] + c2[i]) + c3[i], R[0][i]);
    }
}

// Everything after the cofactor rows: velocity gradient, Vreman, the two
// weighted terms.  c[1..3] = cofactor rows, D = det, du[b] = u_b - u_0
// (b = 1..3), U = the four corner velocities.  R = 4x3 element RHS; with
// ACC the FMA chains of R start from R's incoming values (the ring kernel
// folds its running sums into them instead of separate adds).  With NEG3 the
// c3 argument holds -c3 (the ring kernel carries c2 of the previous tet; the
// negation becomes a free operand modifier instead of three DADDs).
// Optional SUPG stabilisation of the convective residual (SURVEY.md section
// 8 f4; no reference counterpart, parity pinned by this repo's own oracle):
//   r_a[i] += -int tau (rho u.grad N_a) (rho u.grad u_i)
//           = -tau rho^2 / (24 |D|) * c_a . (M Gh)[:, i],
// M = sum_g u_g u_g^T = sum_bc pmat[b][c] u_b u_c^T (exact for P1 u with the
// degree-2 Gauss rule), tau = 1 / (c1 vis / h^2 + c2 rho |S/4| / h),
// 1/h = r3 = |D|^(-1/3) (the Vreman filter width), vis = mu + rho nu_t.
// The viscous part of the strong residual vanishes for P1; the pressure part
// is not included.  ~110 FP64 instructions.
__device__ __forceinline__ void supg_add(const double c1[3], const double c2[3], const double c3[3],
                                         const double Gh[3][3], const double U0[3], const double U1[3],
                                         const double U2[3], const double U3[3], const double S[3], double r3,
                                         double inv, double vis, const ElemConsts &k, double R[4][3])
{
    const double un = sqrt(fma(S[0], S[0], fma(S[1], S[1], S[2] * S[2])));
    const double tau = 1.0 / fma(k.st_c1 * vis, r3 * r3, k.st_c2 * k.rho * (0.25 * un) * r3);
    const double coef = -tau * (k.rho * k.rho) * inv * (1.0 / 24.0);
    double M[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = a; b < 3; ++b) {
            const double q = fma(U0[a], U0[b], fma(U1[a], U1[b], fma(U2[a], U2[b], U3[a] * U3[b])));
            M[a][b] = fma(k.st_po, S[a] * S[b], k.st_dq * q);
            M[b][a] = M[a][b];
        }
    double MG[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int i = 0; i < 3; ++i)
            MG[a][i] = coef * fma(M[a][0], Gh[0][i], fma(M[a][1], Gh[1][i], M[a][2] * Gh[2][i]));
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double t1 = fma(c1[0], MG[0][i], fma(c1[1], MG[1][i], c1[2] * MG[2][i]));
        const double t2 = fma(c2[0], MG[0][i], fma(c2[1], MG[1][i], c2[2] * MG[2][i]));
        const double t3 = fma(c3[0], MG[0][i], fma(c3[1], MG[1][i], c3[2] * MG[2][i]));
        R[1][i] += t1;
        R[2][i] += t2;
        R[3][i] += t3;
        R[0][i] -= (t1 + t2) + t3;
    }
}

// POS: the caller guarantees det > 0 (patches oriented on the host), so
// |det| = det and the sign folds vanish.  ST: add the SUPG term (supg_add).
template <bool ACC, bool NEG3 = false, bool POS = false, bool ST = false>
__device__ __forceinline__ void tet_tail(const double c1[3], const double c2[3], const double c3[3],
                                         double det, const double du1[3], const double du2[3],
                                         const double du3[3], const double U0[3], const double U1[3],
                                         const double S01[3], const double U2[3], const double U3[3],
                                         const ElemConsts &k, double R[4][3])
{
    const double ad = POS ? det : abs_bits(det);
    double c3v[3];
#pragma unroll
    for (int kk = 0; kk < 3; ++kk)
        c3v[kk] = NEG3 ? -c3[kk] : c3[kk];
    double Gh[3][3];
#pragma unroll
    for (int kk = 0; kk < 3; ++kk)
#pragma unroll
        for (int i = 0; i < 3; ++i)
            Gh[kk][i] = fma(c1[kk], du1[i], fma(c2[kk], du2[i], c3v[kk] * du3[i]));

    // |Gh|^2 (three row partial sums) and the nine squared 2x2 minors
    // (rows m<n, columns i<j; three column-pair partial sums)
    double ar[3];
#pragma unroll
    for (int r = 0; r < 3; ++r)
        ar[r] = fma(Gh[r][0], Gh[r][0], fma(Gh[r][1], Gh[r][1], Gh[r][2] * Gh[r][2]));
    const double aah = ar[0] + ar[1] + ar[2];
    double sp[3];
#pragma unroll
    for (int cp = 0; cp < 3; ++cp) {
        const int ci = (cp == 2) ? 1 : 0, cj = (cp == 0) ? 1 : 2;
        double d[3];
#pragma unroll
        for (int rp = 0; rp < 3; ++rp) {
            const int m = (rp == 2) ? 1 : 0, n = (rp == 0) ? 1 : 2;
            d[rp] = fma(Gh[m][ci], Gh[n][cj], -(Gh[m][cj] * Gh[n][ci]));
        }
        sp[cp] = fma(d[0], d[0], fma(d[1], d[1], d[2] * d[2]));
    }
    const double ssqh = sp[0] + sp[1] + sp[2];
    const double t = ssqh * aah;
    const double r3 = is_normal_pos(ad) ? rcbrt_fast(ad) : rcbrt(ad);
    const double inv = (r3 * r3) * r3;  // 1/|D|
    double f = 0.0;                     // -rho * nu_t / (6 ssqh)
    if (aah * inv * inv > 1e-30 && t > 0.0)  // kernel.py:24 guard, in G units
        f = (k.rc6 * r3) * (is_normal_pos(t) ? rsqrt_fast(t) : rsqrt(t));
    const double B = fma(f, ssqh, k.mu6) * inv;  // -(mu + rho nu_t) / (6 |D|)
    const double As = POS ? k.a_po : mul_sign(k.a_po, det), Aq = POS ? k.a_q : mul_sign(k.a_q, det);
    const double A4 = POS ? k.a_4 : mul_sign(k.a_4, det);
    double w[4][3];
#pragma unroll
    for (int cc = 0; cc < 3; ++cc) {
        const double S = S01[cc] + (U2[cc] + U3[cc]);  // S01 = u_0 + u_1
        const double AsS = As * S;
        w[1][cc] = fma(Aq, U1[cc], fma(B, c1[cc], AsS));
        w[2][cc] = fma(Aq, U2[cc], fma(B, c2[cc], AsS));
        w[3][cc] = fma(Aq, U3[cc], fma(B, c3v[cc], AsS));
        // sum_a w_a = (4 As + Aq) S because the cofactor rows sum to zero
        w[0][cc] = fma(A4, S, -((w[1][cc] + w[2][cc]) + w[3][cc]));
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const double last = ACC ? fma(w[a][2], Gh[2][i], R[a][i]) : w[a][2] * Gh[2][i];
            R[a][i] = fma(w[a][0], Gh[0][i], fma(w[a][1], Gh[1][i], last));
        }
    if constexpr (ST) {
        double Sv[3];
#pragma unroll
        for (int cc = 0; cc < 3; ++cc)
            Sv[cc] = S01[cc] + (U2[cc] + U3[cc]);
        const double vis = fma(-6.0 * f, ssqh, k.mu);  // f ssqh = -rho nu_t / 6
        supg_add(c1, c2, c3v, Gh, U0, U1, U2, U3, Sv, r3, inv, vis, k, R);
    }
}

// Symmetric-rule element (pmat = po * ones + (pd - po) * I); p4 = nodal
// pressures or nullptr; ST: with the SUPG term.
template <bool ST = false>
__device__ __forceinline__ void element_rhs_sym(const double X[4][3], const double U[4][3],
                                                const double *p4, const ElemConsts &k, double R[4][3])
{
    double e[3][3], du[3][3], c1[3], c2[3], c3[3];
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            e[b][c] = X[b + 1][c] - X[0][c];
            du[b][c] = U[b + 1][c] - U[0][c];
        }
    cross3(e[1], e[2], c1);  // e2 x e3
    cross3(e[2], e[0], c2);  // e3 x e1
    cross3(e[0], e[1], c3);  // e1 x e2
    const double det = fma(e[0][0], c1[0], fma(e[0][1], c1[1], e[0][2] * c1[2]));
    const double S01[3] = {U[0][0] + U[1][0], U[0][1] + U[1][1], U[0][2] + U[1][2]};
    tet_tail<false, false, false, ST>(c1, c2, c3, det, du[0], du[1], du[2], U[0], U[1], S01, U[2], U[3], k, R);
    if (p4)
        pressure_add(0.25 * ((p4[0] + p4[1]) + (p4[2] + p4[3])), det, c1, c2, c3, R);
}

// Geometry + gradient + Vreman for the general-pmat element: cofactor rows
// cf[1..3], the unscaled gradient Gh, sgn(D) and B = -vis / (6 |D|).
__device__ __forceinline__ void element_core(const double X[4][3], const double U[4][3],
                                             const ElemConsts &k, double cf[4][3],
                                             double Gh[3][3], double &sg, double &B, double &det_out)
{
    double e[3][3], du[3][3];
#pragma unroll
    for (int b = 0; b < 3; ++b)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            e[b][c] = X[b + 1][c] - X[0][c];
            du[b][c] = U[b + 1][c] - U[0][c];
        }
    cross3(e[1], e[2], cf[1]);
    cross3(e[2], e[0], cf[2]);
    cross3(e[0], e[1], cf[3]);
    const double det = fma(e[0][0], cf[1][0], fma(e[0][1], cf[1][1], e[0][2] * cf[1][2]));
    det_out = det;
    const double ad = fabs(det);
    sg = (det < 0.0) ? -1.0 : 1.0;
    const double r3 = rcbrt(ad);
    const double inv = r3 * r3 * r3;
#pragma unroll
    for (int kk = 0; kk < 3; ++kk)
#pragma unroll
        for (int i = 0; i < 3; ++i)
            Gh[kk][i] = fma(cf[1][kk], du[0][i], fma(cf[2][kk], du[1][i], cf[3][kk] * du[2][i]));
    double aah = 0.0, ssqh = 0.0;
#pragma unroll
    for (int q = 0; q < 9; ++q)
        aah = fma(Gh[q / 3][q % 3], Gh[q / 3][q % 3], aah);
#pragma unroll
    for (int cp = 0; cp < 3; ++cp) {
        const int ci = (cp == 2) ? 1 : 0, cj = (cp == 0) ? 1 : 2;
#pragma unroll
        for (int rp = 0; rp < 3; ++rp) {
            const int m = (rp == 2) ? 1 : 0, n = (rp == 0) ? 1 : 2;
            const double d = fma(Gh[m][ci], Gh[n][cj], -(Gh[m][cj] * Gh[n][ci]));
            ssqh = fma(d, d, ssqh);
        }
    }
    double nut = 0.0;
    if (aah * inv * inv > 1e-30 && ssqh > 0.0)
        nut = k.cvre * r3 * sqrt(ssqh / aah);
    const double vis = fma(k.rho, nut, k.mu);
    B = vis * (inv * (-1.0 / 6.0));
}

__device__ __forceinline__ void rhs_rows(const double w[4][3], const double Gh[3][3], double R[4][3])
{
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int i = 0; i < 3; ++i)
            R[a][i] = fma(w[a][0], Gh[0][i], fma(w[a][1], Gh[1][i], w[a][2] * Gh[2][i]));
}

// General pmat (any 4x4 interpolation table): m_a = sum_b pmat[a][b] u_b.
__device__ __forceinline__ void element_rhs_gen(const double X[4][3], const double U[4][3],
                                                const double *p4, const ElemConsts &k, double R[4][3])
{
    double cf[4][3], Gh[3][3], sg, B, det;
    element_core(X, U, k, cf, Gh, sg, B, det);
#pragma unroll
    for (int c = 0; c < 3; ++c)
        cf[0][c] = -(cf[1][c] + cf[2][c] + cf[3][c]);
    const double A = sg * (-k.rho / 24.0);
    double w[4][3];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const double m = fma(k.pm[4 * a + 0], U[0][c],
                                 fma(k.pm[4 * a + 1], U[1][c],
                                     fma(k.pm[4 * a + 2], U[2][c], k.pm[4 * a + 3] * U[3][c])));
            w[a][c] = fma(A, m, B * cf[a][c]);
        }
    rhs_rows(w, Gh, R);
    if (p4)
        pressure_add(0.25 * ((p4[0] + p4[1]) + (p4[2] + p4[3])), det, cf[1], cf[2], cf[3], R);
}

template <bool SYM, bool ST = false>
__device__ __forceinline__ void element_rhs(const double X[4][3], const double U[4][3],
                                            const double *p4, const ElemConsts &k, double R[4][3])
{
    if constexpr (SYM)
        element_rhs_sym<ST>(X, U, p4, k, R);
    else
        element_rhs_gen(X, U, p4, k, R);  // SUPG needs the symmetric rule (host-checked)
}

}  // namespace tal
