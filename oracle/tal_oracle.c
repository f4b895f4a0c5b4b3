/*
 * tal_oracle.c -- CPU restatement of the reference momentum-RHS assembly.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker and the CPU
 * baseline ("port") for bench.py.  The product path (paper_2403_08777_b200)
 * never links, loads or calls it; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs do.
 *
 * Every function restates one piece of the reference package
 * tet-assembly-lab 0.1.0 (/root/reference/pkg/src/tet_assembly_lab):
 *
 *   orc_assemble_elements   _rsp_kernels.py:20-164  (the numba hot loop;
 *                           same operation order, no FMA contraction --
 *                           build with -ffp-contract=off)
 *   orc_assemble_private    variants.py:573-596     (T threads, per-thread
 *                           accumulators over vector_dim-aligned slabs,
 *                           merged in thread order)
 *   orc_assemble_reference  kernel.py:146-191 + mesh.py:187-218 (scalar
 *                           oracle: explicit 4-point Gauss loop)
 *   orc_box_mesh            mesh.py:145-184  (Kuhn 6-tet split of a box)
 *   orc_color_elements      mesh.py:235-257  (greedy lowest-free colour)
 *   orc_signed_volumes      mesh.py:110-123
 *
 * Parity of this restatement is pinned against golden vectors produced by
 * importing the reference itself (oracle/gen_golden.py -> tests/golden/).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_DENOM_EPSILON 1e-30 /* kernel.py:24 */

/* ------------------------------------------------------------------------ */
/* Vreman eddy viscosity from a velocity gradient g[k][i] = du_i/dx_k.       */
/* kernel.py:99-143; minor order d0..d8 and the running sum follow           */
/* _rsp_kernels.py:87-120 exactly (rank-1 gradients clamp to exact 0).       */
/* ------------------------------------------------------------------------ */
static double orc_vreman(const double g[3][3], double dlt, double cvre)
{
    double aa = 0.0;
    /* _rsp_kernels.py:87-91: row-major left-to-right sum of squares */
    aa = g[0][0] * g[0][0] + g[0][1] * g[0][1];
    aa = aa + g[0][2] * g[0][2];
    aa = aa + g[1][0] * g[1][0];
    aa = aa + g[1][1] * g[1][1];
    aa = aa + g[1][2] * g[1][2];
    aa = aa + g[2][0] * g[2][0];
    aa = aa + g[2][1] * g[2][1];
    aa = aa + g[2][2] * g[2][2];
    if (aa <= ORC_DENOM_EPSILON)
        return 0.0;
    /* (row pair, column pair) of each 2x2 minor, in the reference order */
    static const int mr[9][2] = {{0, 1}, {0, 2}, {1, 2}, {0, 1}, {0, 2},
                                 {1, 2}, {0, 1}, {0, 2}, {1, 2}};
    static const int mc[9][2] = {{0, 1}, {0, 1}, {0, 1}, {0, 2}, {0, 2},
                                 {0, 2}, {1, 2}, {1, 2}, {1, 2}};
    /* _rsp_kernels.py uses (m,n) x (i,j) = rows (0,1),(0,2),(1,2) for the
       first column pair, etc.  Its d = g[m][i]*g[n][j] - g[m][j]*g[n][i]. */
    double ssq = 0.0;
    for (int q = 0; q < 9; ++q) {
        const int m = mr[q][0], n = mr[q][1];
        const int i = mc[q][0], j = mc[q][1];
        const double d = g[m][i] * g[n][j] - g[m][j] * g[n][i];
        ssq = (q == 0) ? d * d : ssq + d * d;
    }
    const double d2 = dlt * dlt;
    const double bb = d2 * d2 * ssq;
    if (bb < 0.0)
        return 0.0;
    return cvre * sqrt(bb / aa);
}

/* np.cbrt as numba lowers it inside the njit kernel: numba/np/npyfuncs.py   */
/* np_real_cbrt_impl = sign-symmetric pow(x, 1/3) (not libm cbrt; they      */
/* differ in the last ulp).  The scalar oracle below uses numpy's np.cbrt,  */
/* which is libm cbrt (kernel.py:89-91).                                     */
static double orc_numba_cbrt(double x)
{
    if (isnan(x))
        return x;
    if (x < 0.0)
        return -pow(-x, 1.0 / 3.0);
    return pow(x, 1.0 / 3.0);
}

/* ------------------------------------------------------------------------ */
/* The privatised element loop: _rsp_kernels.py:20-164.                     */
/* coords f64[N][3], conn i64[E][4], u f64[N][3], pmat f64[4][4],           */
/* ids i64[k]; accumulates (+=) into rhs f64[N][3].                          */
/* ------------------------------------------------------------------------ */
void orc_assemble_elements(const double *coords, const int64_t *conn,
                           const double *u, double rho, double mu, double cvre,
                           const double *pmat, const int64_t *ids, int64_t k,
                           double *rhs)
{
    for (int64_t t = 0; t < k; ++t) {
        const int64_t e = ids[t];
        int64_t n[4];
        double x[4][3], uu[4][3];
        for (int a = 0; a < 4; ++a) {
            n[a] = conn[4 * e + a];
            for (int c = 0; c < 3; ++c) {
                x[a][c] = coords[3 * n[a] + c];
                uu[a][c] = u[3 * n[a] + c];
            }
        }
        double ed[4][3]; /* ed[1..3] = x_b - x_0 (_rsp_kernels.py:45-47) */
        for (int b = 1; b < 4; ++b)
            for (int c = 0; c < 3; ++c)
                ed[b][c] = x[b][c] - x[0][c];
        /* cofactors c1 = e2 x e3, c2 = e3 x e1, c3 = e1 x e2 (:49-58) */
        double cf[4][3];
        for (int b = 1; b < 4; ++b) {
            /* b=1: e2 x e3 ; b=2: e3 x e1 ; b=3: e1 x e2 */
            const double *pp = (b == 1) ? ed[2] : (b == 2) ? ed[3] : ed[1];
            const double *qq = (b == 1) ? ed[3] : (b == 2) ? ed[1] : ed[2];
            cf[b][0] = pp[1] * qq[2] - pp[2] * qq[1];
            cf[b][1] = pp[2] * qq[0] - pp[0] * qq[2];
            cf[b][2] = pp[0] * qq[1] - pp[1] * qq[0];
        }
        const double det =
            ed[1][0] * cf[1][0] + ed[1][1] * cf[1][1] + ed[1][2] * cf[1][2];
        const double vol = fabs(det) / 6.0; /* :61 */
        const double dlt = orc_numba_cbrt(6.0 * vol); /* :62 */
        double bg[4][3];                    /* shape gradients :64-69 */
        for (int b = 1; b < 4; ++b)
            for (int c = 0; c < 3; ++c)
                bg[b][c] = cf[b][c] / det;
        for (int c = 0; c < 3; ++c)
            bg[0][c] = -(bg[1][c] + bg[2][c] + bg[3][c]);
        /* g[k][i] = sum_a b_a[k] u_a[i] (:76-85) */
        double g[3][3];
        for (int kk = 0; kk < 3; ++kk)
            for (int i = 0; i < 3; ++i) {
                double s = bg[0][kk] * uu[0][i] + bg[1][kk] * uu[1][i];
                s = s + bg[2][kk] * uu[2][i];
                s = s + bg[3][kk] * uu[3][i];
                g[kk][i] = s;
            }
        const double nut = orc_vreman(g, dlt, cvre); /* :87-120 */
        const double vis = mu + rho * nut;           /* :122 */
        const double nrv = -(rho * vol * 0.25);      /* :123 */
        const double nvv = -(vis * vol);             /* :124 */
        for (int a = 0; a < 4; ++a) {                /* :126-164 */
            double m[3];
            for (int c = 0; c < 3; ++c) {
                double s = pmat[4 * a + 0] * uu[0][c] + pmat[4 * a + 1] * uu[1][c];
                s = s + pmat[4 * a + 2] * uu[2][c];
                s = s + pmat[4 * a + 3] * uu[3][c];
                m[c] = s;
            }
            for (int i = 0; i < 3; ++i) {
                double cv = m[0] * g[0][i] + m[1] * g[1][i];
                cv = cv + m[2] * g[2][i];
                double df = bg[a][0] * g[0][i] + bg[a][1] * g[1][i];
                df = df + bg[a][2] * g[2][i];
                const double r = nrv * cv + nvv * df;
                rhs[3 * n[a] + i] += r;
            }
        }
    }
}

/* ------------------------------------------------------------------------ */
/* Threaded private-accumulator driver: variants.py:573-596 and            */
/* _slab_bounds (variants.py:467-475).  rhs (N*3) is overwritten.           */
/* ------------------------------------------------------------------------ */
typedef struct {
    const double *coords, *u, *pmat;
    const int64_t *conn, *ids;
    double rho, mu, cvre;
    int64_t k;
    double *buf;
} orc_job;

static void *orc_worker(void *arg)
{
    orc_job *j = (orc_job *)arg;
    orc_assemble_elements(j->coords, j->conn, j->u, j->rho, j->mu, j->cvre,
                          j->pmat, j->ids, j->k, j->buf);
    return NULL;
}

int orc_assemble_private(const double *coords, const int64_t *conn,
                         const double *u, double rho, double mu, double cvre,
                         const double *pmat, int64_t n_nodes, int64_t n_elems,
                         int n_threads, int64_t vector_dim, double *rhs)
{
    if (n_threads < 1 || vector_dim < 1)
        return -1;
    int64_t *ids = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_elems > 0 ? n_elems : 1));
    if (!ids)
        return -2;
    for (int64_t e = 0; e < n_elems; ++e)
        ids[e] = e;
    memset(rhs, 0, sizeof(double) * (size_t)(3 * n_nodes));
    if (n_threads == 1) {
        orc_assemble_elements(coords, conn, u, rho, mu, cvre, pmat, ids,
                              n_elems, rhs);
        free(ids);
        return 0;
    }
    /* slabs of whole vector_dim chunks, near-equal split */
    const int64_t n_chunks = (n_elems + vector_dim - 1) / vector_dim;
    const int64_t q = n_chunks / n_threads, r = n_chunks % n_threads;
    orc_job *jobs = (orc_job *)calloc((size_t)n_threads, sizeof(orc_job));
    pthread_t *th = (pthread_t *)calloc((size_t)n_threads, sizeof(pthread_t));
    int rc = 0;
    int64_t lo = 0;
    for (int t = 0; t < n_threads; ++t) {
        const int64_t hi = lo + q + (t < r ? 1 : 0);
        const int64_t e0 = lo * vector_dim;
        int64_t e1 = hi * vector_dim;
        if (e1 > n_elems)
            e1 = n_elems;
        jobs[t].coords = coords;
        jobs[t].conn = conn;
        jobs[t].u = u;
        jobs[t].pmat = pmat;
        jobs[t].rho = rho;
        jobs[t].mu = mu;
        jobs[t].cvre = cvre;
        jobs[t].ids = ids + e0;
        jobs[t].k = e1 > e0 ? e1 - e0 : 0;
        jobs[t].buf = (t == 0) ? rhs
                               : (double *)calloc((size_t)(3 * n_nodes > 0 ? 3 * n_nodes : 1),
                                                  sizeof(double));
        if (!jobs[t].buf)
            rc = -2;
        lo = hi;
    }
    if (rc == 0) {
        for (int t = 0; t < n_threads; ++t)
            pthread_create(&th[t], NULL, orc_worker, &jobs[t]);
        for (int t = 0; t < n_threads; ++t)
            pthread_join(th[t], NULL);
        /* merge in thread order (variants.py:594-596) */
        for (int t = 1; t < n_threads; ++t)
            for (int64_t i = 0; i < 3 * n_nodes; ++i)
                rhs[i] += jobs[t].buf[i];
    }
    for (int t = 1; t < n_threads; ++t)
        free(jobs[t].buf);
    free(jobs);
    free(th);
    free(ids);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* Scalar oracle with an explicit Gauss loop: kernel.py:146-191 with        */
/* tet_gradients (mesh.py:187-218) and quadrature_tet4 (kernel.py:71-86).   */
/* ------------------------------------------------------------------------ */
void orc_assemble_reference(const double *coords, const int64_t *conn,
                            const double *u, double rho, double mu,
                            double cvre, int64_t n_nodes, int64_t n_elems,
                            double *rhs)
{
    const double qa = (5.0 + 3.0 * sqrt(5.0)) / 20.0;
    const double qb = (5.0 - sqrt(5.0)) / 20.0;
    double pts[4][4];
    for (int g = 0; g < 4; ++g)
        for (int a = 0; a < 4; ++a)
            pts[g][a] = (g == a) ? qa : qb;
    memset(rhs, 0, sizeof(double) * (size_t)(3 * n_nodes));
    for (int64_t e = 0; e < n_elems; ++e) {
        int64_t n[4];
        double x[4][3], ue[4][3];
        for (int a = 0; a < 4; ++a) {
            n[a] = conn[4 * e + a];
            for (int c = 0; c < 3; ++c) {
                x[a][c] = coords[3 * n[a] + c];
                ue[a][c] = u[3 * n[a] + c];
            }
        }
        /* tet_gradients: reciprocal edge vectors, corner closes the sum */
        double e1[3], e2[3], e3[3];
        for (int c = 0; c < 3; ++c) {
            e1[c] = x[1][c] - x[0][c];
            e2[c] = x[2][c] - x[0][c];
            e3[c] = x[3][c] - x[0][c];
        }
        const double c23[3] = {e2[1] * e3[2] - e2[2] * e3[1], e2[2] * e3[0] - e2[0] * e3[2],
                               e2[0] * e3[1] - e2[1] * e3[0]};
        const double c31[3] = {e3[1] * e1[2] - e3[2] * e1[1], e3[2] * e1[0] - e3[0] * e1[2],
                               e3[0] * e1[1] - e3[1] * e1[0]};
        const double c12[3] = {e1[1] * e2[2] - e1[2] * e2[1], e1[2] * e2[0] - e1[0] * e2[2],
                               e1[0] * e2[1] - e1[1] * e2[0]};
        const double det = e1[0] * c23[0] + e1[1] * c23[1] + e1[2] * c23[2];
        double gr[4][3];
        for (int c = 0; c < 3; ++c) {
            gr[1][c] = c23[c] / det;
            gr[2][c] = c31[c] / det;
            gr[3][c] = c12[c] / det;
        }
        for (int c = 0; c < 3; ++c)
            gr[0][c] = -(gr[1][c] + gr[2][c] + gr[3][c]);
        const double vol = fabs(det) / 6.0;
        /* G = grad_n^T @ u_elem (kernel.py:94-96), numpy matmul order */
        double G[3][3];
        for (int k = 0; k < 3; ++k)
            for (int i = 0; i < 3; ++i) {
                double s = 0.0;
                for (int a = 0; a < 4; ++a)
                    s += gr[a][k] * ue[a][i];
                G[k][i] = s;
            }
        const double nut = orc_vreman(G, cbrt(6.0 * vol), cvre);
        const double visc = mu + rho * nut;
        /* u at Gauss points, convective term, weighted node projection */
        double conv[4][3] = {{0}};
        for (int g = 0; g < 4; ++g) {
            double ug[3];
            for (int i = 0; i < 3; ++i) {
                double s = 0.0;
                for (int a = 0; a < 4; ++a)
                    s += pts[g][a] * ue[a][i];
                ug[i] = s;
            }
            double cg[3];
            for (int i = 0; i < 3; ++i) {
                double s = 0.0;
                for (int k = 0; k < 3; ++k)
                    s += ug[k] * G[k][i];
                cg[i] = s;
            }
            for (int a = 0; a < 4; ++a)
                for (int i = 0; i < 3; ++i)
                    conv[a][i] += (pts[g][a] * 0.25) * cg[i];
        }
        for (int a = 0; a < 4; ++a)
            for (int i = 0; i < 3; ++i) {
                double df = 0.0;
                for (int k = 0; k < 3; ++k)
                    df += gr[a][k] * G[k][i];
                rhs[3 * n[a] + i] += -(rho * vol) * conv[a][i] - (visc * vol) * df;
            }
    }
}

/* ------------------------------------------------------------------------ */
/* Kuhn box mesh: mesh.py:126-184.  coords (N,3), conn (E,4) preallocated.   */
/* ------------------------------------------------------------------------ */
void orc_box_mesh(int64_t nx, int64_t ny, int64_t nz, double ex, double ey,
                  double ez, double *coords, int64_t *conn)
{
    const int64_t sx = 1, sy = nx + 1, sz = (nx + 1) * (ny + 1);
    /* np.linspace(0, ext, n+1): step * i, last point exactly ext */
    for (int64_t k = 0; k <= nz; ++k)
        for (int64_t j = 0; j <= ny; ++j)
            for (int64_t i = 0; i <= nx; ++i) {
                double *p = coords + 3 * (i * sx + j * sy + k * sz);
                p[0] = (i == nx) ? ex : (double)i * (ex / (double)nx);
                p[1] = (j == ny) ? ey : (double)j * (ey / (double)ny);
                p[2] = (k == nz) ? ez : (double)k * (ez / (double)nz);
            }
    /* axis-permutation paths from corner to opposite corner */
    static const int perms[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2},
                                    {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    static const int odd[6] = {0, 1, 1, 0, 0, 1};
    const int64_t step[3] = {sx, sy, sz};
    int64_t e = 0;
    for (int64_t k = 0; k < nz; ++k)
        for (int64_t j = 0; j < ny; ++j)
            for (int64_t i = 0; i < nx; ++i) {
                const int64_t c0 = i * sx + j * sy + k * sz;
                for (int t = 0; t < 6; ++t, ++e) {
                    const int64_t p1 = c0 + step[perms[t][0]];
                    const int64_t p2 = p1 + step[perms[t][1]];
                    const int64_t p3 = p2 + step[perms[t][2]];
                    int64_t *q = conn + 4 * e;
                    q[0] = c0;
                    q[1] = p1;
                    q[2] = odd[t] ? p3 : p2;
                    q[3] = odd[t] ? p2 : p3;
                }
            }
}

/* signed volumes det/6: mesh.py:110-123 */
void orc_signed_volumes(const double *coords, const int64_t *conn,
                        int64_t n_elems, double *vols)
{
    for (int64_t e = 0; e < n_elems; ++e) {
        const double *x0 = coords + 3 * conn[4 * e + 0];
        const double *x1 = coords + 3 * conn[4 * e + 1];
        const double *x2 = coords + 3 * conn[4 * e + 2];
        const double *x3 = coords + 3 * conn[4 * e + 3];
        double e1[3], e2[3], e3[3];
        for (int c = 0; c < 3; ++c) {
            e1[c] = x1[c] - x0[c];
            e2[c] = x2[c] - x0[c];
            e3[c] = x3[c] - x0[c];
        }
        const double det = e1[0] * (e2[1] * e3[2] - e2[2] * e3[1]) +
                           e1[1] * (e2[2] * e3[0] - e2[0] * e3[2]) +
                           e1[2] * (e2[0] * e3[1] - e2[1] * e3[0]);
        vols[e] = det / 6.0;
    }
}

/* greedy colouring in element order (mesh.py:235-257); colours < 64.      */
/* returns number of colours, or -1 if more than 64 would be needed.        */
int orc_color_elements(const int64_t *conn, int64_t n_nodes, int64_t n_elems,
                       int64_t *colors)
{
    uint64_t *used = (uint64_t *)calloc((size_t)(n_nodes > 0 ? n_nodes : 1), sizeof(uint64_t));
    if (!used)
        return -2;
    int ncol = 0;
    for (int64_t e = 0; e < n_elems; ++e) {
        const int64_t *q = conn + 4 * e;
        const uint64_t m = used[q[0]] | used[q[1]] | used[q[2]] | used[q[3]];
        if (m == ~(uint64_t)0) {
            free(used);
            return -1;
        }
        const uint64_t f = ~m & (m + 1);
        const int c = __builtin_ctzll(f);
        colors[e] = c;
        if (c + 1 > ncol)
            ncol = c + 1;
        for (int a = 0; a < 4; ++a)
            used[q[a]] |= f;
    }
    free(used);
    return ncol;
}
