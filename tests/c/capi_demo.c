/* A plain-C caller of the drop-in boundary (include/tal_b200.h), no Python:
 * build a Kuhn box with tal_box_mesh, upload it, assemble one velocity field
 * through tal_assemble (host buffers in, host rhs out) and through the numba
 * seam tal_assemble_elements, and write u and both rhs vectors as raw
 * doubles so tests/test_capi_c.py can check them against the oracle.
 *
 *   capi_demo --abi                 print the ABI version (no device needed)
 *   capi_demo nx ny nz out.bin      assemble on device 0
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "tal_b200.h"

static int check(int rc, const char *what)
{
    if (rc) {
        fprintf(stderr, "%s failed (%d): %s\n", what, rc, tal_last_error());
        exit(1);
    }
    return rc;
}

int main(int argc, char **argv)
{
    if (argc == 2 && strcmp(argv[1], "--abi") == 0) {
        printf("%d\n", tal_abi_version());
        return 0;
    }
    if (argc != 5) {
        fprintf(stderr, "usage: capi_demo --abi | nx ny nz out.bin\n");
        return 2;
    }
    const int64_t nx = atoll(argv[1]), ny = atoll(argv[2]), nz = atoll(argv[3]);
    const int64_t N = (nx + 1) * (ny + 1) * (nz + 1), E = 6 * nx * ny * nz;
    double *coords = malloc(sizeof(double) * 3 * N), *u = malloc(sizeof(double) * 3 * N);
    double *rhs = malloc(sizeof(double) * 3 * N), *rhs_seam = calloc((size_t)(3 * N), sizeof(double));
    int64_t *conn = malloc(sizeof(int64_t) * 4 * E), *ids = malloc(sizeof(int64_t) * E);
    check(tal_box_mesh(nx, ny, nz, 1.0, 1.0, 1.0, coords, conn), "tal_box_mesh");
    for (int64_t i = 0; i < N; ++i) { /* a smooth non-trivial field */
        const double x = coords[3 * i], y = coords[3 * i + 1], z = coords[3 * i + 2];
        u[3 * i + 0] = sin(3.0 * x) * cos(2.0 * y) + 0.3 * z;
        u[3 * i + 1] = -cos(3.0 * x) * sin(2.0 * y) + 0.1 * x * z;
        u[3 * i + 2] = 0.5 * sin(x + y + z);
    }
    for (int64_t e = 0; e < E; ++e)
        ids[e] = e;
    /* the 4-point rule's P^T P (variants.py:559): diagonal (5+3s5)^2/400 +
       3 (5-s5)^2/400, off-diagonal 2 a b + 2 b^2 with a, b the rule's values */
    tal_params p = {1.0, 1e-3, 0.07, {0}};
    const double s5 = sqrt(5.0), a = (5.0 + 3.0 * s5) / 20.0, b = (5.0 - s5) / 20.0;
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c)
            p.pmat[4 * r + c] = (r == c) ? a * a + 3.0 * b * b : 2.0 * a * b + 2.0 * b * b;

    tal_handle *h = NULL;
    tal_mesh_opts o;
    check(tal_default_mesh_opts(&o), "tal_default_mesh_opts");
    check(tal_create(0, &h), "tal_create");
    check(tal_upload_mesh(h, coords, conn, N, E, NULL, &o), "tal_upload_mesh");
    tal_timings t;
    check(tal_assemble(h, u, &p, rhs, TAL_SCATTER_PRIVATE, &t), "tal_assemble");
    check(tal_assemble_elements(0, coords, conn, N, E, u, p.rho, p.mu, p.c_vreman, p.pmat, ids, E, rhs_seam),
          "tal_assemble_elements");
    check(tal_destroy(h), "tal_destroy");

    FILE *f = fopen(argv[4], "wb");
    if (!f)
        return 1;
    fwrite(u, sizeof(double), (size_t)(3 * N), f);
    fwrite(rhs, sizeof(double), (size_t)(3 * N), f);
    fwrite(rhs_seam, sizeof(double), (size_t)(3 * N), f);
    fclose(f);
    printf("ok %lld tets, kernel %.3f ms, %lld launches\n", (long long)E, t.kernel_ms,
           (long long)t.kernel_launches);
    free(coords), free(u), free(rhs), free(rhs_seam), free(conn), free(ids);
    return 0;
}
