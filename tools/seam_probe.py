"""Where the numba-seam call's time goes at 128^3 (whole-mesh ids, the
reference's one-thread driver shape): fresh calloc'd rhs vs a pre-touched one,
a pageable vs a page-locked u."""
import sys
import time
import numpy as np
sys.path.insert(0, ".")
import paper_2403_08777_b200 as tb

m = tb.generate_box_mesh(128, 128, 128)
u = tb.make_velocity(m, "random:1")
pm = tb.interpolation_table()
ids = np.arange(m.n_elems, dtype=np.int64)
coords, conn = m.coords, m.connectivity


def call(rhs, uu=u):
    t = time.perf_counter()
    tb.assemble_elements(coords, conn, uu, 1.0, 1e-3, 0.07, pm, ids, rhs)
    return 1e3 * (time.perf_counter() - t)


call(np.zeros((m.n_nodes, 3)))  # context + first use
res = {}
res["fresh_zeros"] = np.median([call(np.zeros((m.n_nodes, 3))) for _ in range(5)])
r = np.ones((m.n_nodes, 3))
res["pretouched"] = np.median([call(r) for _ in range(5)])
uc = np.array(u)  # a different, unregistered array each call
res["fresh_u_pageable"] = np.median([call(r, np.array(u)) for _ in range(3)])
t = time.perf_counter(); a = np.arange(m.n_elems, dtype=np.int64); res["np_arange_E"] = 1e3 * (time.perf_counter() - t)
t = time.perf_counter(); z = np.zeros((m.n_nodes, 3)); z += 1.0; res["np_zeros_touch"] = 1e3 * (time.perf_counter() - t)
print({k: round(v, 2) for k, v in res.items()})
