"""Small assemblies in every scatter mode / shape / pressure setting, for
compute-sanitizer (memcheck, racecheck, synccheck, initcheck) runs."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2403_08777_b200 as tb  # noqa: E402

# default: 10x9x8 (every path once); "big": 64^3 = 2048 chunks, so each of the
# 592 persistent CTAs walks 3-4 chunks (blob/record buffer reuse across iterations)
dims = (64, 64, 64) if "big" in sys.argv else (10, 9, 8)
m = tb.generate_box_mesh(*dims)
u = tb.make_velocity(m, "random:1")
p = np.random.default_rng(3).uniform(-1, 1, m.n_nodes)
P = tb.PhysParams()
modes = ("private", "private-atomic") if "big" in sys.argv else tb.SCATTER_MODES
for mode in modes:
    tb.assemble_rsp(m, u, P, tb.RunConfig(scatter=mode))
    if mode != "sequential":  # the reference-order mode has no pressure term
        tb.assemble_rsp(m, u, P, tb.RunConfig(scatter=mode), pressure=p)
if "big" not in sys.argv:  # the numba seam, fast and strict
    from paper_2403_08777_b200.fields import interpolation_table
    rhs = np.zeros_like(u)
    ids = np.arange(m.n_elems, dtype=np.int64)
    pm = interpolation_table()
    tb.assemble_elements(m.coords, m.connectivity, u, 1.0, 1e-3, 0.07, pm, ids, rhs)
    tb.assemble_elements(m.coords, m.connectivity, u, 1.0, 1e-3, 0.07, pm, ids, rhs, strict=True)
if "big" not in sys.argv:  # round 2 paths: SUPG, caller layout, seam subsets
    for mode in ("private", "private-atomic", "atomic", "colored"):
        tb.assemble_rsp(m, u, P, tb.RunConfig(scatter=mode), stabilization=True)
    import torch
    a2 = tb.Assembler(m, tb.RunConfig())
    du = torch.as_tensor(u, device="cuda:0").contiguous()
    dr = torch.empty_like(du)
    for mode in ("private", "private-atomic"):
        a2.run_caller(P, du.data_ptr(), dr.data_ptr(), scatter=mode, stream=0)
    torch.cuda.synchronize()
    a2.close()
    ids2 = np.arange(5, m.n_elems // 2, dtype=np.int64)
    tb.assemble_elements(m.coords, m.connectivity, u, 1.0, 1e-3, 0.07, pm, ids2, rhs)
    tb.assemble_elements(m.coords, m.connectivity, u, 1.0, 1e-3, 0.07, pm, ids2[::3].copy(), rhs)
if "big" not in sys.argv:  # an unstructured mesh: open arcs, 1..8-tet rings, ring-sorted chunks
    md = tb.generate_delaunay_mesh(3000, seed=2)
    ud = tb.make_velocity(md, "random:4")
    for mode in ("private", "private-atomic", "atomic"):
        tb.assemble_rsp(md, ud, P, tb.RunConfig(scatter=mode))
for fn in () if "big" in sys.argv else (tb.assemble_baseline, tb.assemble_rs):
    fn(m, u, P, tb.RunConfig(scatter="atomic"))
asm = tb.Assembler(m, tb.RunConfig(scatter="private-atomic", cta_patches=64, chunk_nodes=144))
asm.assemble(u, P)
asm.close()
tb.clear_cache()
print("sanitize workload done")
