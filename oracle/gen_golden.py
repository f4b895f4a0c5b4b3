"""Generate tests/golden/*.npz by importing the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python oracle/gen_golden.py

The fixtures pin (a) the C/numpy oracle restatement in oracle/ and (b) the
GPU path, against outputs of tet-assembly-lab 0.1.0 computed here:

* ``meshes.npz``      connectivity/coords of small Kuhn boxes (mesh.py:145-184)
                       and the reference greedy colouring (mesh.py:235-257)
* ``rhs_small.npz``   assemble_reference (kernel.py:173-191) and assemble_rsp
                       (variants.py:553-616, 1 thread) for 5 initialisers x
                       small meshes (the matrix of test_variants.py:29-35),
                       the reference tet, a 2-element mesh, a permuted 6^3 box
* ``rhs_mid.npz``     8^3 and 16^3 boxes, random:1 / taylor-green, full rhs
* ``checksums.npz``   (sum, sum|.|) of 1-thread assemble_rsp at 32^3 (TG and
                       random:1) -- harness.py:124-125 convention
* ``vreman.npz``      vreman_viscosity known answers on random tensors
* ``pmat.npz``        quadrature_tet4 points and pmat = P^T P
* ``rhs_shapes.npz``  assemble_baseline / assemble_rs (variants.py:522-550)
                       on the test_variants.py matrix + the 4^3 TG box
                       (``--shapes`` writes only this file)
* ``meshio/``         files written by the reference's save_mesh, a commented
                       file with inverted elements and malformed files with the
                       line numbers of the reference's load_mesh errors
                       (mesh.py:280-371; ``--meshio`` writes only these)
This script is the only file in the repo that imports /root/reference; it is
never run on the GPU box.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
if str(REF_SRC) not in sys.path:
    sys.path.insert(0, str(REF_SRC))

import numba  # noqa: E402
import tet_assembly_lab as tal  # noqa: E402
from tet_assembly_lab.variants import RunConfig  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
INITS = ["zero", "constant:0.7,-0.3,0.25", "shear:1.5", "taylor-green", "random:1"]
SMALL_DIMS = [(1, 1, 1), (2, 2, 2), (3, 2, 1), (3, 3, 3), (4, 4, 4)]


def versions() -> dict:
    return {
        "numpy": np.__version__,
        "numba": numba.__version__,
        "tet_assembly_lab": tal.__version__,
    }


def shapes() -> None:
    """The B and RS code shapes of the reference (variants.py:522-550)."""
    params = tal.PhysParams()
    store = {}
    for dims in [(2, 2, 2), (3, 2, 1)]:
        m = tal.generate_box_mesh(*dims)
        key = "x".join(map(str, dims))
        for init in INITS:
            u = tal.make_velocity(m, init)
            ik = init.split(":")[0]
            store[f"b_{key}_{ik}"] = tal.assemble_baseline(m, u, params, RunConfig(vector_dim=8)).rhs
            store[f"rs_{key}_{ik}"] = tal.assemble_rs(m, u, params, RunConfig(vector_dim=8)).rhs
    m = tal.generate_box_mesh(4, 4, 4)
    u = tal.make_velocity(m, "taylor-green")
    store["b_4x4x4_taylor-green"] = tal.assemble_baseline(m, u, params, RunConfig()).rhs
    store["rs_4x4x4_taylor-green"] = tal.assemble_rs(m, u, params, RunConfig()).rhs
    np.savez_compressed(OUT / "rhs_shapes.npz", **store, **{f"meta_{k}": v for k, v in versions().items()})
    print("wrote rhs_shapes.npz", len(store))


def meshio() -> None:
    """Reference save_mesh / load_mesh behaviour (mesh.py:280-371)."""
    import json
    import warnings
    from tet_assembly_lab import mesh as M
    d = OUT / "meshio"
    d.mkdir(exist_ok=True)
    store = {}
    box = tal.generate_box_mesh(3, 2, 2)
    store["box3x2x2_coords"], store["box3x2x2_conn"] = box.coords, box.connectivity
    tal.save_mesh(box, d / "box3x2x2.txt")
    # awkward values: tiny, huge, negative zero, 17-digit mantissas
    c = np.array([[0.0, 0.0, 0.0], [1e-5, 0.1, 1.0 / 3.0], [0.0, 1.0, 2.0 / 3.0],
                  [-0.0, 1e300 * 0 + 3.0, 1e-300], [np.pi, -np.e, 1e22], [1.5, 2.5, -7.0]])
    q = np.array([[0, 1, 2, 3], [1, 2, 4, 5]], dtype=np.int64)
    vols = M.signed_volumes(c, q)
    q[vols < 0] = q[vols < 0][:, [0, 1, 3, 2]]
    odd = tal.Mesh(coords=c, connectivity=q)
    store["odd_coords"], store["odd_conn"] = odd.coords, odd.connectivity
    tal.save_mesh(odd, d / "odd.txt")
    # comments, blank lines, two inverted elements (re-oriented on load)
    b2 = tal.generate_box_mesh(2, 1, 1)
    conn = b2.connectivity.copy()
    conn[[1, 4]] = conn[[1, 4]][:, [0, 1, 3, 2]]
    lines = ["# a hand-edited file", "", f"nodes {b2.n_nodes}   # count"]
    lines += [f"  {x!r} {y!r} {z!r}  " for x, y, z in b2.coords.tolist()]
    lines += ["", "elems %d" % b2.n_elems] + [" ".join(map(str, r)) + "  # tet" for r in conn.tolist()]
    (d / "commented_inverted.txt").write_text("\n".join(lines) + "\n")
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        ci = tal.load_mesh(d / "commented_inverted.txt")
    store["commented_inverted_coords"], store["commented_inverted_conn"] = ci.coords, ci.connectivity
    np.savez_compressed(d / "meshes.npz", **store)
    good = (d / "box3x2x2.txt").read_text().splitlines()
    bad = {
        "err_header.txt": ["node 5"] + good[1:],
        "err_count.txt": ["nodes five"] + good[1:],
        "err_ncoord.txt": good[:3] + ["0.5 0.5"] + good[4:],
        "err_coord.txt": good[:4] + ["0.5 x 0.5"] + good[5:],
        "err_elems.txt": good[:good.index("elems 72")] + ["elements 72"] + good[good.index("elems 72") + 1:],
        "err_nidx.txt": good[:-1] + ["1 2 3"],
        "err_idx.txt": good[:-2] + ["1 2 3 q"] + good[-1:],
        "err_eof_nodes.txt": good[:10],
        "err_eof_elems.txt": good[:-5],
        "err_trailing.txt": good + ["", "extra 1"],
        "err_range.txt": good[:-1] + ["0 1 2 999"],
        "err_empty.txt": ["# nothing here"],
    }
    errors = {}
    for name, ls in bad.items():
        (d / name).write_text("\n".join(ls) + "\n")
        try:
            tal.load_mesh(d / name)
            raise AssertionError(f"{name} loaded")
        except M.MeshFormatError as e:
            errors[name] = {"type": "MeshFormatError", "line": e.line, "message": str(e)}
        except ValueError as e:
            errors[name] = {"type": "ValueError", "message": str(e)}
    (d / "errors.json").write_text(json.dumps(errors, indent=1) + "\n")
    print("wrote meshio goldens", sorted(p.name for p in d.iterdir()))


def main() -> None:
    if "--shapes" in sys.argv:
        shapes()
        return
    OUT.mkdir(parents=True, exist_ok=True)
    params = tal.PhysParams()
    one = RunConfig(n_threads=1)
    meta = versions()

    # ---- meshes + colourings -------------------------------------------
    mesh_store = {}
    for dims in SMALL_DIMS + [(5, 4, 3)]:
        m = tal.generate_box_mesh(*dims)
        key = "x".join(map(str, dims))
        mesh_store[f"coords_{key}"] = m.coords
        mesh_store[f"conn_{key}"] = m.connectivity
        mesh_store[f"colors_{key}"] = tal.color_elements(m).colors
    m = tal.generate_box_mesh(4, 3, 2, extents=(2.0, 0.5, 3.0))
    mesh_store["coords_4x3x2_ext"] = m.coords
    mesh_store["conn_4x3x2_ext"] = m.connectivity
    np.savez_compressed(OUT / "meshes.npz", **mesh_store, **{f"meta_{k}": v for k, v in meta.items()})

    # ---- small rhs matrix ----------------------------------------------
    store = {}
    for dims in SMALL_DIMS:
        m = tal.generate_box_mesh(*dims)
        key = "x".join(map(str, dims))
        for init in INITS:
            u = tal.make_velocity(m, init)
            ik = init.split(":")[0]
            store[f"u_{key}_{ik}"] = u
            store[f"oracle_{key}_{ik}"] = tal.assemble_reference(m, u, params)
            store[f"rsp_{key}_{ik}"] = tal.assemble_rsp(m, u, params, one).rhs
    # reference tet, random:3 (test_kernel.py:235-242)
    coords = np.array([[0.0, 0, 0], [1.0, 0, 0], [0.0, 1, 0], [0.0, 0, 1]])
    conn = np.array([[0, 1, 2, 3]])
    rt = tal.Mesh(coords=coords, connectivity=conn)
    u = tal.make_velocity(rt, "random:3")
    store["reftet_coords"] = coords
    store["reftet_conn"] = conn
    store["reftet_u"] = u
    store["reftet_oracle"] = tal.assemble_reference(rt, u, params)
    store["reftet_rsp"] = tal.assemble_rsp(rt, u, params, one).rhs
    # u=(x,0,0), mu=1, rho=1, c=0 (test_kernel.py:205-223)
    p2 = tal.PhysParams(rho=1.0, mu=1.0, c_vreman=0.0)
    ux = np.zeros((4, 3))
    ux[:, 0] = coords[:, 0]
    store["reftet_linx_u"] = ux
    store["reftet_linx_oracle"] = tal.assemble_reference(rt, ux, p2)
    # non-default physics on a 3^3 box
    m = tal.generate_box_mesh(3, 3, 3)
    u = tal.make_velocity(m, "random:4")
    p3 = tal.PhysParams(rho=1.7, mu=0.02, c_vreman=0.3)
    store["phys_u"] = u
    store["phys_oracle"] = tal.assemble_reference(m, u, p3)
    store["phys_rsp"] = tal.assemble_rsp(m, u, p3, one).rhs
    store["phys_params"] = np.array([1.7, 0.02, 0.3])
    # permuted numbering on a 6^3 box (SURVEY 8d config 3 construction)
    m = tal.generate_box_mesh(6, 6, 6)
    perm = np.random.default_rng(0).permutation(m.n_nodes)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size)
    pm = tal.Mesh(coords=m.coords[perm], connectivity=inv[m.connectivity])
    u = tal.make_velocity(pm, "random:1")
    store["perm6_coords"] = pm.coords
    store["perm6_conn"] = pm.connectivity
    store["perm6_u"] = u
    store["perm6_oracle"] = tal.assemble_reference(pm, u, params)
    store["perm6_rsp"] = tal.assemble_rsp(pm, u, params, one).rhs
    # translated 3^3 box (test_kernel.py:255-264)
    m = tal.generate_box_mesh(3, 3, 3)
    sh = tal.Mesh(coords=m.coords + np.array([10.0, -20.0, 5.0]), connectivity=m.connectivity)
    u = tal.make_velocity(m, "random:5")
    store["shift_u"] = u
    store["shift_oracle"] = tal.assemble_reference(sh, u, params)
    store["base_oracle"] = tal.assemble_reference(m, u, params)
    np.savez_compressed(OUT / "rhs_small.npz", **store)

    # ---- mid-size full vectors -----------------------------------------
    mid = {}
    for n in (8, 16):
        m = tal.generate_box_mesh(n, n, n)
        for init in ("random:1", "taylor-green"):
            u = tal.make_velocity(m, init)
            ik = init.split(":")[0]
            mid[f"rsp_{n}_{ik}"] = tal.assemble_rsp(m, u, params, one).rhs
            if n == 8:
                mid[f"oracle_{n}_{ik}"] = tal.assemble_reference(m, u, params)
    np.savez_compressed(OUT / "rhs_mid.npz", **mid)

    # ---- 32^3 checksums -------------------------------------------------
    cs = {}
    m = tal.generate_box_mesh(32, 32, 32)
    for init in ("taylor-green", "random:1"):
        u = tal.make_velocity(m, init)
        rhs = tal.assemble_rsp(m, u, params, one).rhs
        ik = init.split(":")[0]
        cs[f"sum_32_{ik}"] = np.array([rhs.sum(), np.abs(rhs).sum(), np.abs(rhs).max()])
        cs[f"l2_32_{ik}"] = np.array([np.linalg.norm(rhs)])
    np.savez_compressed(OUT / "checksums.npz", **cs)

    # ---- Vreman known answers ------------------------------------------
    rng = np.random.default_rng(11)
    G = rng.uniform(-3.0, 3.0, size=(64, 3, 3))
    G[0] = 0.0
    G[1] = np.eye(3)
    G[2] = 0.0
    G[2, 1, 0] = 3.7
    deltas = rng.uniform(0.01, 2.0, size=64)
    deltas[1] = 1.0
    nut = np.array([tal.vreman_viscosity(G[i], deltas[i], 0.07) for i in range(64)])
    np.savez_compressed(OUT / "vreman.npz", G=G, delta=deltas, c=np.array(0.07), nut=nut)

    rule = tal.quadrature_tet4()
    np.savez_compressed(OUT / "pmat.npz", points=rule.points, weights=rule.weights,
                        pmat=rule.points.T @ rule.points)
    shapes()
    print("wrote", sorted(p.name for p in OUT.glob("*.npz")), meta)


if __name__ == "__main__" and "--meshio" in sys.argv:
    meshio()
    sys.exit(0)
if __name__ == "__main__":
    main()
