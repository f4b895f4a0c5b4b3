"""CPU tests of the product's host side: the C-ABI library loads and exports
every symbol include/tal_b200.h declares, the native mesh utilities match the
reference generator/colouring bitwise, and the Python mirror validates its
inputs like the reference (ValueError).  No compute call needs a GPU here.
"""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2403_08777_b200 as tb
from paper_2403_08777_b200 import _native as N
from conftest import SMALL_DIMS, dims_key

HEADER = Path(__file__).resolve().parent.parent / "include" / "tal_b200.h"


def header_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tal_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    declared = header_functions()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    bound = {s[0] for s in N.SIGNATURES}
    assert set(declared) == bound, set(declared) ^ bound
    assert lib.tal_abi_version() == 1


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("dims", SMALL_DIMS + [(5, 4, 3)])
def test_native_box_mesh_matches_reference(golden_meshes, dims):
    m = tb.generate_box_mesh(*dims)
    k = dims_key(dims)
    np.testing.assert_array_equal(m.connectivity, golden_meshes[f"conn_{k}"])
    np.testing.assert_array_equal(m.coords, golden_meshes[f"coords_{k}"])
    assert not m.coords.flags.writeable and not m.connectivity.flags.writeable


def test_native_box_mesh_extents(golden_meshes):
    m = tb.generate_box_mesh(4, 3, 2, extents=(2.0, 0.5, 3.0))
    np.testing.assert_array_equal(m.coords, golden_meshes["coords_4x3x2_ext"])


@pytest.mark.parametrize("dims", SMALL_DIMS + [(5, 4, 3)])
def test_native_coloring_matches_reference(golden_meshes, dims):
    m = tb.color_elements(tb.generate_box_mesh(*dims))
    np.testing.assert_array_equal(m.colors, golden_meshes[f"colors_{dims_key(dims)}"])
    assert m.n_colors == int(golden_meshes[f"colors_{dims_key(dims)}"].max()) + 1


def test_signed_volumes_positive_and_sum():
    m = tb.generate_box_mesh(3, 4, 5, extents=(1.0, 2.0, 3.0))
    v = tb.signed_volumes(m.coords, m.connectivity)
    assert v.min() > 0 and abs(v.sum() - 6.0) < 1e-12


@pytest.mark.parametrize("method", ["rcm", "sfc", "none"])
def test_renumbering_is_a_permutation(method):
    m = tb.generate_box_mesh(5, 4, 3)
    perm = tb.renumber_nodes(m, method)
    assert np.array_equal(np.sort(perm), np.arange(m.n_nodes))
    if method == "none":
        assert np.array_equal(perm, np.arange(m.n_nodes))


def test_rcm_reduces_bandwidth():
    m = tb.generate_box_mesh(6, 6, 6)
    conn = m.connectivity
    bw0 = int((conn.max(axis=1) - conn.min(axis=1)).max())
    pm = tb.permute_nodes(m, np.random.default_rng(0).permutation(m.n_nodes))
    rnd = pm.connectivity
    bw_rand = int((rnd.max(axis=1) - rnd.min(axis=1)).max())
    rcm = tb.permute_nodes(pm, tb.renumber_nodes(pm, "rcm")).connectivity
    bw_rcm = int((rcm.max(axis=1) - rcm.min(axis=1)).max())
    assert bw_rcm < bw_rand and bw_rcm <= 2 * bw0


def test_mesh_validation_errors():
    coords = np.array([[0.0, 0, 0], [1.0, 0, 0], [0.0, 1, 0], [0.0, 0, 1]])
    with pytest.raises(ValueError):
        tb.Mesh(coords=coords[:, :2], connectivity=[[0, 1, 2, 3]])
    with pytest.raises(ValueError):
        tb.Mesh(coords=coords, connectivity=[[0, 1, 2, 4]])
    with pytest.raises(ValueError):  # inverted element
        tb.Mesh(coords=coords, connectivity=[[0, 2, 1, 3]])
    with pytest.raises(ValueError):  # invalid colouring: 2 elems sharing nodes, same colour
        cube = tb.generate_box_mesh(1, 1, 1)
        tb.Mesh(coords=cube.coords, connectivity=cube.connectivity, colors=np.zeros(6, np.int64))
    ok = tb.Mesh(coords=coords, connectivity=[[0, 1, 2, 3]])
    assert ok.n_elems == 1 and ok.n_nodes == 4 and ok.n_colors is None


def test_runconfig_validation():
    for kw in [dict(vector_dim=0), dict(n_threads=0), dict(reps=0), dict(scatter="bogus"),
               dict(renumber="x"), dict(element_order="x"), dict(cta_patches=0),
               dict(cta_patches=257), dict(chunk_nodes=8), dict(chunk_nodes=257),
               dict(cta_patches=64, chunk_nodes=145), dict(patches="x"), dict(device=-1),
               dict(cache_capacity_bytes=-1)]:
        with pytest.raises(ValueError):
            tb.RunConfig(**kw)
    for s in ("private", "colored", "atomic", "private-atomic"):
        assert tb.RunConfig(scatter=s).scatter == s


def test_physparams_validation():
    for kw in [dict(rho=0.0), dict(mu=-1.0), dict(c_vreman=-0.1), dict(filter_width_rule="x")]:
        with pytest.raises(ValueError):
            tb.PhysParams(**kw)


def test_make_velocity_matches_golden(golden_small):
    for dims in SMALL_DIMS:
        m = tb.generate_box_mesh(*dims)
        for spec, ik in [("zero", "zero"), ("constant:0.7,-0.3,0.25", "constant"),
                         ("shear:1.5", "shear"), ("taylor-green", "taylor-green"),
                         ("random:1", "random")]:
            np.testing.assert_array_equal(tb.make_velocity(m, spec),
                                          golden_small[f"u_{dims_key(dims)}_{ik}"])


@pytest.mark.parametrize("spec", ["nosuch", "constant:1,2", "shear:1:2", "zero:5",
                                  "taylor-green:3", "random:1,2"])
def test_make_velocity_rejects_bad_specs(spec):
    with pytest.raises(ValueError):
        tb.make_velocity(tb.generate_box_mesh(2, 2, 2), spec)


def test_validate_velocity():
    m = tb.generate_box_mesh(2, 2, 2)
    u = tb.validate_velocity(m, np.zeros((m.n_nodes, 3), dtype=np.float32))
    assert u.dtype == np.float64
    bad = np.zeros((m.n_nodes, 3))
    bad[3, 1] = np.nan
    with pytest.raises(ValueError):
        tb.validate_velocity(m, bad)
    with pytest.raises(ValueError):
        tb.validate_velocity(m, np.zeros((3, m.n_nodes)))


def test_pmat_matches_reference(golden_small):
    g = np.load(Path(__file__).resolve().parent / "golden" / "pmat.npz")
    np.testing.assert_array_equal(tb.interpolation_table(), g["pmat"])
    np.testing.assert_array_equal(tb.quadrature_tet4().points, g["points"])


def test_ledger_is_reference_rsp():
    led = tb.make_ledger(tb.VariantId.RSP, tb.RunConfig())
    assert (led.flops_per_elem, led.loadstore_per_elem, led.intermediate_arrays,
            led.bytes_dram_est) == (448, 48, 0, 384.0)


def test_no_gpu_fails_loudly_without_fallback():
    """Without a CUDA device the product path raises (never a CPU fallback)."""
    if N.device_count() > 0:
        pytest.skip("GPU present")
    m = tb.generate_box_mesh(2, 2, 2)
    with pytest.raises(RuntimeError):
        tb.assemble_rsp(m, np.zeros((m.n_nodes, 3)), tb.PhysParams())
    with pytest.raises(RuntimeError):
        tb.assemble_elements(m.coords, m.connectivity, np.zeros((m.n_nodes, 3)), 1.0, 1e-3, 0.07,
                             tb.interpolation_table(), np.arange(m.n_elems),
                             np.zeros((m.n_nodes, 3)))


def test_product_never_imports_oracle():
    pkg = Path(tb.__file__).resolve().parent
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\S+)", src, flags=re.M), f
        assert "tal_oracle" not in src, f


def _patch_tets(patches):
    tets = []
    for a, b, ring, closed in patches:
        m = len(ring)
        k = m if closed else m - 1
        for i in range(k):
            tets.append(tuple(sorted((a, b, ring[i], ring[(i + 1) % m]))))
    return tets


@pytest.mark.parametrize("dims", [(1, 1, 1), (2, 3, 2), (4, 4, 4), (7, 5, 3)])
@pytest.mark.parametrize("mode", ["star", "tet"])
def test_patches_cover_every_tet_once(dims, mode):
    from paper_2403_08777_b200.mesh import edge_star_patches
    m = tb.generate_box_mesh(*dims)
    pt = _patch_tets(edge_star_patches(m, mode))
    ref = sorted(tuple(sorted(t)) for t in m.connectivity.tolist())
    assert sorted(pt) == ref


def test_kuhn_box_decomposes_into_closed_six_rings():
    """Every Kuhn cell is the closed ring of 6 tets around its main diagonal."""
    from paper_2403_08777_b200.mesh import edge_star_patches
    m = tb.generate_box_mesh(6, 5, 4)
    p = edge_star_patches(m, "star")
    assert len(p) == 6 * 5 * 4
    assert all(closed and len(ring) == 6 for _, _, ring, closed in p)


def test_patches_on_permuted_and_perturbed_mesh():
    """General (non-box) connectivity: random node numbering plus a mesh with
    tets removed still decompose exactly."""
    from paper_2403_08777_b200.mesh import edge_star_patches
    base = tb.generate_box_mesh(5, 4, 4)
    pm = tb.permute_nodes(base, np.random.default_rng(3).permutation(base.n_nodes))
    keep = np.random.default_rng(4).random(pm.n_elems) < 0.7
    sub = tb.Mesh(coords=pm.coords, connectivity=pm.connectivity[keep])
    for mesh in (pm, sub):
        pt = _patch_tets(edge_star_patches(mesh, "star"))
        assert sorted(pt) == sorted(tuple(sorted(t)) for t in mesh.connectivity.tolist())


@pytest.mark.parametrize("dims", [(16, 16, 16), (24, 24, 24), (40, 20, 12)])
def test_chunks_are_compact_cell_blocks(dims):
    """Element Morton order on an element-size grid: every CTA chunk of a
    Kuhn box is a full 8x4x4 block of cells (128 rings, 5*5*9 = 225 nodes),
    also when the extents are not powers of two (160^3 measured 255 nodes per
    chunk with a bounding-box-scaled Morton key)."""
    from paper_2403_08777_b200.mesh import plan_layout
    m = tb.generate_box_mesh(*dims)
    info = plan_layout(m)
    assert info["n_patches"] == m.n_elems // 6
    assert info["n_chunks"] == info["n_patches"] // 128
    assert info["n_chunk_nodes"] == 225 * info["n_chunks"]


def test_plan_layout_general_mesh_and_errors():
    from paper_2403_08777_b200.mesh import plan_layout
    base = tb.generate_box_mesh(6, 5, 4)
    pm = tb.permute_nodes(base, np.random.default_rng(3).permutation(base.n_nodes))
    for cfg in (tb.RunConfig(), tb.RunConfig(renumber="sfc", element_order="node"),
                tb.RunConfig(patches="tet", cta_patches=64, chunk_nodes=144)):
        info = plan_layout(pm, cfg)
        assert info["n_chunks"] >= 1 and info["n_chunk_nodes"] >= base.n_nodes
    bad = tb.Mesh.__new__(tb.Mesh)
    object.__setattr__(bad, "coords", base.coords)
    object.__setattr__(bad, "connectivity", base.connectivity + base.n_nodes)
    with pytest.raises(ValueError):
        plan_layout(bad)


def test_bank_aware_record_placement_reduces_conflicts():
    """The chunk record slots are coloured mod 8 (tal_prep.cpp bank_place):
    the estimated LDS.128 wavefronts of the ring walk's record loads drop
    against ascending-id slots and never go below one per quarter-warp."""
    import ctypes
    from paper_2403_08777_b200 import _native as N
    from paper_2403_08777_b200.mesh import plan_layout
    a0 = (ctypes.c_int64 * 6)()
    N.lib().tal_layout_bank_stats(a0)
    plan_layout(tb.generate_box_mesh(24, 16, 16))
    a1 = (ctypes.c_int64 * 6)()
    N.lib().tal_layout_bank_stats(a1)
    groups, before, after, sgroups, sbefore, safter = (a1[i] - a0[i] for i in range(6))
    assert groups > 0 and sgroups > 0
    assert groups <= after < before
    assert after / groups < 1.6 < before / groups
    # contribution stores (half-warp STS.64 groups): levels / equal-count ranks
    assert sgroups <= safter < sbefore


def test_delaunay_mesh_generator():
    """The unstructured synthetic mesh: deterministic per seed, every element
    positively oriented, irregular edge rings (open and closed) for the
    patch builder."""
    a = tb.generate_delaunay_mesh(3000, seed=1)
    b = tb.generate_delaunay_mesh(3000, seed=1)
    assert np.array_equal(a.connectivity, b.connectivity)
    assert (tb.signed_volumes(a.coords, a.connectivity) > 0).all()
    assert 5.0 < a.n_elems / a.n_nodes < 7.5
    rings = {len(r) for _, _, r, _ in tb.mesh.edge_star_patches(a)}
    assert len(rings) >= 4
