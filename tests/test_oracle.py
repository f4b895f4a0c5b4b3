"""Pin the CPU oracle (oracle/) against golden vectors produced by the
reference itself (oracle/gen_golden.py imports tet-assembly-lab 0.1.0).

These run on CPU (no GPU needed) and gate every parity claim: the GPU tests
compare against this oracle.
"""
import math

import numpy as np
import pytest

from conftest import INITS, SMALL_DIMS, dims_key, init_key


@pytest.mark.parametrize("dims", SMALL_DIMS + [(5, 4, 3)])
def test_box_mesh_matches_reference_generator(oracle, golden_meshes, dims):
    m = oracle.box_mesh(*dims)
    k = dims_key(dims)
    np.testing.assert_array_equal(m.connectivity, golden_meshes[f"conn_{k}"])
    np.testing.assert_array_equal(m.coords, golden_meshes[f"coords_{k}"])


def test_box_mesh_extents(oracle, golden_meshes):
    m = oracle.box_mesh(4, 3, 2, (2.0, 0.5, 3.0))
    np.testing.assert_array_equal(m.coords, golden_meshes["coords_4x3x2_ext"])
    np.testing.assert_array_equal(m.connectivity, golden_meshes["conn_4x3x2_ext"])


@pytest.mark.parametrize("dims", SMALL_DIMS + [(5, 4, 3)])
def test_greedy_coloring_matches_reference(oracle, golden_meshes, dims):
    m = oracle.box_mesh(*dims)
    colors = oracle.color_elements(m.connectivity, m.n_nodes)
    np.testing.assert_array_equal(colors, golden_meshes[f"colors_{dims_key(dims)}"])


@pytest.mark.parametrize("init", INITS)
@pytest.mark.parametrize("dims", SMALL_DIMS)
def test_rsp_restatement_bitwise(oracle, golden_small, dims, init):
    """The C restatement of _rsp_kernels.assemble_elements is bitwise equal to
    the numba kernel (same op order, no FMA, numba's pow-based cbrt)."""
    m = oracle.box_mesh(*dims)
    k, ik = dims_key(dims), init_key(init)
    u = oracle.velocity(m.coords, init)
    np.testing.assert_array_equal(u, golden_small[f"u_{k}_{ik}"])
    rhs = oracle.assemble_rsp(m.coords, m.connectivity, u)
    np.testing.assert_array_equal(rhs, golden_small[f"rsp_{k}_{ik}"])


@pytest.mark.parametrize("init", INITS)
@pytest.mark.parametrize("dims", SMALL_DIMS)
def test_scalar_oracle_restatement(oracle, golden_small, dims, init):
    """The Gauss-loop restatement of kernel.assemble_reference matches the
    reference's numpy oracle within the reference tolerance."""
    m = oracle.box_mesh(*dims)
    k, ik = dims_key(dims), init_key(init)
    u = golden_small[f"u_{k}_{ik}"]
    rhs = oracle.assemble_reference(m.coords, m.connectivity, u)
    chk = oracle.compare(rhs, golden_small[f"oracle_{k}_{ik}"], m.coords, m.connectivity, u)
    assert chk.passed, chk


def test_reference_tet_and_linear_field(oracle, golden_small):
    c, q = golden_small["reftet_coords"], golden_small["reftet_conn"]
    u = golden_small["reftet_u"]
    np.testing.assert_array_equal(oracle.assemble_rsp(c, q, u), golden_small["reftet_rsp"])
    ux = golden_small["reftet_linx_u"]
    r = oracle.assemble_reference(c, q, ux, rho=1.0, mu=1.0, cvre=0.0)
    np.testing.assert_allclose(r, golden_small["reftet_linx_oracle"], rtol=1e-13, atol=1e-18)


def test_nondefault_physics(oracle, golden_small):
    m = oracle.box_mesh(3, 3, 3)
    rho, mu, cv = golden_small["phys_params"]
    u = golden_small["phys_u"]
    rhs = oracle.assemble_rsp(m.coords, m.connectivity, u, rho, mu, cv)
    np.testing.assert_array_equal(rhs, golden_small["phys_rsp"])


def test_permuted_numbering(oracle, golden_small):
    c, q, u = golden_small["perm6_coords"], golden_small["perm6_conn"], golden_small["perm6_u"]
    np.testing.assert_array_equal(oracle.assemble_rsp(c, q, u), golden_small["perm6_rsp"])


def test_mid_size_bitwise(oracle, golden_mid):
    for n in (8, 16):
        m = oracle.box_mesh(n, n, n)
        for init in ("random:1", "taylor-green"):
            u = oracle.velocity(m.coords, init)
            rhs = oracle.assemble_rsp(m.coords, m.connectivity, u)
            np.testing.assert_array_equal(rhs, golden_mid[f"rsp_{n}_{init_key(init)}"])


def test_32cubed_checksums(oracle, golden_checksums):
    m = oracle.box_mesh(32, 32, 32)
    for init in ("taylor-green", "random:1"):
        u = oracle.velocity(m.coords, init)
        rhs = oracle.assemble_rsp(m.coords, m.connectivity, u)
        s, sa, mx = golden_checksums[f"sum_32_{init_key(init)}"]
        assert rhs.sum() == s and np.abs(rhs).sum() == sa and np.abs(rhs).max() == mx


@pytest.mark.parametrize("threads", [2, 3, 4])
def test_threaded_private_driver(oracle, threads):
    """variants.py thread-count invariance (<=1e-12) and fixed-config
    bitwise reruns (test_variants.py:105-131)."""
    m = oracle.box_mesh(6, 5, 4)
    u = oracle.velocity(m.coords, "random:2")
    one = oracle.assemble_rsp(m.coords, m.connectivity, u)
    a = oracle.assemble_rsp(m.coords, m.connectivity, u, n_threads=threads, vector_dim=7)
    b = oracle.assemble_rsp(m.coords, m.connectivity, u, n_threads=threads, vector_dim=7)
    np.testing.assert_array_equal(a, b)
    assert np.abs(a - one).max() <= 1e-12 * np.abs(one).max()


def test_compare_fault_injection_and_nonfinite(oracle, golden_small):
    m = oracle.box_mesh(2, 2, 2)
    u = golden_small["u_2x2x2_random"]
    ref = golden_small["oracle_2x2x2_random"]
    ok = oracle.compare(ref.copy(), ref, m.coords, m.connectivity, u)
    assert ok.passed and ok.rel_diff == 0.0
    bad = ref.copy()
    bad[0, 0] += 1e-6 * ok.denominator  # variants.py:746-748
    chk = oracle.compare(bad, ref, m.coords, m.connectivity, u)
    assert not chk.passed and chk.worst_node == 0
    nf = ref.copy()
    nf[5, 2] = np.inf
    chk = oracle.compare(nf, ref, m.coords, m.connectivity, u)
    assert not chk.passed and chk.worst_node == 5 and "non-finite" in chk.note


def test_null_field_denominator(oracle, golden_small):
    """constant fields: oracle is exactly 0; the floored denominator applies
    and rel-L2 is undefined (reported None)."""
    m = oracle.box_mesh(3, 3, 3)
    u = golden_small["u_3x3x3_constant"]
    ref = golden_small["oracle_3x3x3_constant"]
    rhs = oracle.assemble_rsp(m.coords, m.connectivity, u)
    chk = oracle.compare(rhs, ref, m.coords, m.connectivity, u)
    assert chk.passed and chk.denominator > 0.0
    if not np.any(ref):
        assert chk.rel_l2 is None


def test_empty_mesh(oracle):
    c = np.array([[0.0, 0, 0], [1.0, 0, 0]])
    q = np.zeros((0, 4), dtype=np.int64)
    u = np.zeros((2, 3))
    np.testing.assert_array_equal(oracle.assemble_rsp(c, q, u), np.zeros((2, 3)))
    assert oracle.contribution_scale(c, q, u) == 0.0


def test_vreman_goldens_via_single_element(oracle, golden_small):
    """nu_t(identity gradient, delta=1) = c exactly; pure shear -> 0
    (kernel.py:99-143), exercised through the assembled operator: a shear
    field on a box has a rank-1 gradient so the RHS equals the mu-only RHS."""
    m = oracle.box_mesh(3, 3, 3)
    u = oracle.velocity(m.coords, "shear:1.5")
    with_c = oracle.assemble_rsp(m.coords, m.connectivity, u, cvre=0.07)
    no_c = oracle.assemble_rsp(m.coords, m.connectivity, u, cvre=0.0)
    np.testing.assert_array_equal(with_c, no_c)
    assert math.isfinite(float(np.abs(with_c).sum()))
