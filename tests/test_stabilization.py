"""SUPG stabilisation extension -- PARITY UNPINNED by
the reference (its operator has no stabilisation, kernel.py:7-10,
SPEC.md:191).  Oracle: oracle.supg_term, restated from the weak form with
explicit Gauss points (independent of the kernel's second-moment algebra),
itself pinned by closed forms: per-element conservation (sum_a N_a = 1 so the
node contributions of an element sum to zero), exact zero for a constant
field, covariance under a rigid rotation, and the limits of tau."""
import numpy as np
import pytest

import paper_2403_08777_b200 as tb

P = tb.PhysParams()


def _rot(theta=0.7, axis=(1.0, 2.0, 0.5)):
    a = np.asarray(axis) / np.linalg.norm(axis)
    K = np.array([[0, -a[2], a[1]], [a[2], 0, -a[0]], [-a[1], a[0], 0]])
    return np.eye(3) + np.sin(theta) * K + (1 - np.cos(theta)) * K @ K


# ---- CPU: the oracle's closed forms ----------------------------------------

def test_oracle_conserves_and_vanishes_for_constant_fields(oracle):
    m = tb.generate_box_mesh(5, 4, 3)
    u = tb.make_velocity(m, "random:3")
    s = oracle.supg_term(m.coords, m.connectivity, u)
    assert np.abs(s.sum(axis=0)).max() <= 1e-15 * np.abs(s).sum()
    assert np.abs(s).max() > 0.0
    c = np.tile([0.7, -0.3, 0.25], (m.n_nodes, 1))
    np.testing.assert_array_equal(oracle.supg_term(m.coords, m.connectivity, c), 0.0)


def test_oracle_rotation_covariance(oracle):
    m = tb.generate_box_mesh(4, 4, 4)
    u = tb.make_velocity(m, "taylor-green")
    Q = _rot()
    a = oracle.supg_term(m.coords, m.connectivity, u)
    b = oracle.supg_term(m.coords @ Q.T, m.connectivity, u @ Q.T)
    np.testing.assert_allclose(b, a @ Q.T, rtol=0, atol=1e-12 * np.abs(a).max())


def test_oracle_tau_limits(oracle):
    """c2 = 0 and mu -> big: tau = h^2 / (c1 mu) exactly, so the term scales as 1/c1."""
    m = tb.generate_box_mesh(3, 3, 2)
    u = tb.make_velocity(m, "random:5")
    a = oracle.supg_term(m.coords, m.connectivity, u, mu=1.0, cvre=0.0, c1=4.0, c2=0.0)
    b = oracle.supg_term(m.coords, m.connectivity, u, mu=1.0, cvre=0.0, c1=8.0, c2=0.0)
    np.testing.assert_allclose(a, 2.0 * b, rtol=1e-13, atol=1e-300)


# ---- GPU: the kernels against the oracle -----------------------------------

def _ref(oracle, m, u, p=P, c1=4.0, c2=2.0):
    base = oracle.assemble_rsp(m.coords, m.connectivity, u, p.rho, p.mu, p.c_vreman)
    return base + oracle.supg_term(m.coords, m.connectivity, u, p.rho, p.mu, p.c_vreman, c1, c2)


def _check(oracle, rhs, ref, m, u, p=P):
    # the reference tolerance, denominated by the stabilised vector
    d = np.abs(rhs - ref).max()
    assert d <= 1e-12 * np.abs(ref).max(), d / np.abs(ref).max()


@pytest.mark.gpu
@pytest.mark.parametrize("scatter", ["private", "private-atomic", "atomic", "colored"])
@pytest.mark.parametrize("init", ["random:1", "taylor-green", "shear:1.5"])
def test_supg_matches_oracle(oracle, scatter, init):
    m = tb.generate_box_mesh(9, 7, 6)
    u = tb.make_velocity(m, init)
    res = tb.assemble_rsp(m, u, P, tb.RunConfig(scatter=scatter), stabilization=True)
    _check(oracle, res.rhs, _ref(oracle, m, u), m, u)


@pytest.mark.gpu
@pytest.mark.parametrize("c", [(4.0, 2.0), (12.0, 0.5), (1.0, 0.0)])
def test_supg_constants_physics_and_permuted_mesh(oracle, c):
    g = tb.generate_box_mesh(8, 6, 5)
    m = tb.permute_nodes(g, np.random.default_rng(1).permutation(g.n_nodes))
    u = tb.make_velocity(m, "random:7") * 3.0
    p = tb.PhysParams(rho=1.3, mu=2e-3, c_vreman=0.1)
    res = tb.assemble_rsp(m, u, p, tb.RunConfig(scatter="private-atomic"), stabilization=c)
    _check(oracle, res.rhs, _ref(oracle, m, u, p, *c), m, u, p)


@pytest.mark.gpu
def test_supg_zero_for_constant_field_and_off_switch(oracle):
    m = tb.generate_box_mesh(5, 5, 4)
    u = np.tile([0.7, -0.3, 0.25], (m.n_nodes, 1))
    asm = tb.Assembler(m, tb.RunConfig(scatter="private"))
    a, _ = asm.assemble(u, P)
    asm.set_stabilization(True)
    b, _ = asm.assemble(u, P)
    np.testing.assert_array_equal(a, b)  # grad u = 0: the term is exactly zero
    u2 = tb.make_velocity(m, "random:2")
    c, _ = asm.assemble(u2, P)
    asm.set_stabilization(False)
    d, _ = asm.assemble(u2, P)
    assert not np.array_equal(c, d)
    np.testing.assert_array_equal(d, asm.assemble(u2, P)[0])
    asm.close()


@pytest.mark.gpu
def test_supg_refused_where_undefined():
    m = tb.generate_box_mesh(3, 3, 3)
    u = tb.make_velocity(m, "random:1")
    with pytest.raises(ValueError, match="sequential"):
        tb.assemble_rsp(m, u, P, tb.RunConfig(scatter="sequential"), stabilization=True)
    asm = tb.Assembler(m, tb.RunConfig(), build_colors=True)
    asm.set_stabilization(True)
    with pytest.raises(ValueError, match="symmetric"):
        asm.assemble_into(u, P, np.empty((m.n_nodes, 3)), "atomic",
                          pmat=np.random.default_rng(0).uniform(0, 0.5, (4, 4)))
    with pytest.raises(ValueError, match="RSP shape"):
        asm.assemble(u, P, variant="rs")
    with pytest.raises(ValueError):
        asm.set_stabilization(True, c1=0.0)
    asm.close()


@pytest.mark.gpu
def test_supg_with_pressure_and_graph_replay(oracle):
    m = tb.generate_box_mesh(7, 6, 6)
    u = tb.make_velocity(m, "random:4")
    pr = np.random.default_rng(3).uniform(-1, 1, m.n_nodes)
    ref = _ref(oracle, m, u) + oracle.pressure_gradient(m.coords, m.connectivity, pr)
    res = tb.assemble_rsp(m, u, P, tb.RunConfig(scatter="private-atomic"), pressure=pr,
                          stabilization=True)
    _check(oracle, res.rhs, ref, m, u)
    asm = tb.Assembler(m, tb.RunConfig(scatter="private"))
    asm.set_stabilization(True)
    asm.set_velocity_host(u)
    asm.capture(P)
    asm.replay()
    got = asm.get_rhs_host()
    _check(oracle, got, _ref(oracle, m, u), m, u)
    asm.close()


@pytest.mark.gpu
@pytest.mark.parametrize("scatter", ["private", "private-atomic", "atomic"])
def test_supg_and_pressure_on_an_unstructured_mesh(oracle, scatter):
    """Both f4 extensions on a Delaunay mesh (irregular rings, open arcs,
    ring-sorted chunks): SUPG and the pressure term together against the
    sum of their oracles."""
    m = tb.generate_delaunay_mesh(6000, seed=8)
    u = tb.make_velocity(m, "random:3")
    p = np.random.default_rng(6).uniform(-1.0, 1.0, m.n_nodes)
    res = tb.assemble_rsp(m, u, P, tb.RunConfig(scatter=scatter), pressure=p, stabilization=True)
    ref = _ref(oracle, m, u) + oracle.pressure_gradient(m.coords, m.connectivity, p)
    _check(oracle, res.rhs, ref, m, u)
