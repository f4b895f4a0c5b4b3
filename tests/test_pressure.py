"""Optional P1 pressure-gradient term.

The reference operator has no pressure term (kernel.py:7-10), so
this extension's parity is UNPINNED by the reference: the oracle
(oracle.pressure_gradient) is restated from the weak form
r_a[i] = int p dN_a/dx_i dV and pinned here only by closed-form answers.
"""
import numpy as np
import pytest

import paper_2403_08777_b200 as tb

P = tb.PhysParams()


def _interior(cells):
    nx, ny, nz = cells
    i, j, k = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    inside = (i > 0) & (i < nx) & (j > 0) & (j < ny) & (k > 0) & (k < nz)
    # node id = i + (nx+1)(j + (ny+1) k)  (mesh.py:160-171)
    return (i + (nx + 1) * (j + (ny + 1) * k))[inside]


# ---------------------------------------------------------------------------
# CPU: the oracle against closed forms
# ---------------------------------------------------------------------------

def test_oracle_constant_pressure_balances_at_interior_nodes(oracle):
    m = tb.generate_box_mesh(5, 4, 3)
    r = oracle.pressure_gradient(m.coords, m.connectivity, np.full(m.n_nodes, 2.5))
    assert np.abs(r[_interior((5, 4, 3))]).max() <= 1e-15
    assert np.abs(r.sum(axis=0)).max() <= 1e-14  # sum_a dN_a/dx = 0 per element


def test_oracle_linear_pressure_gives_minus_gradient_times_lumped_volume(oracle):
    """For p = g.x, integration by parts on an interior node's support gives
    r_a = -g int N_a = -g h_x h_y h_z (24 Kuhn tets of h^3/6, each N_a-integral vol/4)."""
    cells, ext = (6, 5, 4), (1.2, 1.0, 0.8)
    m = tb.generate_box_mesh(*cells, extents=ext)
    g = np.array([0.3, -1.7, 2.2])
    r = oracle.pressure_gradient(m.coords, m.connectivity, m.coords @ g)
    h3 = np.prod(np.asarray(ext) / np.asarray(cells))
    np.testing.assert_allclose(r[_interior(cells)], np.tile(-g * h3, (len(_interior(cells)), 1)),
                               rtol=1e-12, atol=1e-15)


# ---------------------------------------------------------------------------
# GPU: every scatter mode against the oracle
# ---------------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("scatter", ["private", "private-atomic", "atomic", "colored"])
@pytest.mark.parametrize("dims", [(3, 2, 2), (12, 10, 9)])
def test_pressure_term_matches_oracle(oracle, dims, scatter):
    m = tb.generate_box_mesh(*dims)
    u = tb.make_velocity(m, "random:1")
    p = np.random.default_rng(5).uniform(-2.0, 2.0, m.n_nodes)
    cfg = tb.RunConfig(scatter=scatter)
    full = tb.assemble_rsp(m, u, P, cfg, pressure=p).rhs
    ref = oracle.assemble_rsp(m.coords, m.connectivity, u) + \
        oracle.pressure_gradient(m.coords, m.connectivity, p)
    chk = oracle.compare(full, ref, m.coords, m.connectivity, u)
    assert chk.passed, chk
    # the term alone (u = 0): pressure part to 1e-12 of its max-norm
    only = tb.assemble_rsp(m, np.zeros_like(u), P, cfg, pressure=p).rhs
    pref = oracle.pressure_gradient(m.coords, m.connectivity, p)
    assert np.abs(only - pref).max() <= 1e-12 * np.abs(pref).max()
    # switched off again after the call (cached assembler)
    plain = tb.assemble_rsp(m, u, P, cfg).rhs
    assert oracle.compare(plain, oracle.assemble_rsp(m.coords, m.connectivity, u),
                          m.coords, m.connectivity, u).passed


@pytest.mark.gpu
def test_pressure_closed_form_and_reproducibility(oracle):
    cells = (16, 16, 16)
    m = tb.generate_box_mesh(*cells)
    g = np.array([1.0, -2.0, 0.5])
    res = [tb.assemble_rsp(m, np.zeros((m.n_nodes, 3)), P, tb.RunConfig(), pressure=m.coords @ g).rhs
           for _ in range(2)]
    np.testing.assert_array_equal(res[0], res[1])  # 'private' stays bitwise reproducible
    inner = _interior(cells)
    np.testing.assert_allclose(res[0][inner], np.tile(-g / 16 ** 3, (len(inner), 1)), rtol=1e-11)


@pytest.mark.gpu
def test_pressure_device_resident_and_permuted(oracle, golden_small):
    import torch
    pm = tb.Mesh(coords=golden_small["perm6_coords"], connectivity=golden_small["perm6_conn"])
    u = golden_small["perm6_u"]
    p = np.sin(3.0 * pm.coords[:, 0]) * pm.coords[:, 2]
    asm = tb.Assembler(pm, tb.RunConfig(scatter="private-atomic"))
    dp = torch.as_tensor(p, device="cuda:0")
    asm.set_pressure_device(dp.data_ptr(), stream=0)
    asm.set_velocity_host(u, stream=0)
    asm.run(P, stream=0)
    rhs = asm.get_rhs_host(stream=0)
    asm.synchronize(stream=0)
    ref = oracle.assemble_rsp(pm.coords, pm.connectivity, u) + \
        oracle.pressure_gradient(pm.coords, pm.connectivity, p)
    assert oracle.compare(rhs, ref, pm.coords, pm.connectivity, u).passed
    with pytest.raises(ValueError):  # implemented for the RSP shape only
        asm.run(P, stream=0, variant=tb.VariantId.RS)
    with pytest.raises(ValueError):
        asm.set_pressure(np.zeros(3))
    asm.set_pressure(None)
    asm.run(P, stream=0)
    rhs = asm.get_rhs_host(stream=0)
    asm.synchronize(stream=0)
    assert oracle.compare(rhs, oracle.assemble_rsp(pm.coords, pm.connectivity, u), pm.coords,
                          pm.connectivity, u).passed
    asm.close()
