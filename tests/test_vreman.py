"""Vreman eddy viscosity known answers through the assembled operator
(reference: kernel.py:99-143 ``vreman_viscosity``; its tests
pkg/tests/test_kernel.py:130-185).

The device never exposes nu_t, so it is read back from one element: with
corners ``delta * (reference tet)`` (|det| = delta^3, hence the reference's
filter width cbrt(6 vol) = delta) and the linear field u = G^T x (constant
gradient G), the element RHS is

    r(rho, mu, c) = rho * C  -  (mu + rho * nu_t(c)) * V

(C convective, V the viscous stiffness action), so three assemblies give
nu_t = <r(1,0,c) - r(1,0,0), r(1,1,0) - r(1,0,0)> / |r(1,1,0) - r(1,0,0)|^2.
The goldens (tests/golden/vreman.npz) are the reference's own
``vreman_viscosity`` on 64 tensors (oracle/gen_golden.py): G = 0, the
identity (nu_t = c exactly), a rank-1 shear (exactly 0), 61 random ones.
The CPU test pins the read-back on the C restatement of the reference
kernel; the GPU tests run it through the production kernels.  The quiescent
guard aa <= 1e-30 (kernel.py:24) is probed from both sides.
"""
from pathlib import Path

import numpy as np
import pytest

import paper_2403_08777_b200 as tb

GOLD = np.load(Path(__file__).resolve().parent / "golden" / "vreman.npz")
REF_TET = np.array([[0.0, 0, 0], [1.0, 0, 0], [0.0, 1, 0], [0.0, 0, 1]])
CONN = np.array([[0, 1, 2, 3]], dtype=np.int64)
NU_RTOL = 1e-10  # the read-back differences cost a few digits (see test_readback_on_oracle)


def element(G, delta, shift=0.0):
    X = delta * REF_TET + shift
    return X, X @ G


def read_nu(assemble, G, delta, c):
    """nu_t of one element from three assemblies ``assemble(X, U, rho, mu, c)``."""
    X, U = element(G, delta)
    r0 = assemble(X, U, 1.0, 0.0, 0.0)
    r1 = assemble(X, U, 1.0, 0.0, c)
    rm = assemble(X, U, 1.0, 1.0, 0.0)
    v = (rm - r0).ravel()
    d = (r1 - r0).ravel()
    vv = float(v @ v)
    return (float(d @ v) / vv if vv > 0.0 else 0.0), r0, r1


def _oracle_assemble(oracle):
    def f(X, U, rho, mu, c):
        return oracle.assemble_rsp(X, CONN, U, rho, mu, c)
    return f


def _gpu_assemble(scatter):
    def f(X, U, rho, mu, c):
        m = tb.Mesh(coords=X, connectivity=CONN)
        return tb.assemble_rsp(m, U, tb.PhysParams(rho=rho, mu=mu, c_vreman=c),
                               tb.RunConfig(scatter=scatter)).rhs
    return f


def _check_goldens(assemble):
    c = float(GOLD["c"])
    for i in range(GOLD["G"].shape[0]):
        G, delta, want = GOLD["G"][i], float(GOLD["delta"][i]), float(GOLD["nut"][i])
        nu, r0, r1 = read_nu(assemble, G, delta, c)
        if want == 0.0:  # zero / rank-1 gradient: c must be inert, bit for bit
            np.testing.assert_array_equal(r1, r0, err_msg=f"tensor {i}")
        else:
            assert abs(nu - want) <= NU_RTOL * want, (i, nu, want)
    # identity, delta = 1: nu_t = c (kernel.py docstring; test_kernel.py:130-140)
    assert float(GOLD["nut"][1]) == c


def test_readback_on_oracle(oracle):
    """The read-back itself, on the bitwise restatement of the reference kernel."""
    _check_goldens(_oracle_assemble(oracle))


def _guard_cases():
    # G = eps * I: aa = 3 eps^2 straddles DENOM_EPSILON = 1e-30 (kernel.py:24)
    eps0 = np.sqrt(tb.DENOM_EPSILON / 3.0)
    return [(eps0 * (1.0 + 1e-6), True), (eps0 * (1.0 - 1e-6), False),
            (eps0 * 4.0, True), (eps0 / 4.0, False)]


@pytest.mark.parametrize("eps,active", _guard_cases())
def test_quiescent_guard_on_oracle(oracle, eps, active):
    nu, r0, r1 = read_nu(_oracle_assemble(oracle), eps * np.eye(3), 1.0, 0.07)
    if active:  # nu_t(eps I, delta = 1) = c eps
        assert nu == pytest.approx(0.07 * eps, rel=1e-9)
    else:
        np.testing.assert_array_equal(r1, r0)


@pytest.mark.gpu
@pytest.mark.parametrize("scatter", ["private-atomic", "private", "atomic", "colored"])
def test_vreman_goldens_on_gpu(scatter):
    _check_goldens(_gpu_assemble(scatter))


@pytest.mark.gpu
@pytest.mark.parametrize("scatter", ["private-atomic", "atomic"])
@pytest.mark.parametrize("eps,active", _guard_cases())
def test_quiescent_guard_on_gpu(scatter, eps, active):
    """Elements on either side of aa = 1e-30: the device applies the guard in
    unscaled (cofactor) units, aah / D^2 <= 1e-30, the same decision."""
    nu, r0, r1 = read_nu(_gpu_assemble(scatter), eps * np.eye(3), 1.0, 0.07)
    if active:
        assert nu == pytest.approx(0.07 * eps, rel=1e-9)
    else:
        np.testing.assert_array_equal(r1, r0)


@pytest.mark.gpu
def test_vreman_scaled_and_shifted_elements(oracle):
    """Tiny and large elements away from the origin: the filter width is
    cbrt(|det|) whatever the scale (MUFU-seeded rcbrt in the kernel)."""
    rng = np.random.default_rng(5)
    for delta in (1e-4, 3e-3, 0.5, 40.0):
        G = rng.uniform(-2.0, 2.0, (3, 3))
        X, U = element(G, delta, shift=7.0)
        for c in (0.07, 0.3):
            p = tb.PhysParams(c_vreman=c)
            got = tb.assemble_rsp(tb.Mesh(coords=X, connectivity=CONN), U, p,
                                  tb.RunConfig(scatter="private-atomic")).rhs
            ref = oracle.assemble_rsp(X, CONN, U, p.rho, p.mu, c)
            assert oracle.compare(got, ref, X, CONN, U, p.rho, p.mu, c).passed
