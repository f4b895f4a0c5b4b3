"""CPU oracle for the momentum-RHS assembly -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module, and
only as the checker / the timed CPU baseline.  The product package
``paper_2403_08777_b200`` never imports it and has no CPU fallback.

Contents (each a restatement of the reference package tet-assembly-lab
0.1.0 under /root/reference/pkg/src/tet_assembly_lab):

* ctypes bindings to ``tal_oracle.c`` (the numba hot loop
  ``_rsp_kernels.py:20-164``, the threaded private driver
  ``variants.py:573-596``, the Gauss-loop scalar oracle ``kernel.py:146-191``,
  the Kuhn box generator ``mesh.py:145-184``, greedy colouring
  ``mesh.py:235-257``);
* numpy restatements of the velocity initialisers (``kernel.py:203-278``),
  the quadrature/pmat setup (``kernel.py:71-86``, ``variants.py:558-559``)
  and the verification arithmetic (``variants.py:653-711``:
  ``contribution_scale``, ``_oracle_denominator``, ``_compare_rhs``).

Parity of the restatement is pinned against ``tests/golden/*.npz``, which
``oracle/gen_golden.py`` produced by importing the reference itself.

Exception -- parity UNPINNED: ``pressure_gradient``
has no counterpart in the reference (its operator has no pressure term,
kernel.py:7-10); it is restated here from the weak form and
checked only against closed-form answers (tests/test_pressure.py).
The same holds for ``supg_term`` (the SUPG stabilisation extension): restated
from its weak form with explicit Gauss points and the reference's Vreman
formula (kernel.py:99-143), pinned by closed forms (tests/test_stabilization.py).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path
from typing import Optional

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libtal_oracle.so"

REL_TOL = 1e-12  # variants.py:64
NULL_SCALE_FRACTION = 0.01  # variants.py:65
NS_REL_L2_TOL = 1e-12  # north_star: relative L2
NS_ENTRY_TOL = 1e-10  # north_star: per-entry error relative to max-norm

_lib = None


def build() -> Path:
    """Compile tal_oracle.c with the committed Makefile (gcc)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(LIB_PATH))
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        D = ctypes.c_double
        L.orc_assemble_elements.argtypes = [P, P, P, D, D, D, P, P, I64, P]
        L.orc_assemble_elements.restype = None
        L.orc_assemble_private.argtypes = [P, P, P, D, D, D, P, I64, I64, ctypes.c_int, I64, P]
        L.orc_assemble_private.restype = ctypes.c_int
        L.orc_assemble_reference.argtypes = [P, P, P, D, D, D, I64, I64, P]
        L.orc_assemble_reference.restype = None
        L.orc_box_mesh.argtypes = [I64, I64, I64, D, D, D, P, P]
        L.orc_box_mesh.restype = None
        L.orc_signed_volumes.argtypes = [P, P, I64, P]
        L.orc_signed_volumes.restype = None
        L.orc_color_elements.argtypes = [P, I64, I64, P]
        L.orc_color_elements.restype = ctypes.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------------------
# mesh + fields
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class OracleMesh:
    coords: np.ndarray  # (N,3) f64
    connectivity: np.ndarray  # (E,4) i64
    colors: Optional[np.ndarray] = None

    @property
    def n_nodes(self) -> int:
        return self.coords.shape[0]

    @property
    def n_elems(self) -> int:
        return self.connectivity.shape[0]


def box_mesh(nx: int, ny: int, nz: int, extents=(1.0, 1.0, 1.0)) -> OracleMesh:
    """Kuhn 6-tet box (mesh.py:145-184), x-fastest nodes, elements 6c..6c+5."""
    n_nodes = (nx + 1) * (ny + 1) * (nz + 1)
    n_elems = 6 * nx * ny * nz
    coords = np.empty((n_nodes, 3))
    conn = np.empty((n_elems, 4), dtype=np.int64)
    lib().orc_box_mesh(nx, ny, nz, float(extents[0]), float(extents[1]), float(extents[2]),
                       _p(coords), _p(conn))
    return OracleMesh(coords, conn)


def signed_volumes(coords, conn) -> np.ndarray:
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    conn = np.ascontiguousarray(conn, dtype=np.int64)
    out = np.empty(conn.shape[0])
    lib().orc_signed_volumes(_p(coords), _p(conn), conn.shape[0], _p(out))
    return out


def color_elements(conn, n_nodes) -> np.ndarray:
    conn = np.ascontiguousarray(conn, dtype=np.int64)
    colors = np.empty(conn.shape[0], dtype=np.int64)
    rc = lib().orc_color_elements(_p(conn), n_nodes, conn.shape[0], _p(colors))
    if rc < 0:
        raise RuntimeError("oracle colouring needs more than 64 colours")
    return colors


def pmat() -> np.ndarray:
    """pmat = P^T P of the symmetric 4-point rule (kernel.py:71-86, variants.py:558-559)."""
    a = (5.0 + 3.0 * math.sqrt(5.0)) / 20.0
    b = (5.0 - math.sqrt(5.0)) / 20.0
    pts = np.array([[a, b, b, b], [b, a, b, b], [b, b, a, b], [b, b, b, a]])
    return pts.T @ pts


def velocity(coords: np.ndarray, spec: str) -> np.ndarray:
    """Velocity initialisers (kernel.py:203-278) for the specs the tests use."""
    n = coords.shape[0]
    name, _, arg = spec.partition(":")
    args = [s for s in arg.replace(",", " ").split()] if arg else []
    if name == "zero":
        return np.zeros((n, 3))
    if name == "constant":
        return np.tile(np.array([float(a) for a in args], dtype=np.float64), (n, 1))
    if name == "shear":
        g = float(args[0]) if args else 1.0
        u = np.zeros((n, 3))
        u[:, 0] = g * coords[:, 1]
        return u
    if name == "taylor-green":
        lo = coords.min(axis=0)
        hi = coords.max(axis=0)
        span = np.where(hi > lo, hi - lo, 1.0)
        s = np.pi * (coords - lo) / span
        u = np.zeros((n, 3))
        u[:, 0] = np.sin(s[:, 0]) * np.cos(s[:, 1]) * np.cos(s[:, 2])
        u[:, 1] = -np.cos(s[:, 0]) * np.sin(s[:, 1]) * np.cos(s[:, 2])
        return u
    if name == "random":
        seed = int(args[0]) if args else 0
        return np.random.default_rng(seed).uniform(-1.0, 1.0, size=(n, 3))
    raise ValueError(f"unknown initializer {name!r}")


# ---------------------------------------------------------------------------
# assembly
# ---------------------------------------------------------------------------

def assemble_rsp(coords, conn, u, rho=1.0, mu=1e-3, cvre=0.07, n_threads=1,
                 vector_dim=16) -> np.ndarray:
    """The reference's privatised assembly ('private' scatter), CPU restatement."""
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    conn = np.ascontiguousarray(conn, dtype=np.int64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    pm = np.ascontiguousarray(pmat())
    rhs = np.empty((coords.shape[0], 3))
    rc = lib().orc_assemble_private(_p(coords), _p(conn), _p(u), rho, mu, cvre, _p(pm),
                                    coords.shape[0], conn.shape[0], int(n_threads),
                                    int(vector_dim), _p(rhs))
    if rc != 0:
        raise RuntimeError(f"orc_assemble_private failed ({rc})")
    return rhs


def assemble_elements(coords, conn, u, rho, mu, cvre, pm, ids, rhs) -> None:
    """Mirror of the numba seam: accumulate elements ``ids`` into ``rhs``."""
    lib().orc_assemble_elements(_p(coords), _p(conn), _p(u), rho, mu, cvre, _p(pm),
                                _p(ids), ids.shape[0], _p(rhs))


def assemble_reference(coords, conn, u, rho=1.0, mu=1e-3, cvre=0.07) -> np.ndarray:
    """Scalar Gauss-loop oracle (kernel.py:173-191)."""
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    conn = np.ascontiguousarray(conn, dtype=np.int64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    rhs = np.empty((coords.shape[0], 3))
    lib().orc_assemble_reference(_p(coords), _p(conn), _p(u), rho, mu, cvre,
                                 coords.shape[0], conn.shape[0], _p(rhs))
    return rhs


def pressure_gradient(coords, conn, p) -> np.ndarray:
    """r_a[i] = sum over tets of int_T p dN_a/dx_i dV for P1 p (parity
    unpinned, see the module header): per tet vol * mean(p) * dN_a/dx_i, with
    dN_a/dx_i = c_a[i] / det from the cofactor rows (mesh.py:187-218 form)."""
    coords = np.asarray(coords, dtype=np.float64)
    conn = np.asarray(conn, dtype=np.int64)
    p = np.asarray(p, dtype=np.float64)
    rhs = np.zeros((coords.shape[0], 3))
    if conn.shape[0] == 0:
        return rhs
    x = coords[conn]
    e1, e2, e3 = x[:, 1] - x[:, 0], x[:, 2] - x[:, 0], x[:, 3] - x[:, 0]
    c = np.stack([np.cross(e2, e3), np.cross(e3, e1), np.cross(e1, e2)], axis=1)  # (E,3,3)
    det = np.einsum("ek,ek->e", e1, c[:, 0])
    grad = np.concatenate([-c.sum(axis=1, keepdims=True), c], axis=1) / det[:, None, None]
    vol = np.abs(det) / 6.0
    pbar = p[conn].mean(axis=1)
    contrib = (vol * pbar)[:, None, None] * grad  # (E, 4, 3)
    for a in range(4):
        np.add.at(rhs, conn[:, a], contrib[:, a])
    return rhs


def _vreman_np(G, delta, c):
    """kernel.py:99-143 (the minor form), vectorised over elements: G (E,3,3)
    with G[e,k,i] = du_i/dx_k."""
    a = G.reshape(-1, 9)
    aa = (a * a).sum(axis=1)
    g = G
    d = np.stack([g[:, 0, 0] * g[:, 1, 1] - g[:, 0, 1] * g[:, 1, 0],
                  g[:, 0, 0] * g[:, 2, 1] - g[:, 0, 1] * g[:, 2, 0],
                  g[:, 1, 0] * g[:, 2, 1] - g[:, 1, 1] * g[:, 2, 0],
                  g[:, 0, 0] * g[:, 1, 2] - g[:, 0, 2] * g[:, 1, 0],
                  g[:, 0, 0] * g[:, 2, 2] - g[:, 0, 2] * g[:, 2, 0],
                  g[:, 1, 0] * g[:, 2, 2] - g[:, 1, 2] * g[:, 2, 0],
                  g[:, 0, 1] * g[:, 1, 2] - g[:, 0, 2] * g[:, 1, 1],
                  g[:, 0, 1] * g[:, 2, 2] - g[:, 0, 2] * g[:, 2, 1],
                  g[:, 1, 1] * g[:, 2, 2] - g[:, 1, 2] * g[:, 2, 1]], axis=1)
    ssq = (d * d).sum(axis=1)
    bb = delta ** 4 * ssq
    nut = np.zeros_like(aa)
    ok = (aa > 1e-30) & (bb >= 0.0)
    nut[ok] = c * np.sqrt(bb[ok] / aa[ok])
    return nut


def supg_term(coords, conn, u, rho=1.0, mu=1e-3, cvre=0.07, c1=4.0, c2=2.0) -> np.ndarray:
    """SUPG stabilisation of the convective residual (parity unpinned, see the
    module header), from its weak form with the 4-point Gauss rule
    (kernel.py:71-86):
        r_a[i] -= sum_g w_g |det|/6 tau (rho u_g . grad N_a)(rho u_g . grad u_i),
        tau = 1 / (c1 (mu + rho nu_t) / h^2 + c2 rho |u_mean| / h), h = cbrt(6 vol),
    nu_t the reference's Vreman viscosity with filter width h."""
    coords = np.asarray(coords, dtype=np.float64)
    conn = np.asarray(conn, dtype=np.int64)
    u = np.asarray(u, dtype=np.float64)
    rhs = np.zeros((coords.shape[0], 3))
    if conn.shape[0] == 0:
        return rhs
    x, ue = coords[conn], u[conn]                         # (E,4,3)
    J = np.stack([x[:, 1] - x[:, 0], x[:, 2] - x[:, 0], x[:, 3] - x[:, 0]], axis=1)  # rows = edges
    det = np.linalg.det(J)
    vol = np.abs(det) / 6.0
    dref = np.array([[-1.0, -1.0, -1.0], [1.0, 0, 0], [0, 1.0, 0], [0, 0, 1.0]])  # dN/dxi
    grad = np.einsum("ekl,al->eak", np.linalg.inv(J), dref)  # (E,4,3): dN_a/dx_k
    G = np.einsum("eak,eai->eki", grad, ue)              # du_i/dx_k
    h = np.cbrt(6.0 * vol)
    nut = _vreman_np(G, h, cvre)
    vis = mu + rho * nut
    umean = np.linalg.norm(ue.mean(axis=1), axis=1)
    tau = 1.0 / (c1 * vis / h ** 2 + c2 * rho * umean / h)
    qa, qb = (5.0 + 3.0 * math.sqrt(5.0)) / 20.0, (5.0 - math.sqrt(5.0)) / 20.0
    P = np.full((4, 4), qb) + np.eye(4) * (qa - qb)         # N_b(x_g) = P[g, b]
    ug = np.einsum("gb,ebi->egi", P, ue)                   # (E,4g,3)
    adv_N = np.einsum("egk,eak->ega", ug, grad)            # u_g . grad N_a
    adv_u = np.einsum("egk,eki->egi", ug, G)               # u_g . grad u_i
    contrib = -(0.25 * vol * tau * rho * rho)[:, None, None] * np.einsum("ega,egi->eai", adv_N, adv_u)
    for a in range(4):
        np.add.at(rhs, conn[:, a], contrib[:, a])
    return rhs


# ---------------------------------------------------------------------------
# verification arithmetic (variants.py:653-711) + the north_star criteria
# ---------------------------------------------------------------------------

def contribution_scale(coords, conn, u, rho=1.0, mu=1e-3, cvre=0.07) -> float:
    """variants.py:653-676: bound on one element's raw contribution."""
    if conn.shape[0] == 0 or u.size == 0:
        return 0.0
    x = coords[conn]
    e1 = x[:, 1] - x[:, 0]
    e2 = x[:, 2] - x[:, 0]
    e3 = x[:, 3] - x[:, 0]
    cof = np.stack([np.cross(e2, e3), np.cross(e3, e1), np.cross(e1, e2)], axis=1)
    det = np.einsum("ek,ek->e", e1, cof[:, 0])
    vols = np.abs(det) / 6.0
    gmax = 4.0 * np.abs(cof).max(axis=(1, 2)) / np.abs(det)
    umax = np.abs(u[conn]).max(axis=(1, 2))
    delta2 = np.cbrt(6.0 * vols) ** 2
    nut_cap = 24.0 * cvre * delta2 * gmax * umax
    scale = vols * umax * gmax * (rho * umax + mu + rho * nut_cap)
    return float(scale.max())


@dataclass(frozen=True)
class Check:
    max_abs_diff: float
    rel_diff: float  # reference criterion: max|d| / denominator
    denominator: float
    worst_node: int
    rel_l2: Optional[float]  # None when ||oracle||_2 == 0 (undefined)
    entry_rel: float  # max|d| / ||oracle||_inf (inf if oracle is null and d != 0)
    passed_reference: bool
    passed_north_star: bool
    note: str = ""

    @property
    def passed(self) -> bool:
        return self.passed_reference and self.passed_north_star


def compare(rhs, oracle, coords, conn, u, rho=1.0, mu=1e-3, cvre=0.07) -> Check:
    """Both parity criteria.

    reference (variants.py:679-711): max|rhs-oracle| / max(||oracle||_inf,
    0.01 * contribution_scale) <= 1e-12, non-finite output fails with its node.
    north_star: rel-L2 <= 1e-12 and max|d| <= 1e-10 * ||oracle||_inf.  For a
    null field (||oracle||_inf below the reference floor 0.01 *
    contribution_scale: constant / zero velocity, whose exact RHS is 0 and
    whose computed oracle is pure cancellation noise) the max-norm is
    replaced by the same floored denominator and rel-L2 is reported None
    (undefined), exactly as the reference floors its own criterion.
    """
    rhs = np.asarray(rhs)
    oracle = np.asarray(oracle)
    max_oracle = float(np.abs(oracle).max()) if oracle.size else 0.0
    denom = max(max_oracle, NULL_SCALE_FRACTION * contribution_scale(coords, conn, u, rho, mu, cvre))
    finite = np.isfinite(rhs)
    if not finite.all():
        bad = int(np.argwhere(~finite)[0][0])
        return Check(math.inf, math.inf, denom, bad, math.inf, math.inf, False, False,
                     f"non-finite output at node {bad}")
    diff = np.abs(rhs - oracle)
    max_abs = float(diff.max()) if diff.size else 0.0
    worst = int(np.argmax(diff) // 3) if diff.size else 0
    if denom > 0.0:
        rel = max_abs / denom
    else:
        rel = 0.0 if max_abs == 0.0 else math.inf
    # null (cancellation-noise) oracle: its max-norm is below the reference's
    # noise floor, so norm-relative criteria are ill-posed; like the
    # reference, measure against the floored denominator and skip rel-L2
    null = max_oracle < denom
    on = float(np.linalg.norm(oracle)) if oracle.size else 0.0
    rel_l2 = float(np.linalg.norm(rhs - oracle)) / on if (on > 0.0 and not null) else None
    norm_inf = denom
    if norm_inf > 0.0:
        entry = max_abs / norm_inf
    else:
        entry = 0.0 if max_abs == 0.0 else math.inf
    ok_ref = rel <= REL_TOL
    ok_ns = entry <= NS_ENTRY_TOL and (rel_l2 is None or rel_l2 <= NS_REL_L2_TOL)
    return Check(max_abs, rel, denom, worst, rel_l2, entry, ok_ref, ok_ns)


def checksums(rhs) -> tuple[float, float]:
    """harness.py:124-125 convention: (sum, sum of |.|)."""
    return float(np.sum(rhs)), float(np.abs(rhs).sum())


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
