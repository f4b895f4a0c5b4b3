"""Physical parameters, quadrature and velocity initialisers.

A near-verbatim restatement (deliberately, not a redesign) of the
reference's ``kernel.py`` data API (tet-assembly-lab 0.1.0): ``PhysParams``
(kernel.py:27-49), ``QuadratureRule``/``quadrature_tet4`` (kernel.py:52-86),
``validate_velocity`` (kernel.py:194-200) and the ``make_velocity``
initialisers (kernel.py:203-278), with the same field names, defaults,
formulas and error strings.  The drop-in contract needs exactly that: the
synthetic velocity fields must be bitwise the reference's (the golden
vectors are generated from them) and callers catch the same ValueErrors.
These are host-side input preparation, not part of the device hot path.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

DENOM_EPSILON = 1e-30  # kernel.py:24 (applied inside the device kernel)


@dataclass(frozen=True)
class PhysParams:
    rho: float = 1.0
    mu: float = 1e-3
    c_vreman: float = 0.07
    filter_width_rule: str = "cbrt_volume"

    def __post_init__(self):
        if not self.rho > 0.0:
            raise ValueError(f"rho must be positive, got {self.rho}")
        if self.mu < 0.0:
            raise ValueError(f"mu must be non-negative, got {self.mu}")
        if self.c_vreman < 0.0:
            raise ValueError(f"c_vreman must be non-negative, got {self.c_vreman}")
        if self.filter_width_rule != "cbrt_volume":
            raise ValueError(f"unknown filter_width_rule {self.filter_width_rule!r}")


@dataclass(frozen=True)
class QuadratureRule:
    points: np.ndarray
    weights: np.ndarray

    @property
    def n_points(self) -> int:
        return self.weights.shape[0]


def quadrature_tet4() -> QuadratureRule:
    """Degree-2 symmetric rule: a=(5+3 sqrt5)/20, b=(5-sqrt5)/20, w=1/4."""
    a = (5.0 + 3.0 * math.sqrt(5.0)) / 20.0
    b = (5.0 - math.sqrt(5.0)) / 20.0
    points = np.full((4, 4), b)
    np.fill_diagonal(points, a)
    weights = np.full(4, 0.25)
    points.setflags(write=False)
    weights.setflags(write=False)
    return QuadratureRule(points=points, weights=weights)


def interpolation_table(rule: Optional[QuadratureRule] = None) -> np.ndarray:
    """pmat = P^T P, the folded Gauss interpolation table (variants.py:559)."""
    rule = rule or quadrature_tet4()
    return np.ascontiguousarray(rule.points.T @ rule.points)


def validate_velocity(mesh, u: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.float64)
    n = mesh.coords.shape[0]
    if u.shape != (n, 3):
        raise ValueError(f"velocity must have shape ({n}, 3), got {u.shape}")
    if not np.isfinite(u).all():
        raise ValueError("velocity contains non-finite entries")
    return u


def velocity_zero(mesh) -> np.ndarray:
    return np.zeros((mesh.coords.shape[0], 3))


def velocity_constant(mesh, vx: float, vy: float, vz: float) -> np.ndarray:
    return np.tile(np.array([vx, vy, vz], dtype=np.float64), (mesh.coords.shape[0], 1))


def velocity_shear(mesh, gamma: float = 1.0) -> np.ndarray:
    u = np.zeros((mesh.coords.shape[0], 3))
    u[:, 0] = gamma * mesh.coords[:, 1]
    return u


def velocity_taylor_green(mesh) -> np.ndarray:
    c = mesh.coords
    lo = c.min(axis=0)
    hi = c.max(axis=0)
    span = np.where(hi > lo, hi - lo, 1.0)
    s = np.pi * (c - lo) / span
    u = np.zeros((c.shape[0], 3))
    u[:, 0] = np.sin(s[:, 0]) * np.cos(s[:, 1]) * np.cos(s[:, 2])
    u[:, 1] = -np.cos(s[:, 0]) * np.sin(s[:, 1]) * np.cos(s[:, 2])
    return u


def velocity_random(mesh, seed: int = 0) -> np.ndarray:
    return np.random.default_rng(int(seed)).uniform(-1.0, 1.0, size=(mesh.coords.shape[0], 3))


INITIALIZERS: dict[str, Callable] = {
    "zero": velocity_zero,
    "constant": velocity_constant,
    "shear": velocity_shear,
    "taylor-green": velocity_taylor_green,
    "random": velocity_random,
}


def make_velocity(mesh, spec: str, seed: Optional[int] = None) -> np.ndarray:
    """'name[:arg,...]' -> nodal velocity (same grammar as kernel.py:245-278)."""
    name, _, argstr = spec.partition(":")
    name = name.strip()
    if name not in INITIALIZERS:
        raise ValueError(f"unknown initializer {name!r} (known: {', '.join(sorted(INITIALIZERS))})")
    args = [s for s in argstr.replace(",", " ").split()] if argstr else []
    if name == "zero":
        if args:
            raise ValueError("zero takes no arguments")
        return velocity_zero(mesh)
    if name == "constant":
        if len(args) != 3:
            raise ValueError("constant requires vx,vy,vz")
        return velocity_constant(mesh, *(float(a) for a in args))
    if name == "shear":
        if len(args) > 1:
            raise ValueError("shear takes a single gamma")
        return velocity_shear(mesh, float(args[0]) if args else 1.0)
    if name == "taylor-green":
        if args:
            raise ValueError("taylor-green takes no arguments")
        return velocity_taylor_green(mesh)
    if len(args) > 1:
        raise ValueError("random takes a single seed")
    if args:
        return velocity_random(mesh, int(args[0]))
    return velocity_random(mesh, seed if seed is not None else 0)
