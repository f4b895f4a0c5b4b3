"""Tetrahedral mesh value type and native generators.

Mirrors the reference's mesh layer (``mesh.py`` of tet-assembly-lab 0.1.0):
``Mesh`` (mesh.py:36-89) with the same fields, validation and immutability,
``generate_box_mesh`` (mesh.py:145-184), ``signed_volumes`` (mesh.py:110-123),
``color_elements`` (mesh.py:235-257).  The per-element loops run in the
native library (C++), not in Python.  ``assemble_rsp`` accepts this Mesh or
the reference's own ``tet_assembly_lab.Mesh`` (anything with ``coords``,
``connectivity`` and optional ``colors``).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, replace
from typing import Optional

import numpy as np

from ._native import check, lib, ptr

VOLUME_EPSILON = 1e-300  # mesh.py:20


@dataclass(frozen=True)
class Mesh:
    """coords (n_nodes,3) f64; connectivity (n_elems,4) int64, positively
    oriented; optional colors (n_elems,) int64 with no two node-sharing
    elements in one colour."""

    coords: np.ndarray
    connectivity: np.ndarray
    colors: Optional[np.ndarray] = None

    def __post_init__(self):
        coords = np.ascontiguousarray(self.coords, dtype=np.float64)
        conn = np.ascontiguousarray(self.connectivity, dtype=np.int64)
        if coords.ndim != 2 or coords.shape[1] != 3:
            raise ValueError(f"coords must have shape (n_nodes, 3), got {coords.shape}")
        if conn.ndim != 2 or conn.shape[1] != 4:
            raise ValueError(f"connectivity must have shape (n_elems, 4), got {conn.shape}")
        if conn.size and (conn.min() < 0 or conn.max() >= coords.shape[0]):
            raise ValueError("connectivity index out of range [0, n_nodes)")
        vols = signed_volumes(coords, conn)
        if vols.size and vols.min() <= 0.0:
            bad = int(np.argmin(vols))
            raise ValueError(f"element {bad} has non-positive signed volume {vols[bad]:g}")
        colors = self.colors
        if colors is not None:
            colors = np.ascontiguousarray(colors, dtype=np.int64)
            if colors.shape != (conn.shape[0],):
                raise ValueError("colors must be one index per element")
            if not check_coloring(conn, colors, coords.shape[0]):
                raise ValueError("coloring invalid: elements sharing a node share a color")
            colors.setflags(write=False)
        for name, arr in (("coords", coords), ("connectivity", conn), ("colors", colors)):
            if arr is not None:
                arr.setflags(write=False)
            object.__setattr__(self, name, arr)

    @property
    def n_nodes(self) -> int:
        return self.coords.shape[0]

    @property
    def n_elems(self) -> int:
        return self.connectivity.shape[0]

    @property
    def n_colors(self) -> Optional[int]:
        if self.colors is None:
            return None
        return int(self.colors.max()) + 1 if self.colors.size else 0

    __hash__ = object.__hash__
    __eq__ = object.__eq__


def signed_volumes(coords: np.ndarray, connectivity: np.ndarray) -> np.ndarray:
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    conn = np.ascontiguousarray(connectivity, dtype=np.int64)
    out = np.empty(conn.shape[0])
    if conn.shape[0]:
        check(lib().tal_signed_volumes(ptr(coords), ptr(conn), conn.shape[0], ptr(out)))
    return out


def check_coloring(conn: np.ndarray, colors: np.ndarray, n_nodes: int) -> bool:
    v = ctypes.c_int(0)
    check(lib().tal_check_coloring(ptr(conn), ptr(colors), n_nodes, conn.shape[0], ctypes.byref(v)))
    return bool(v.value)


def _box_arrays(nx: int, ny: int, nz: int, extents=(1.0, 1.0, 1.0)):
    for name, v in (("nx", nx), ("ny", ny), ("nz", nz)):
        if int(v) != v or v < 1:
            raise ValueError(f"{name} must be a positive integer, got {v!r}")
    nx, ny, nz = int(nx), int(ny), int(nz)
    ext = np.asarray(extents, dtype=np.float64)
    if ext.shape != (3,) or not np.all(ext > 0.0):
        raise ValueError(f"extents must be 3 positive lengths, got {extents!r}")
    coords = np.empty(((nx + 1) * (ny + 1) * (nz + 1), 3))
    conn = np.empty((6 * nx * ny * nz, 4), dtype=np.int64)
    check(lib().tal_box_mesh(nx, ny, nz, float(ext[0]), float(ext[1]), float(ext[2]),
                             ptr(coords), ptr(conn)))
    return coords, conn


def generate_box_mesh(nx: int, ny: int, nz: int, extents=(1.0, 1.0, 1.0)) -> Mesh:
    """Structured box of nx*ny*nz hex cells, each split into 6 tetrahedra
    (Kuhn split), nodes x-fastest, cell c -> elements 6c..6c+5."""
    coords, conn = _box_arrays(nx, ny, nz, extents)
    return Mesh(coords=coords, connectivity=conn)


def generate_delaunay_mesh(n_points: int, seed: int = 0) -> Mesh:
    """Unstructured tetrahedral mesh of the unit cube: the Delaunay
    tetrahedralisation (scipy.spatial) of ``n_points`` uniform random points
    (``default_rng(seed)``), every element oriented positively (last two nodes
    swapped where the volume is negative), zero-volume slivers dropped.  A
    synthetic stand-in for the general meshes the reference's Mesh accepts:
    irregular valences, open and closed edge rings of every size, ~6.7 tets
    per node.  Host-side input preparation (scipy needed)."""
    from scipy.spatial import Delaunay
    if n_points < 4:
        raise ValueError(f"n_points must be >= 4, got {n_points}")
    pts = np.random.default_rng(seed).random((int(n_points), 3))
    conn = np.ascontiguousarray(Delaunay(pts).simplices, dtype=np.int64)
    x = pts[conn]
    det = np.einsum("ij,ij->i", x[:, 1] - x[:, 0], np.cross(x[:, 2] - x[:, 0], x[:, 3] - x[:, 0]))
    neg = det < 0.0
    conn[neg, 2], conn[neg, 3] = conn[neg, 3].copy(), conn[neg, 2].copy()
    conn = np.ascontiguousarray(conn[det != 0.0])
    return Mesh(coords=pts, connectivity=conn)


def color_elements(mesh) -> Mesh:
    """Greedy lowest-free colouring in element order (mesh.py:235-257)."""
    conn = np.ascontiguousarray(mesh.connectivity, dtype=np.int64)
    colors = np.empty(conn.shape[0], dtype=np.int64)
    nc = ctypes.c_int64(0)
    check(lib().tal_color_elements(ptr(conn), mesh.coords.shape[0], conn.shape[0], ptr(colors),
                                   ctypes.byref(nc)))
    if isinstance(mesh, Mesh):
        return replace(mesh, colors=colors)
    return Mesh(coords=mesh.coords, connectivity=conn, colors=colors)


def renumber_nodes(mesh, method: str = "rcm") -> np.ndarray:
    """Node permutation perm[new] = old (rcm | sfc | none)."""
    from ._native import RENUMBER
    if method not in RENUMBER:
        raise ValueError(f"unknown renumber method {method!r}")
    coords = np.ascontiguousarray(mesh.coords, dtype=np.float64)
    conn = np.ascontiguousarray(mesh.connectivity, dtype=np.int64)
    perm = np.empty(coords.shape[0], dtype=np.int64)
    check(lib().tal_renumber_nodes(ptr(coords), ptr(conn), coords.shape[0], conn.shape[0],
                                   RENUMBER[method], ptr(perm)))
    return perm


def permute_nodes(mesh, perm: np.ndarray) -> Mesh:
    """Mesh with node i' = perm[i'] of the input."""
    perm = np.asarray(perm, dtype=np.int64)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(perm.size)
    return Mesh(coords=np.asarray(mesh.coords)[perm], connectivity=inv[np.asarray(mesh.connectivity)])


def edge_star_patches(mesh, mode: str = "star"):
    """The private scatter's work decomposition (tal_prep.hpp): a list of
    (a, b, ring, closed) with tets (a, b, ring[i], ring[i+1])."""
    from ._native import PATCHES
    conn = np.ascontiguousarray(mesh.connectivity, dtype=np.int64)
    n_nodes = mesh.coords.shape[0]
    npch = ctypes.c_int64(0)
    nn = ctypes.c_int64(0)
    L = lib()
    check(L.tal_build_patches(ptr(conn), n_nodes, conn.shape[0], PATCHES[mode], ctypes.byref(npch),
                              ctypes.byref(nn), None, None, None))
    off = np.empty(npch.value + 1, dtype=np.int32)
    nodes = np.empty(nn.value, dtype=np.int32)
    closed = np.empty(npch.value, dtype=np.uint8)
    check(L.tal_build_patches(ptr(conn), n_nodes, conn.shape[0], PATCHES[mode], ctypes.byref(npch),
                              ctypes.byref(nn), ptr(off), ptr(nodes), ptr(closed)))
    out = []
    for g in range(npch.value):
        seg = nodes[off[g]:off[g + 1]]
        out.append((int(seg[0]), int(seg[1]), [int(x) for x in seg[2:]], bool(closed[g])))
    return out


def plan_blobs(mesh, cfg=None) -> dict:
    """Host-only dump of the private-scatter chunk blobs (tal_plan_blobs):
    ``blobs`` (uint8), ``blob_off`` (int32, 16-B units), ``threads`` (table
    stride) and ``perm`` (internal -> caller node id, or None for identity).
    The layout is documented at k_assemble_private (csrc/tal_kernels.cuh)."""
    from . import _native as N
    from .assembly import RunConfig
    cfg = cfg or RunConfig()
    coords = np.ascontiguousarray(mesh.coords, dtype=np.float64)
    conn = np.ascontiguousarray(mesh.connectivity, dtype=np.int64)
    o = N.TalMeshOpts()
    check(lib().tal_default_mesh_opts(ctypes.byref(o)))
    o.renumber, o.element_order = N.RENUMBER[cfg.renumber], N.EORDER[cfg.element_order]
    o.cta_patches, o.chunk_nodes, o.patch_mode = cfg.cta_patches, cfg.chunk_nodes, N.PATCHES[cfg.patches]
    sizes = np.zeros(4, dtype=np.int64)
    args = (ptr(coords), ptr(conn), coords.shape[0], conn.shape[0], ctypes.byref(o), ptr(sizes))
    check(lib().tal_plan_blobs(*args, None, None, None))
    blobs = np.zeros(max(int(sizes[0]), 1), dtype=np.uint8)
    off = np.zeros(max(int(sizes[1]), 1), dtype=np.int32)
    perm = np.zeros(max(int(sizes[3]), 1), dtype=np.int32)
    check(lib().tal_plan_blobs(*args, ptr(blobs), ptr(off), ptr(perm)))
    return {"blobs": blobs[:sizes[0]], "blob_off": off[:sizes[1]], "threads": int(sizes[2]),
            "perm": perm[:sizes[3]] if sizes[3] else None}


def plan_layout(mesh, cfg=None) -> dict:
    """Host-only dry run of the device upload (tal_plan_layout): renumbering,
    element order, edge-star patches and CTA chunks for ``cfg`` (a RunConfig);
    returns the chunking statistics without touching a GPU."""
    from . import _native as N
    from .assembly import RunConfig
    cfg = cfg or RunConfig()
    coords = np.ascontiguousarray(mesh.coords, dtype=np.float64)
    conn = np.ascontiguousarray(mesh.connectivity, dtype=np.int64)
    o = N.TalMeshOpts()
    check(lib().tal_default_mesh_opts(ctypes.byref(o)))
    o.renumber, o.element_order = N.RENUMBER[cfg.renumber], N.EORDER[cfg.element_order]
    o.cta_patches, o.chunk_nodes, o.patch_mode = cfg.cta_patches, cfg.chunk_nodes, N.PATCHES[cfg.patches]
    inf = N.TalMeshInfo()
    check(lib().tal_plan_layout(ptr(coords), ptr(conn), coords.shape[0], conn.shape[0],
                                ctypes.byref(o), ctypes.byref(inf)))
    return {k: getattr(inf, k) for k, _ in N.TalMeshInfo._fields_
            if k not in ("n_colors", "device_bytes")}


# ---------------------------------------------------------------------------
# mesh IO (native, csrc/tal_meshio.cpp)
# ---------------------------------------------------------------------------

class MeshFormatError(ValueError):
    """Unparseable mesh file; ``line`` is the 1-based offending line number
    (the reference's mesh.MeshFormatError, mesh.py:22-29)."""

    def __init__(self, message: str, line: Optional[int] = None):
        # the native message already carries the "line N: " prefix
        super().__init__(message)
        self.line = line


def _path(path) -> bytes:
    import os
    return os.fsencode(os.fspath(path))


def save_mesh(mesh, path) -> None:
    """The reference's text format (mesh.py:280-290), byte for byte:
    ``nodes <n>``, n ``x y z`` lines (%.17g), ``elems <m>``, m lines of 4
    zero-based node ids.  Formatted in parallel native blocks."""
    coords = np.ascontiguousarray(mesh.coords, dtype=np.float64)
    conn = np.ascontiguousarray(mesh.connectivity, dtype=np.int64)
    check(lib().tal_mesh_save_text(_path(path), ptr(coords), ptr(conn), coords.shape[0], conn.shape[0]))


def save_mesh_binary(mesh, path) -> None:
    """Binary TALMESH1 file (64-byte header with sizes and a content hash,
    coords f64 (N,3), connectivity i64 (E,4)): exact round trip for meshes
    too large for the text format."""
    coords = np.ascontiguousarray(mesh.coords, dtype=np.float64)
    conn = np.ascontiguousarray(mesh.connectivity, dtype=np.int64)
    check(lib().tal_mesh_save_binary(_path(path), ptr(coords), ptr(conn), coords.shape[0], conn.shape[0]))


def load_mesh(path) -> Mesh:
    """Read a mesh file: TALMESH1 binary (detected by its magic) or the
    reference's text format with its semantics (mesh.py:293-371): ``#``
    comments and blank lines skipped, MeshFormatError with the line number on
    malformed input, ValueError for out-of-range ids, inverted elements
    re-oriented (last two nodes swapped) with a warning."""
    import warnings
    from pathlib import Path
    p = _path(path)
    n, e, is_bin = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
    check(lib().tal_mesh_probe_binary(p, ctypes.byref(n), ctypes.byref(e), ctypes.byref(is_bin)))
    if is_bin.value:
        coords = np.empty((n.value, 3))
        conn = np.empty((e.value, 4), dtype=np.int64)
        check(lib().tal_mesh_load_binary(p, ptr(coords), n.value, ptr(conn), e.value))
        return Mesh(coords=coords, connectivity=conn)
    h = ctypes.c_void_p()
    rc = lib().tal_mesh_load_text(p, ctypes.byref(h))
    if rc != 0:
        line = int(lib().tal_last_error_line())
        if line > 0:
            raise MeshFormatError((lib().tal_last_error() or b"").decode(errors="replace"), line)
        check(rc)
    try:
        nr = ctypes.c_int64()
        check(lib().tal_meshbuf_info(h, ctypes.byref(n), ctypes.byref(e), ctypes.byref(nr)))
        coords = np.empty((n.value, 3))
        conn = np.empty((e.value, 4), dtype=np.int64)
        check(lib().tal_meshbuf_copy(h, ptr(coords), ptr(conn)))
    finally:
        lib().tal_meshbuf_free(h)
    if nr.value:
        warnings.warn(f"{Path(path).name}: re-oriented {nr.value} inverted element(s)", stacklevel=2)
    return Mesh(coords=coords, connectivity=conn)
