"""The drop-in assembly operator: ``assemble_rsp`` on a B200.

Reference interface mirrored (tet-assembly-lab 0.1.0, variants.py):

* ``RunConfig`` (variants.py:74-101) -- same fields and validation; the
  GPU adds scatter modes and device-layout knobs (superset).
* ``CounterLedger`` / ``VariantInfo`` / ``AssemblyResult`` (variants.py:104-135).
* ``assemble_rsp(mesh, u, params, cfg) -> AssemblyResult`` (variants.py:553-616),
  registered in ``ASSEMBLERS`` and dispatched by ``assemble`` (:619-627).
* ``assemble_baseline`` / ``assemble_rs`` (variants.py:522-550): the paper's
  B and RS code shapes as sm_100a kernels (csrc/tal_shapes.cuh), for the
  code-shape study on B200.
* ``verify_variants`` / ``oracle_compare`` / ``contribution_scale``
  (variants.py:634-755): the reference comparison arithmetic.
* ``assemble_elements(coords, conn, u, rho, mu, cvre, pmat, ids, rhs)`` --
  the numba seam (_rsp_kernels.py:20-21), accumulating into ``rhs``.

Everything numerical runs in ``libtal_b200.so`` on the GPU; there is no CPU
fallback (a missing library raises ImportError, a missing GPU RuntimeError).
"""

from __future__ import annotations

import ctypes
import enum
import math
from collections import OrderedDict
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _native as N
from .fields import PhysParams, interpolation_table, validate_velocity


class VariantId(enum.Enum):
    B = "b"
    RS = "rs"
    RSP = "rsp"


# relative tolerance of the oracle comparison and the floor of its
# denominator for cancellation-null fields (variants.py:62-65)
REL_TOL = 1e-12
NULL_SCALE_FRACTION = 0.01


SCATTER_MODES = tuple(N.SCATTER)


@dataclass(frozen=True)
class RunConfig:
    """Execution shape.

    Reference fields (variants.py:74-101): ``vector_dim``, ``n_threads``,
    ``reps``, ``scatter``, ``cache_capacity_bytes`` -- validated identically
    (vector_dim / n_threads / cache_capacity_bytes have no effect on the GPU
    path).  ``scatter`` is a superset:

    * ``private``        CTA-private shared-memory sums, ordered merge (bitwise
                         reproducible; the reference default),
    * ``colored``        colour-by-colour plain read-modify-write (bitwise
                         reproducible; uses ``mesh.colors`` or a greedy colouring),
    * ``atomic``         12 FP64 REDs per element,
    * ``private-atomic`` CTA-private sums, one FP64 RED per shared node,
    * ``sequential``     reference order: the numba kernel's operations without
                         FMA contraction, summed node by node in ascending
                         element id -- bitwise identical to the reference's
                         one-thread ``assemble_rsp`` (parity/debug path,
                         tal_strict.cuh; 4x the arithmetic).

    GPU knobs: ``device``, ``renumber`` (rcm | sfc | none), ``element_order``
    (sfc | node | keep), ``patches`` (star: edge-star patches, the rings of
    tets around an edge; tet: one tet per thread), ``cta_patches`` (patches =
    threads per CTA chunk: <= 64 | 128 | 256 select 64 | 128 | 256-thread CTAs)
    and ``chunk_nodes`` (max distinct nodes per chunk: <= 144 | 256 | 512).
    """

    vector_dim: int = 16
    n_threads: int = 1
    reps: int = 5
    scatter: str = "private"
    cache_capacity_bytes: int = 1 << 20
    device: int = 0
    renumber: str = "rcm"
    element_order: str = "sfc"
    patches: str = "star"
    cta_patches: int = 128
    chunk_nodes: int = 256

    def __post_init__(self):
        if self.vector_dim < 1:
            raise ValueError(f"vector_dim must be >= 1, got {self.vector_dim}")
        if self.n_threads < 1:
            raise ValueError(f"n_threads must be >= 1, got {self.n_threads}")
        if self.reps < 1:
            raise ValueError(f"reps must be >= 1, got {self.reps}")
        if self.scatter not in SCATTER_MODES:
            raise ValueError(f"scatter must be one of {SCATTER_MODES}, got {self.scatter!r}")
        if self.cache_capacity_bytes < 0:
            raise ValueError("cache_capacity_bytes must be >= 0")
        if self.device < 0:
            raise ValueError("device must be >= 0")
        if self.renumber not in N.RENUMBER:
            raise ValueError(f"renumber must be one of {tuple(N.RENUMBER)}, got {self.renumber!r}")
        if self.element_order not in N.EORDER:
            raise ValueError(f"element_order must be one of {tuple(N.EORDER)}")
        if self.patches not in N.PATCHES:
            raise ValueError(f"patches must be one of {tuple(N.PATCHES)}, got {self.patches!r}")
        if not 1 <= self.cta_patches <= 256:
            raise ValueError("cta_patches must be in [1, 256]")
        # CTA shapes (tal_kernels.cuh PrivCfg): <= 64 | 128 | 256 patches run
        # 64 | 128 | 256 threads with room for 144 | 256 | 512 nodes
        nmax = 144 if self.cta_patches <= 64 else 256 if self.cta_patches <= 128 else 512
        if not 16 <= self.chunk_nodes <= nmax:
            raise ValueError(f"chunk_nodes must be in [16, {nmax}] for cta_patches={self.cta_patches}")


_REF_FIELDS = ("vector_dim", "n_threads", "reps", "scatter", "cache_capacity_bytes")


def as_run_config(cfg) -> RunConfig:
    """Accept this package's ``RunConfig``, ``None`` or any object with the
    reference's five fields (``tet_assembly_lab.variants.RunConfig``, which
    the reference's ``verify_variants``, ``run_bench`` and CLI pass to
    whatever sits in ``ASSEMBLERS``).  GPU-only knobs a foreign config lacks
    take their defaults; its values are validated like ours."""
    if cfg is None:
        return RunConfig()
    if isinstance(cfg, RunConfig):
        return cfg
    missing = [f for f in _REF_FIELDS if not hasattr(cfg, f)]
    if missing:
        raise TypeError(f"not a RunConfig: {type(cfg).__name__} lacks {missing}")
    gpu = {f: getattr(cfg, f) for f in ("device", "renumber", "element_order", "patches",
                                        "cta_patches", "chunk_nodes") if hasattr(cfg, f)}
    return RunConfig(**{f: getattr(cfg, f) for f in _REF_FIELDS}, **gpu)


@dataclass(frozen=True)
class CounterLedger:
    """Static per-element counts (1 FMA = 2 Flop); bytes_dram_est is modeled."""

    flops_per_elem: int
    loadstore_per_elem: int
    intermediate_doubles_per_elem: int
    intermediate_arrays: int
    bytes_dram_est: float


@dataclass(frozen=True)
class VariantInfo:
    variant: VariantId
    name: str
    summary: str
    flops_per_elem: int
    loadstore_per_elem: int
    intermediate_doubles_per_elem: int
    intermediate_arrays: int
    flop_formula: str


# Static per-element ledgers of the three code shapes: the reference's
# statement-structure counts (variants.py:182-218), which the B200 kernels
# follow shape for shape; the executed FP64 instructions measured by ncu are
# in DESIGN.md (the RSP kernel executes fewer than its ledger).
VARIANT_INFO: dict[VariantId, VariantInfo] = {
    VariantId.B: VariantInfo(
        variant=VariantId.B,
        name="baseline (B200)",
        summary="one thread per element, generic runtime trip counts, per-Gauss-point "
        "geometry, dense 12x12 elemental matrix in local memory, separate scatter",
        flops_per_elem=3108,
        loadstore_per_elem=4908,
        intermediate_doubles_per_elem=316,
        intermediate_arrays=30,
        flop_formula="4 gauss x 363 (geometry, fields, eddy viscosity) "
        "+ 64 pairs x 21 (elemental matrix) + 300 (matvec) + 12 (scatter)",
    ),
    VariantId.RS: VariantInfo(
        variant=VariantId.RS,
        name="restructured+specialized (B200)",
        summary="one thread per element, tet4 trip counts and constants fixed, one "
        "gradient/viscosity per element, direct RHS entries, registers only",
        flops_per_elem=544,
        loadstore_per_elem=691,
        intermediate_doubles_per_elem=113,
        intermediate_arrays=27,
        flop_formula="62 (geometry) + 63 (velocity gradient) + 67 (eddy viscosity) "
        "+ 4 (factors) + 144 (point velocities and convection) + 192 (rhs entries) "
        "+ 12 (scatter)",
    ),
    VariantId.RSP: VariantInfo(
        variant=VariantId.RSP,
        name="privatized (B200)",
        summary="one sm_100a element kernel, all intermediates in registers, "
        "CTA-private shared-memory scatter",
        flops_per_elem=448,
        loadstore_per_elem=48,
        intermediate_doubles_per_elem=79,
        intermediate_arrays=0,
        flop_formula="62 (geometry) + 63 (velocity gradient) + 64 (eddy viscosity) "
        "+ 7 (factors) + 4 nodes x 63 (moments, rhs entries, scatter)",
    ),
}


def make_ledger(variant: VariantId, cfg: RunConfig) -> CounterLedger:
    """The reference's modeled ledger (variants.py:221-243): 384 B/elem of
    gathers + scatter RMW for every shape, plus a write+read-back of the
    baseline's chunk intermediates once a chunk exceeds the modeled cache."""
    info = VARIANT_INFO[variant]
    spill = 0.0
    if variant is VariantId.B and \
            info.intermediate_doubles_per_elem * 8 * cfg.vector_dim > cfg.cache_capacity_bytes:
        spill = info.intermediate_doubles_per_elem * 8 * 2
    return CounterLedger(
        flops_per_elem=info.flops_per_elem,
        loadstore_per_elem=info.loadstore_per_elem,
        intermediate_doubles_per_elem=info.intermediate_doubles_per_elem,
        intermediate_arrays=info.intermediate_arrays,
        bytes_dram_est=float(4 * 3 * 8 * 2 + 4 * 3 * 8 * 2) + spill,
    )


@dataclass(frozen=True)
class Timings:
    h2d_ms: float
    pack_ms: float
    kernel_ms: float
    unpack_ms: float
    d2h_ms: float
    total_ms: float
    kernel_launches: int


@dataclass(frozen=True)
class AssemblyResult:
    rhs: np.ndarray
    ledger: CounterLedger
    wall_time: float
    elements_per_second: float
    variant: VariantId
    timings: Optional[Timings] = None


def _variant_key(variant) -> str:
    """A VariantId, or "p": the study-only privatised-baseline shape (B with
    literal trip counts, csrc/tal_shapes.cuh), not one of the reference's."""
    if isinstance(variant, str) and variant == "p":
        return "p"
    return VariantId(variant).value


def _params(params: PhysParams, pmat: Optional[np.ndarray] = None) -> N.TalParams:
    p = N.TalParams()
    p.rho = float(params.rho)
    p.mu = float(params.mu)
    p.c_vreman = float(params.c_vreman)
    pm = interpolation_table() if pmat is None else np.asarray(pmat, dtype=np.float64)
    if pm.shape != (4, 4):
        raise ValueError("pmat must be 4x4")
    for i, v in enumerate(pm.ravel()):
        p.pmat[i] = float(v)
    return p


_CUDA_STREAM_LEGACY = 1  # cudaStreamLegacy: the legacy default stream


def _stream(stream):
    """None -> the handle's own stream; 0 -> the legacy default stream (torch's
    default stream); an int or a torch.cuda.Stream -> that stream."""
    if stream is None:
        return None
    s = getattr(stream, "cuda_stream", stream)
    return ctypes.c_void_p(int(s) if int(s) != 0 else _CUDA_STREAM_LEGACY)


class _CudaView:
    """Minimal __cuda_array_interface__ wrapper so torch can view device buffers."""

    def __init__(self, ptr: int, shape, typestr: str = "<f8", strides=None):
        self.__cuda_array_interface__ = {
            "shape": tuple(shape), "typestr": typestr, "data": (int(ptr), False),
            "version": 3, "strides": strides,
        }


class Assembler:
    """One mesh resident on one GPU (a ``tal_handle``).

    Upload once, assemble many times.  ``assemble(u, params)`` is the host
    round trip; ``run(params, stream)`` the device-resident step on the
    internal (renumbered, SoA) buffers exposed by ``device_buffers()``.
    """

    def __init__(self, mesh, cfg: Optional[RunConfig] = None, build_colors: Optional[bool] = None,
                 external_nodes: Optional[np.ndarray] = None):
        cfg = cfg or RunConfig()
        self.cfg = cfg
        L = N.lib()
        h = ctypes.c_void_p()
        N.check(L.tal_create(cfg.device, ctypes.byref(h)))
        self._h = h
        self.n_nodes = int(mesh.coords.shape[0])
        self.n_elems = int(mesh.connectivity.shape[0])
        coords = np.ascontiguousarray(mesh.coords, dtype=np.float64)
        conn = np.ascontiguousarray(mesh.connectivity, dtype=np.int64)
        colors = getattr(mesh, "colors", None)
        colors = None if colors is None else np.ascontiguousarray(colors, dtype=np.int64)
        opts = N.TalMeshOpts()
        opts.renumber = N.RENUMBER[cfg.renumber]
        opts.element_order = N.EORDER[cfg.element_order]
        opts.cta_patches = cfg.cta_patches
        opts.chunk_nodes = cfg.chunk_nodes
        opts.patch_mode = N.PATCHES[cfg.patches]
        opts.validate = 1
        if build_colors is None:
            build_colors = cfg.scatter == "colored"
        opts.build_colors = 1 if build_colors else 0
        try:
            ext = None if external_nodes is None else np.ascontiguousarray(external_nodes, np.int64)
            N.check(L.tal_upload_mesh_ex(h, N.ptr(coords), N.ptr(conn), self.n_nodes, self.n_elems,
                                         N.ptr(colors), ctypes.byref(opts), N.ptr(ext),
                                         0 if ext is None else ext.shape[0]))
        except Exception:
            L.tal_destroy(h)
            self._h = None
            raise

    # -- info ---------------------------------------------------------------
    def info(self) -> dict:
        inf = N.TalMeshInfo()
        N.check(N.lib().tal_mesh_info_get(self._h, ctypes.byref(inf)))
        return {k: getattr(inf, k) for k, _ in N.TalMeshInfo._fields_}

    # -- host round trip -----------------------------------------------------
    def assemble_into(self, u: np.ndarray, params: PhysParams, rhs: np.ndarray,
                      scatter: Optional[str] = None, pmat=None,
                      variant: VariantId = VariantId.RSP) -> Timings:
        scatter = scatter or self.cfg.scatter
        if scatter not in N.SCATTER:
            raise ValueError(f"unknown scatter mode {scatter!r}")
        vkey = _variant_key(variant)
        if u.shape != (self.n_nodes, 3) or rhs.shape != (self.n_nodes, 3):
            raise ValueError("u and rhs must have shape (n_nodes, 3)")
        if not (u.flags.c_contiguous and rhs.flags.c_contiguous and u.dtype == np.float64
                and rhs.dtype == np.float64):
            raise ValueError("u and rhs must be C-contiguous float64")
        t = N.TalTimings()
        N.check(N.lib().tal_assemble_variant(self._h, N.ptr(u), ctypes.byref(_params(params, pmat)),
                                             N.ptr(rhs), N.VARIANT[vkey],
                                             N.SCATTER[scatter], ctypes.byref(t)))
        return Timings(t.h2d_ms, t.pack_ms, t.kernel_ms, t.unpack_ms, t.d2h_ms, t.total_ms,
                       int(t.kernel_launches))

    def assemble_async(self, u: np.ndarray, params: PhysParams, rhs: np.ndarray,
                       scatter: Optional[str] = None) -> int:
        """Pipelined host round trip (tal_assemble_async): enqueue and return a
        ticket; ``u`` and ``rhs`` (C-contiguous float64 (n_nodes,3), ideally
        pinned) must stay untouched until ``wait(ticket)``.  Three calls stay in flight:
        H2D of the next field and D2H of the previous result run beside the
        assembly of the current one."""
        scatter = scatter or self.cfg.scatter
        if scatter not in N.SCATTER:
            raise ValueError(f"unknown scatter mode {scatter!r}")
        for a in (u, rhs):
            if a.shape != (self.n_nodes, 3) or a.dtype != np.float64 or not a.flags.c_contiguous:
                raise ValueError("u and rhs must be C-contiguous float64 (n_nodes, 3)")
        t = ctypes.c_int64(0)
        N.check(N.lib().tal_assemble_async(self._h, N.ptr(u), ctypes.byref(_params(params)),
                                           N.ptr(rhs), N.SCATTER[scatter], ctypes.byref(t)))
        return int(t.value)

    def wait(self, ticket: int) -> None:
        N.check(N.lib().tal_wait(self._h, int(ticket)))

    def assemble(self, u: np.ndarray, params: PhysParams, scatter: Optional[str] = None,
                 variant: VariantId = VariantId.RSP):
        rhs = np.empty((self.n_nodes, 3))
        t = self.assemble_into(np.ascontiguousarray(u, dtype=np.float64), params, rhs, scatter,
                               variant=variant)
        return rhs, t

    # -- device-resident path ----------------------------------------------
    def device_buffers(self) -> dict:
        """Raw device pointers (internal node order): ux,uy,uz,rx,ry,rz,perm,iperm."""
        b = N.TalBuffers()
        N.check(N.lib().tal_buffers_get(self._h, ctypes.byref(b)))
        return {k: getattr(b, k) for k, _ in N.TalBuffers._fields_}

    def torch_views(self):
        """torch tensors viewing the internal SoA buffers (no copy)."""
        import torch
        b = self.device_buffers()
        n = self.n_nodes
        dev = f"cuda:{self.cfg.device}"
        out = {k: torch.as_tensor(_CudaView(b[k], (n,), strides=(8 * b["u_stride"],)), device=dev)
               for k in ("ux", "uy", "uz")}
        out.update({k: torch.as_tensor(_CudaView(b[k], (n,)), device=dev) for k in ("rx", "ry", "rz")})
        return out

    def set_pressure(self, p: Optional[np.ndarray], stream=None) -> None:
        """Nodal pressure (n_nodes,) for the optional pressure-gradient term
        (tal_set_pressure_host, not part of the
        reference operator); None switches the term off.  Applies to every
        later RSP-shape assembly on this handle."""
        if p is None:
            N.check(N.lib().tal_set_pressure_host(self._h, None, _stream(stream)))
            return
        p = np.ascontiguousarray(p, dtype=np.float64)
        if p.shape != (self.n_nodes,):
            raise ValueError(f"pressure must have shape ({self.n_nodes},), got {p.shape}")
        if not np.isfinite(p).all():
            raise ValueError("pressure contains non-finite entries")
        N.check(N.lib().tal_set_pressure_host(self._h, N.ptr(p), _stream(stream)))

    def set_stabilization(self, enable: bool = True, c1: float = 4.0, c2: float = 2.0) -> None:
        """SUPG stabilisation of the convective residual for every later
        RSP-shape assembly on this handle (tal_set_stabilization; an
        extension with no reference counterpart):
        r_a[i] -= int tau (rho u.grad N_a)(rho u.grad u_i),
        tau = 1 / (c1 (mu + rho nu_t) / h^2 + c2 rho |u_mean| / h)."""
        N.check(N.lib().tal_set_stabilization(self._h, 1 if enable else 0, float(c1), float(c2)))

    def set_pressure_device(self, d_p_ptr: Optional[int], stream=None) -> None:
        N.check(N.lib().tal_set_pressure_device(
            self._h, None if d_p_ptr is None else ctypes.c_void_p(d_p_ptr), _stream(stream)))

    def set_velocity_host(self, u: np.ndarray, stream=None) -> None:
        u = np.ascontiguousarray(u, dtype=np.float64)
        if u.shape != (self.n_nodes, 3):
            raise ValueError("u must have shape (n_nodes, 3)")
        N.check(N.lib().tal_set_velocity_host(self._h, N.ptr(u), _stream(stream)))

    def set_velocity_device(self, d_u_ptr: int, stream=None) -> None:
        N.check(N.lib().tal_set_velocity_device(self._h, ctypes.c_void_p(d_u_ptr),
                                                _stream(stream)))

    def run(self, params: PhysParams, scatter: Optional[str] = None, stream=None,
            pmat=None, variant: VariantId = VariantId.RSP) -> int:
        """Enqueue one assembly on internal buffers; returns kernels launched."""
        scatter = scatter or self.cfg.scatter
        if scatter not in N.SCATTER:
            raise ValueError(f"unknown scatter mode {scatter!r}")
        nl = ctypes.c_int64(0)
        N.check(N.lib().tal_run_variant(self._h, ctypes.byref(_params(params, pmat)),
                                        N.VARIANT[_variant_key(variant)], N.SCATTER[scatter],
                                        _stream(stream), ctypes.byref(nl)))
        return int(nl.value)

    def run_caller(self, params: PhysParams, d_u_ptr: int, d_rhs_ptr: int,
                   scatter: Optional[str] = None, stream=None) -> int:
        """One assembly from and to the caller's own device arrays ((N,3)
        float64 in its node numbering; tal_run_caller): the private kernel
        gathers u from d_u and writes d_rhs directly -- no pack/unpack
        kernels.  Returns kernels launched (asynchronous on ``stream``)."""
        scatter = scatter or self.cfg.scatter
        if scatter not in N.SCATTER:
            raise ValueError(f"unknown scatter mode {scatter!r}")
        nl = ctypes.c_int64(0)
        N.check(N.lib().tal_run_caller(self._h, ctypes.byref(_params(params)), N.SCATTER[scatter],
                                       ctypes.c_void_p(d_u_ptr), ctypes.c_void_p(d_rhs_ptr),
                                       _stream(stream), ctypes.byref(nl)))
        return int(nl.value)

    def capture(self, params: PhysParams, scatter: Optional[str] = None, pmat=None,
                variant: VariantId = VariantId.RSP) -> None:
        """Capture one assembly step (zeroing + kernels + merge) as a CUDA
        graph (tal_graph_capture) for cheap replays with ``replay``."""
        scatter = scatter or self.cfg.scatter
        if scatter not in N.SCATTER:
            raise ValueError(f"unknown scatter mode {scatter!r}")
        N.check(N.lib().tal_graph_capture(self._h, ctypes.byref(_params(params, pmat)),
                                          N.VARIANT[_variant_key(variant)], N.SCATTER[scatter]))

    def replay(self, stream=None) -> int:
        """Launch the captured step; returns the kernels it launches."""
        nl = ctypes.c_int64(0)
        N.check(N.lib().tal_graph_launch(self._h, _stream(stream), ctypes.byref(nl)))
        return int(nl.value)

    def get_rhs_host(self, out: Optional[np.ndarray] = None, stream=None) -> np.ndarray:
        out = np.empty((self.n_nodes, 3)) if out is None else out
        N.check(N.lib().tal_get_rhs_host(self._h, N.ptr(out), _stream(stream)))
        return out

    def get_rhs_device(self, d_out_ptr: int, stream=None) -> None:
        N.check(N.lib().tal_get_rhs_device(self._h, ctypes.c_void_p(d_out_ptr),
                                           _stream(stream)))

    def synchronize(self, stream=None) -> None:
        N.check(N.lib().tal_synchronize(self._h, _stream(stream)))

    def map_nodes(self, caller_ids: np.ndarray) -> np.ndarray:
        ids = np.ascontiguousarray(caller_ids, dtype=np.int64)
        out = np.empty(ids.shape[0], dtype=np.int32)
        N.check(N.lib().tal_map_nodes(self._h, N.ptr(ids), ids.shape[0], N.ptr(out)))
        return out

    def halo_pack(self, d_list: int, n: int, d_out: int, stream=None) -> None:
        N.check(N.lib().tal_halo_pack(self._h, ctypes.c_void_p(d_list), n, ctypes.c_void_p(d_out),
                                      _stream(stream)))

    def halo_accumulate(self, d_list: int, n: int, d_in: int, stream=None) -> None:
        N.check(N.lib().tal_halo_accumulate(self._h, ctypes.c_void_p(d_list), n,
                                            ctypes.c_void_p(d_in), _stream(stream)))

    # -- fused interface sum with neighbouring ranks (include/tal_b200.h) ---
    def peer_local(self) -> tuple[int, int, int]:
        """(rhs x pointer, flag-word pointer, n_nodes) for an in-process neighbour."""
        rx, fl, n = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
        N.check(N.lib().tal_peer_local(self._h, ctypes.byref(rx), ctypes.byref(fl), ctypes.byref(n)))
        return rx.value, fl.value, n.value

    def peer_export(self) -> tuple[bytes, int, bytes]:
        """CUDA IPC handles of the RHS and flag words, for a neighbour process."""
        rh = ctypes.create_string_buffer(64)
        fh = ctypes.create_string_buffer(64)
        off = ctypes.c_int64()
        N.check(N.lib().tal_peer_export(self._h, rh, ctypes.byref(off), fh))
        return rh.raw, off.value, fh.raw

    def peer_attach(self, slot: int, rx_ptr: int, peer_n: int, flags_ptr: int,
                    my_ids: np.ndarray, peer_ids: np.ndarray) -> None:
        my = np.ascontiguousarray(my_ids, dtype=np.int64)
        pe = np.ascontiguousarray(peer_ids, dtype=np.int32)
        N.check(N.lib().tal_peer_attach(self._h, slot, ctypes.c_void_p(rx_ptr), peer_n,
                                        ctypes.c_void_p(flags_ptr), N.ptr(my), N.ptr(pe), my.shape[0]))

    def peer_open(self, slot: int, rhs_handle: bytes, rhs_offset: int, flags_handle: bytes,
                  peer_n: int, my_ids: np.ndarray, peer_ids: np.ndarray) -> None:
        my = np.ascontiguousarray(my_ids, dtype=np.int64)
        pe = np.ascontiguousarray(peer_ids, dtype=np.int32)
        N.check(N.lib().tal_peer_open(self._h, slot, ctypes.c_char_p(rhs_handle), rhs_offset,
                                      ctypes.c_char_p(flags_handle), peer_n, N.ptr(my), N.ptr(pe),
                                      my.shape[0]))

    def peer_detach(self) -> None:
        N.check(N.lib().tal_peer_detach(self._h))

    def profile(self, enable: bool = True) -> None:
        """Record CUDA events around the dominant kernel of every run()."""
        N.check(N.lib().tal_profile(self._h, 1 if enable else 0))

    def profile_read(self, cap: int = 4096) -> np.ndarray:
        """Dominant-kernel durations (ms) of the runs since the last read."""
        out = np.empty(cap)
        n = ctypes.c_int64(0)
        N.check(N.lib().tal_profile_read(self._h, N.ptr(out), cap, ctypes.byref(n)))
        return out[: n.value].copy()

    def close(self) -> None:
        if getattr(self, "_h", None):
            N.lib().tal_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


# small LRU of resident meshes so repeated assemble_rsp calls on one mesh do
# not re-upload (the reference likewise does its per-mesh work before t0)
_CACHE: "OrderedDict[tuple, tuple]" = OrderedDict()
_CACHE_SIZE = 4


def _needs_colors(variant: VariantId, scatter: str) -> bool:
    """Colour-by-colour launches: scatter='colored', and the B / RS shapes
    under the reproducible default scatter='private' (tal_b200.h)."""
    return scatter == "colored" or (variant is not VariantId.RSP and scatter == "private")


def _frozen(a) -> bool:
    return isinstance(a, np.ndarray) and not a.flags.writeable


def _cached_assembler(mesh, cfg: RunConfig, variant: VariantId = VariantId.RSP) -> Assembler:
    """The resident mesh for (arrays, layout knobs).  Keys are the arrays'
    identities; a read-only array (the reference ``Mesh`` clears the write
    flags, mesh.py:71-75) cannot change under the key, a writeable one is
    compared with a snapshot taken at upload (memcmp speed) on every hit so a
    mutated duck-typed mesh is re-uploaded instead of served stale."""
    colors = getattr(mesh, "colors", None)
    need_colors = _needs_colors(variant, cfg.scatter)
    key = (id(mesh.coords), id(mesh.connectivity), id(colors), mesh.coords.shape,
           mesh.connectivity.shape, cfg.device, cfg.renumber, cfg.element_order,
           cfg.patches, cfg.cta_patches, cfg.chunk_nodes, need_colors)
    arrays = (mesh.coords, mesh.connectivity, colors)
    hit = _CACHE.get(key)
    if hit is not None:
        asm, held, snaps = hit
        if all(s is None or np.array_equal(a, s) for a, s in zip(held, snaps)):
            _CACHE.move_to_end(key)
            return asm
        del _CACHE[key]
        asm.close()
    asm = Assembler(mesh, cfg, build_colors=need_colors)
    # hold the arrays so their ids cannot be recycled while cached
    snaps = tuple(None if a is None or _frozen(a) else np.array(a, copy=True) for a in arrays)
    _CACHE[key] = (asm, arrays, snaps)
    while len(_CACHE) > _CACHE_SIZE:
        _, (old, *_) = _CACHE.popitem(last=False)
        old.close()
    return asm


def clear_cache() -> None:
    while _CACHE:
        _, (asm, *_) = _CACHE.popitem()
        asm.close()
    while _SEAMS:
        _, (seam, *_) = _SEAMS.popitem()
        seam.close()
    while _PINNED_U:
        _, a = _PINNED_U.popitem()
        N.lib().tal_host_unregister(N.ptr(a))


def _stab_args(stabilization):
    if stabilization is None or stabilization is False:
        return None
    if stabilization is True:
        return (4.0, 2.0)
    c1, c2 = stabilization
    return float(c1), float(c2)


def _assemble_variant(variant: VariantId, mesh, u, params: PhysParams,
                      cfg: Optional[RunConfig], pressure: Optional[np.ndarray] = None,
                      stabilization=None) -> AssemblyResult:
    cfg = as_run_config(cfg)
    u = validate_velocity(mesh, u)
    asm = _cached_assembler(mesh, cfg, variant)
    rhs = np.empty((asm.n_nodes, 3))
    st = _stab_args(stabilization)
    try:
        if pressure is not None:
            asm.set_pressure(pressure)
        if st is not None:
            asm.set_stabilization(True, *st)
        t = asm.assemble_into(u, params, rhs, cfg.scatter, variant=variant)
    finally:
        if pressure is not None:
            asm.set_pressure(None)
        if st is not None:
            asm.set_stabilization(False)
    wall = t.total_ms * 1e-3
    rate = asm.n_elems / wall if wall > 0.0 else 0.0
    return AssemblyResult(rhs=rhs, ledger=make_ledger(variant, cfg), wall_time=wall,
                          elements_per_second=rate, variant=variant, timings=t)


def assemble_rsp(mesh, u: np.ndarray, params: PhysParams,
                 cfg: Optional[RunConfig] = None, pressure: Optional[np.ndarray] = None,
                 stabilization=None) -> AssemblyResult:
    """Drop-in for ``tet_assembly_lab.assemble_rsp`` (variants.py:553-616).

    ``wall_time`` is the CUDA-event time of the call's device timeline
    (velocity H2D + layout pack + assembly kernels + unpack + RHS D2H); the
    one-time mesh upload is excluded like the reference's colouring.
    ``pressure`` (n_nodes,) adds the P1 pressure-gradient term
    ``int p dN_a/dx_i`` -- an extension with no reference counterpart
    (parity pinned only by this repo's oracle).
    ``stabilization`` (True for c1=4, c2=2, or a (c1, c2) pair) adds the SUPG
    term of the convective residual (Assembler.set_stabilization) -- also an
    extension with no reference counterpart.
    """
    return _assemble_variant(VariantId.RSP, mesh, u, params, cfg, pressure, stabilization)


def assemble_baseline(mesh, u: np.ndarray, params: PhysParams,
                      cfg: Optional[RunConfig] = None) -> AssemblyResult:
    """The baseline code shape (variants.py:522-538) as a B200 kernel:
    scatter 'private'/'colored' run colour by colour (bitwise reproducible),
    'atomic'/'private-atomic' with FP64 REDs.  ``vector_dim`` only enters the
    modeled ledger, as in the reference."""
    return _assemble_variant(VariantId.B, mesh, u, params, cfg)


def assemble_rs(mesh, u: np.ndarray, params: PhysParams,
                cfg: Optional[RunConfig] = None) -> AssemblyResult:
    """The restructured+specialised code shape (variants.py:541-550) as a
    B200 kernel; scatter handling as ``assemble_baseline``."""
    return _assemble_variant(VariantId.RS, mesh, u, params, cfg)


ASSEMBLERS: dict[VariantId, Callable] = {
    VariantId.B: assemble_baseline,
    VariantId.RS: assemble_rs,
    VariantId.RSP: assemble_rsp,
}


def assemble(variant: VariantId, mesh, u, params, cfg=None) -> AssemblyResult:
    return ASSEMBLERS[variant](mesh, u, params, cfg)


class _Seam:
    """A tal_seam context (resident mesh + pinned staging) for one (coords, conn)."""

    def __init__(self, coords, conn, device):
        h = ctypes.c_void_p()
        N.check(N.lib().tal_seam_open(device, N.ptr(coords), N.ptr(conn), coords.shape[0],
                                      conn.shape[0], ctypes.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            N.lib().tal_seam_close(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


_SEAMS: "OrderedDict[tuple, tuple]" = OrderedDict()
# velocity arrays page-locked for the seam (cudaHostRegister), held alive here
# so the registration can never outlive the memory; the reference's drivers
# pass the same u to every seam call of an assembly
_PINNED_U: "OrderedDict[int, np.ndarray]" = OrderedDict()


def _pin_velocity(u: np.ndarray) -> None:
    if u.nbytes < (1 << 22) or not u.flags.c_contiguous:
        return
    key = u.ctypes.data
    if key in _PINNED_U and _PINNED_U[key] is u:
        _PINNED_U.move_to_end(key)
        return
    try:
        N.check(N.lib().tal_host_register(N.ptr(u), u.nbytes))
    except RuntimeError:  # e.g. overlapping an existing registration: keep the staged copy
        return
    old = _PINNED_U.pop(key, None)
    if old is not None:
        N.lib().tal_host_unregister(N.ptr(old))
    _PINNED_U[key] = u
    while len(_PINNED_U) > 2:
        _, a = _PINNED_U.popitem(last=False)
        N.lib().tal_host_unregister(N.ptr(a))


def _seam_for(coords, conn, device) -> "_Seam":
    """Seam context cache with the resident-mesh cache's rules (_cached_assembler)."""
    key = (id(coords), id(conn), coords.shape, conn.shape, device)
    hit = _SEAMS.get(key)
    if hit is not None:
        seam, held, snaps = hit
        if all(s is None or np.array_equal(a, s) for a, s in zip(held, snaps)):
            _SEAMS.move_to_end(key)
            return seam
        del _SEAMS[key]
        seam.close()
    seam = _Seam(coords, conn, device)
    snaps = tuple(None if _frozen(a) else np.array(a, copy=True) for a in (coords, conn))
    _SEAMS[key] = (seam, (coords, conn), snaps)
    while len(_SEAMS) > 2:
        _, (old, *_) = _SEAMS.popitem(last=False)
        old.close()
    return seam


def assemble_elements(coords, conn, u, rho, mu, cvre, pmat, ids, rhs, device: int = 0,
                      strict: bool = False) -> None:
    """The numba seam ``_rsp_kernels.assemble_elements`` on the GPU: assemble
    elements ``ids`` and ADD into ``rhs`` (in place, like the numba loop).

    Fast path (``tal_seam_*``): the mesh stays resident per (coords, conn)
    between calls -- the reference's drivers call the seam once per assembly
    (one thread, ``ids`` = all elements: the edge-star kernel) or once per
    thread slab (a contiguous ``ids`` range: the per-element kernel).
    ``strict=True`` (``tal_assemble_elements_strict``) is bitwise the numba
    loop: each node continues from its incoming ``rhs`` through its elements in
    ``ids`` order with the reference's operation order (tal_strict.cuh)."""
    if not strict and isinstance(coords, np.ndarray) and isinstance(conn, np.ndarray) \
            and coords.dtype == np.float64 and conn.dtype == np.int64 \
            and coords.flags.c_contiguous and conn.flags.c_contiguous \
            and coords.ndim == 2 and coords.shape[1:] == (3,) and conn.ndim == 2 and conn.shape[1:] == (4,):
        u = np.ascontiguousarray(u, dtype=np.float64)
        pm = np.ascontiguousarray(pmat, dtype=np.float64)
        ids = np.ascontiguousarray(ids, dtype=np.int64)
        if not (isinstance(rhs, np.ndarray) and rhs.flags.c_contiguous and rhs.dtype == np.float64):
            raise ValueError("rhs must be a C-contiguous float64 array (accumulated in place)")
        if u.shape != coords.shape or rhs.shape != coords.shape or pm.shape != (4, 4):
            raise ValueError("bad array shapes")
        if coords.shape[0] == 0 or ids.shape[0] == 0:
            return
        seam = _seam_for(coords, conn, device)
        _pin_velocity(u)
        N.check(N.lib().tal_seam_assemble(seam.h, N.ptr(u), float(rho), float(mu), float(cvre),
                                          N.ptr(pm), N.ptr(ids), ids.shape[0], N.ptr(rhs)))
        return
    coords = np.ascontiguousarray(coords, dtype=np.float64)
    conn = np.ascontiguousarray(conn, dtype=np.int64)
    u = np.ascontiguousarray(u, dtype=np.float64)
    pm = np.ascontiguousarray(pmat, dtype=np.float64)
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    if not (isinstance(rhs, np.ndarray) and rhs.flags.c_contiguous and rhs.dtype == np.float64):
        raise ValueError("rhs must be a C-contiguous float64 array (accumulated in place)")
    if coords.shape[1:] != (3,) or conn.shape[1:] != (4,) or u.shape != coords.shape \
            or rhs.shape != coords.shape or pm.shape != (4, 4):
        raise ValueError("bad array shapes")
    fn = N.lib().tal_assemble_elements_strict if strict else N.lib().tal_assemble_elements
    N.check(fn(device, N.ptr(coords), N.ptr(conn), coords.shape[0],
                                          conn.shape[0], N.ptr(u), float(rho), float(mu),
                                          float(cvre), N.ptr(pm), N.ptr(ids), ids.shape[0],
                                          N.ptr(rhs)))


# ---------------------------------------------------------------------------
# verification arithmetic (variants.py:634-755)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class VariantCheck:
    variant: VariantId
    max_abs_diff: float
    rel_diff: float
    denominator: float
    worst_node: int
    passed: bool
    note: str = ""


@dataclass(frozen=True)
class VerifyReport:
    tolerance: float
    denominator: float
    checks: tuple
    passed: bool


def contribution_scale(mesh, u: np.ndarray, params: PhysParams) -> float:
    """Bound on one element's raw RHS contribution (variants.py:653-676): the
    denominator floor for fields whose assembled RHS is pure cancellation."""
    conn = np.asarray(mesh.connectivity)
    if conn.shape[0] == 0 or np.asarray(u).size == 0:
        return 0.0
    x = np.asarray(mesh.coords)[conn]
    e = x[:, 1:] - x[:, :1]                                   # (E, 3 edges, 3)
    cof = np.stack([np.cross(e[:, 1], e[:, 2]), np.cross(e[:, 2], e[:, 0]),
                    np.cross(e[:, 0], e[:, 1])], axis=1)
    det = np.einsum("ek,ek->e", e[:, 0], cof[:, 0])
    vol = np.abs(det) / 6.0
    grad_bound = 4.0 * np.abs(cof).max(axis=(1, 2)) / np.abs(det)
    u_max = np.abs(np.asarray(u)[conn]).max(axis=(1, 2))
    nut_cap = 24.0 * params.c_vreman * np.cbrt(6.0 * vol) ** 2 * grad_bound * u_max
    scale = vol * u_max * grad_bound * (params.rho * u_max + params.mu + params.rho * nut_cap)
    return float(scale.max())


def _denominator(mesh, u, params, oracle: np.ndarray) -> float:
    top = float(np.abs(oracle).max()) if oracle.size else 0.0
    return max(top, NULL_SCALE_FRACTION * contribution_scale(mesh, u, params))


def _compare(variant: VariantId, rhs: np.ndarray, oracle: np.ndarray, denom: float) -> VariantCheck:
    bad = ~np.isfinite(rhs)
    if bad.any():
        node = int(np.argwhere(bad)[0][0])
        return VariantCheck(variant, math.inf, math.inf, denom, node, False,
                            f"non-finite output at node {node}")
    diff = np.abs(rhs - oracle)
    max_abs = float(diff.max()) if diff.size else 0.0
    worst = int(np.argmax(diff) // 3) if diff.size else 0
    rel = max_abs / denom if denom > 0.0 else (0.0 if max_abs == 0.0 else math.inf)
    return VariantCheck(variant, max_abs, rel, denom, worst, rel <= REL_TOL)


def reference_order_rhs(mesh, u: np.ndarray, params: PhysParams, device: int = 0) -> np.ndarray:
    """The default oracle vector of ``oracle_compare`` / ``verify_variants``:
    ``scatter='sequential'`` (csrc/tal_strict.cuh), an independent kernel
    that restates ``_rsp_kernels.py:33-164`` operation by operation and sums
    in the reference's order -- bitwise identical to the reference's
    one-thread ``assemble_rsp`` (tests/test_sequential.py), i.e. the role the
    reference gives its scalar ``assemble_reference`` (variants.py:739-741).
    The CPU oracle of this repo (``oracle/``) is test infrastructure and is
    never called from the package; pass its vector as ``oracle=`` instead."""
    return assemble_rsp(mesh, u, params, RunConfig(scatter="sequential", device=device)).rhs


def oracle_compare(mesh, u: np.ndarray, params: PhysParams, rhs: np.ndarray,
                   variant: VariantId, oracle: Optional[np.ndarray] = None,
                   device: int = 0) -> VariantCheck:
    """Compare one assembled vector with an oracle vector (variants.py:714-720);
    without ``oracle`` the reference-order vector (:func:`reference_order_rhs`)."""
    u = validate_velocity(mesh, u)
    note = ""
    if oracle is None:
        oracle, note = reference_order_rhs(mesh, u, params, device), "oracle: sequential (reference order)"
    c = _compare(VariantId(variant), rhs, oracle, _denominator(mesh, u, params, oracle))
    if note and not c.note:
        c = VariantCheck(c.variant, c.max_abs_diff, c.rel_diff, c.denominator, c.worst_node,
                         c.passed, note)
    return c


def verify_variants(mesh, u: np.ndarray, params: PhysParams, cfg: Optional[RunConfig] = None,
                    fault_inject: Optional[str] = None,
                    oracle: Optional[np.ndarray] = None) -> VerifyReport:
    """Run every code shape and compare each with the oracle vector at
    ``REL_TOL`` (variants.py:723-755); ``fault_inject`` (a variant value)
    perturbs that shape's output to prove the check can fail.  ``oracle`` as
    in :func:`oracle_compare`."""
    cfg = as_run_config(cfg)
    u = validate_velocity(mesh, u)
    if oracle is None:
        oracle = reference_order_rhs(mesh, u, params, cfg.device)
    denom = _denominator(mesh, u, params, oracle)
    checks = []
    for variant, fn in ASSEMBLERS.items():
        rhs = fn(mesh, u, params, cfg).rhs
        if fault_inject is not None and variant.value == fault_inject:
            rhs = rhs.copy()
            rhs[0, 0] += 1e-6 * (denom if denom > 0.0 else 1.0)
        checks.append(_compare(variant, rhs, oracle, denom))
    return VerifyReport(REL_TOL, denom, tuple(checks), all(c.passed for c in checks))
