"""ctypes binding of ``libtal_b200.so`` (include/tal_b200.h).

The library is built in-tree by ``paper_2403_08777_b200.build``.  There is no
fallback: if the shared object is missing, :func:`lib` raises ImportError;
if no B200 is present, every compute entry point fails with RuntimeError.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(os.environ.get("TAL_LIB_PATH") or Path(__file__).resolve().parent / "libtal_b200.so")

TAL_OK, TAL_EINVAL, TAL_ECUDA, TAL_ENOMEM, TAL_ESTATE, TAL_EINTERNAL, TAL_EIO = 0, 1, 2, 3, 4, 5, 6

SCATTER = {"private": 0, "colored": 1, "atomic": 2, "private-atomic": 3, "sequential": 4}
VARIANT = {"b": 0, "rs": 1, "rsp": 2, "p": 3}  # TAL_VARIANT_* ("p": study-only shape)
RENUMBER = {"none": 0, "rcm": 1, "sfc": 2}
EORDER = {"keep": 0, "node": 1, "sfc": 2}
PATCHES = {"tet": 0, "star": 1}


class TalParams(ctypes.Structure):
    _fields_ = [("rho", ctypes.c_double), ("mu", ctypes.c_double),
                ("c_vreman", ctypes.c_double), ("pmat", ctypes.c_double * 16)]


class TalMeshOpts(ctypes.Structure):
    _fields_ = [("renumber", ctypes.c_int), ("element_order", ctypes.c_int),
                ("cta_patches", ctypes.c_int), ("chunk_nodes", ctypes.c_int),
                ("validate", ctypes.c_int), ("build_colors", ctypes.c_int),
                ("patch_mode", ctypes.c_int)]


class TalMeshInfo(ctypes.Structure):
    _fields_ = [("n_nodes", ctypes.c_int64), ("n_elems", ctypes.c_int64),
                ("n_colors", ctypes.c_int64), ("n_patches", ctypes.c_int64),
                ("n_chunks", ctypes.c_int64),
                ("n_chunk_nodes", ctypes.c_int64), ("n_shared_nodes", ctypes.c_int64),
                ("device_bytes", ctypes.c_int64), ("prep_seconds", ctypes.c_double)]


class TalTimings(ctypes.Structure):
    _fields_ = [("h2d_ms", ctypes.c_double), ("pack_ms", ctypes.c_double),
                ("kernel_ms", ctypes.c_double), ("unpack_ms", ctypes.c_double),
                ("d2h_ms", ctypes.c_double), ("total_ms", ctypes.c_double),
                ("kernel_launches", ctypes.c_int64)]


class TalBuffers(ctypes.Structure):
    _fields_ = [("ux", ctypes.c_void_p), ("uy", ctypes.c_void_p), ("uz", ctypes.c_void_p),
                ("rx", ctypes.c_void_p), ("ry", ctypes.c_void_p), ("rz", ctypes.c_void_p),
                ("perm", ctypes.c_void_p), ("iperm", ctypes.c_void_p), ("u_stride", ctypes.c_int64)]


# (name, restype, argtypes) of every exported symbol in include/tal_b200.h
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_I = ctypes.c_int
SIGNATURES = [
    ("tal_last_error", ctypes.c_char_p, []),
    ("tal_abi_version", _I, []),
    ("tal_device_count", _I, [ctypes.POINTER(_I)]),
    ("tal_create", _I, [_I, ctypes.POINTER(_P)]),
    ("tal_destroy", _I, [_P]),
    ("tal_host_alloc", _I, [_I64, ctypes.POINTER(_P)]),
    ("tal_host_free", _I, [_P]),
    ("tal_host_register", _I, [_P, _I64]),
    ("tal_host_unregister", _I, [_P]),
    ("tal_upload_mesh", _I, [_P, _P, _P, _I64, _I64, _P, ctypes.POINTER(TalMeshOpts)]),
    ("tal_upload_mesh_ex", _I, [_P, _P, _P, _I64, _I64, _P, ctypes.POINTER(TalMeshOpts), _P, _I64]),
    ("tal_mesh_info_get", _I, [_P, ctypes.POINTER(TalMeshInfo)]),
    ("tal_layout_bank_stats", _I, [_P]),
    ("tal_plan_blobs", _I, [_P, _P, _I64, _I64, ctypes.POINTER(TalMeshOpts), _P, _P, _P, _P]),
    ("tal_plan_layout", _I, [_P, _P, _I64, _I64, ctypes.POINTER(TalMeshOpts),
                             ctypes.POINTER(TalMeshInfo)]),
    ("tal_peer_local", _I, [_P, ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.POINTER(_I64)]),
    ("tal_peer_export", _I, [_P, _P, ctypes.POINTER(_I64), _P]),
    ("tal_peer_attach", _I, [_P, _I, _P, _I64, _P, _P, _P, _I64]),
    ("tal_peer_open", _I, [_P, _I, _P, _I64, _P, _I64, _P, _P, _I64]),
    ("tal_peer_detach", _I, [_P]),
    ("tal_default_mesh_opts", _I, [ctypes.POINTER(TalMeshOpts)]),
    ("tal_assemble", _I, [_P, _P, ctypes.POINTER(TalParams), _P, _I, ctypes.POINTER(TalTimings)]),
    ("tal_assemble_variant", _I, [_P, _P, ctypes.POINTER(TalParams), _P, _I, _I,
                                  ctypes.POINTER(TalTimings)]),
    ("tal_run_variant", _I, [_P, ctypes.POINTER(TalParams), _I, _I, _P, ctypes.POINTER(_I64)]),
    ("tal_assemble_async", _I, [_P, _P, ctypes.POINTER(TalParams), _P, _I, ctypes.POINTER(_I64)]),
    ("tal_wait", _I, [_P, _I64]),
    ("tal_buffers_get", _I, [_P, ctypes.POINTER(TalBuffers)]),
    ("tal_set_velocity_host", _I, [_P, _P, _P]),
    ("tal_set_pressure_host", _I, [_P, _P, _P]),
    ("tal_set_stabilization", _I, [_P, _I, _D, _D]),
    ("tal_set_pressure_device", _I, [_P, _P, _P]),
    ("tal_set_velocity_device", _I, [_P, _P, _P]),
    ("tal_run", _I, [_P, ctypes.POINTER(TalParams), _I, _P, ctypes.POINTER(_I64)]),
    ("tal_run_caller", _I, [_P, ctypes.POINTER(TalParams), _I, _P, _P, _P, ctypes.POINTER(_I64)]),
    ("tal_graph_capture", _I, [_P, ctypes.POINTER(TalParams), _I, _I]),
    ("tal_graph_launch", _I, [_P, _P, ctypes.POINTER(_I64)]),
    ("tal_graph_destroy", _I, [_P]),
    ("tal_get_rhs_host", _I, [_P, _P, _P]),
    ("tal_get_rhs_device", _I, [_P, _P, _P]),
    ("tal_synchronize", _I, [_P, _P]),
    ("tal_assemble_elements", _I, [_I, _P, _P, _I64, _I64, _P, _D, _D, _D, _P, _P, _I64, _P]),
    ("tal_assemble_elements_strict", _I, [_I, _P, _P, _I64, _I64, _P, _D, _D, _D, _P, _P, _I64, _P]),
    ("tal_last_error_line", _I64, []),
    ("tal_mesh_load_text", _I, [ctypes.c_char_p, ctypes.POINTER(_P)]),
    ("tal_meshbuf_info", _I, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
    ("tal_meshbuf_copy", _I, [_P, _P, _P]),
    ("tal_meshbuf_free", _I, [_P]),
    ("tal_mesh_save_text", _I, [ctypes.c_char_p, _P, _P, _I64, _I64]),
    ("tal_mesh_save_binary", _I, [ctypes.c_char_p, _P, _P, _I64, _I64]),
    ("tal_mesh_probe_binary", _I, [ctypes.c_char_p, ctypes.POINTER(_I64), ctypes.POINTER(_I64),
                                   ctypes.POINTER(_I)]),
    ("tal_mesh_load_binary", _I, [ctypes.c_char_p, _P, _I64, _P, _I64]),
    ("tal_rcb_parts", _I, [_P, _I64, _I, _P]),
    ("tal_seam_open", _I, [_I, _P, _P, _I64, _I64, ctypes.POINTER(_P)]),
    ("tal_seam_assemble", _I, [_P, _P, _D, _D, _D, _P, _P, _I64, _P]),
    ("tal_seam_close", _I, [_P]),
    ("tal_halo_pack", _I, [_P, _P, _I64, _P, _P]),
    ("tal_halo_accumulate", _I, [_P, _P, _I64, _P, _P]),
    ("tal_map_nodes", _I, [_P, _P, _I64, _P]),
    ("tal_box_mesh", _I, [_I64, _I64, _I64, _D, _D, _D, _P, _P]),
    ("tal_signed_volumes", _I, [_P, _P, _I64, _P]),
    ("tal_color_elements", _I, [_P, _I64, _I64, _P, ctypes.POINTER(_I64)]),
    ("tal_check_coloring", _I, [_P, _P, _I64, _I64, ctypes.POINTER(_I)]),
    ("tal_renumber_nodes", _I, [_P, _P, _I64, _I64, _I, _P]),
    ("tal_fp64_peak", _I, [_I, _D, ctypes.POINTER(_D), ctypes.POINTER(_D)]),
    ("tal_build_patches", _I, [_P, _I64, _I64, _I, ctypes.POINTER(_I64), ctypes.POINTER(_I64),
                               _P, _P, _P]),
    ("tal_profile", _I, [_P, _I]),
    ("tal_profile_read", _I, [_P, _P, _I64, ctypes.POINTER(_I64)]),
]

_lib = None


def lib() -> ctypes.CDLL:
    """Load libtal_b200.so (building it first if the CUDA toolchain is here)."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists() and os.environ.get("TAL_NO_AUTOBUILD") != "1":
        try:
            from . import build as _build
            _build.build()
        except Exception as err:  # pragma: no cover - toolchain missing
            raise ImportError(f"{LIB_PATH} is missing and could not be built: {err}") from err
    if not LIB_PATH.exists():
        raise ImportError(f"{LIB_PATH} is missing; run python -m paper_2403_08777_b200.build")
    L = ctypes.CDLL(str(LIB_PATH))
    for name, res, args in SIGNATURES:
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.tal_abi_version() != 1:
        raise ImportError("libtal_b200.so ABI mismatch")
    _lib = L
    return L


def check(rc: int) -> None:
    """Map a TAL status to the reference's exception types."""
    if rc == TAL_OK:
        return
    msg = (lib().tal_last_error() or b"").decode(errors="replace")
    if rc == TAL_EINVAL:
        raise ValueError(msg)
    if rc == TAL_ENOMEM:
        raise MemoryError(msg)
    if rc == TAL_EIO:
        raise OSError(msg)
    raise RuntimeError(msg or f"libtal_b200 error {rc}")


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def device_count() -> int:
    n = ctypes.c_int(0)
    rc = lib().tal_device_count(ctypes.byref(n))
    return n.value if rc == TAL_OK else 0


def fp64_peak(device: int = 0, ms_target: float = 0.5) -> tuple[float, float]:
    """Burst FP64 FMA throughput (TFLOP/s) and the SM clock (MHz) measured in
    the best probe launch."""
    tf = ctypes.c_double(0.0)
    mhz = ctypes.c_double(0.0)
    check(lib().tal_fp64_peak(device, ms_target, ctypes.byref(tf), ctypes.byref(mhz)))
    return tf.value, mhz.value


class PinnedArray:
    """A numpy view over page-locked host memory from tal_host_alloc."""

    def __init__(self, shape, dtype=np.float64):
        self.shape = tuple(shape)
        self.dtype = np.dtype(dtype)
        nbytes = int(np.prod(self.shape)) * self.dtype.itemsize
        p = ctypes.c_void_p()
        check(lib().tal_host_alloc(nbytes, ctypes.byref(p)))
        self._p = p
        buf = (ctypes.c_char * max(nbytes, 1)).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=self.dtype, count=int(np.prod(self.shape))).reshape(self.shape)

    def free(self) -> None:
        if self._p is not None and self._p.value:
            self.array = None
            lib().tal_host_free(self._p)
            self._p = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.free()
        except Exception:
            pass
