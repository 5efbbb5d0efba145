"""ctypes binding of the sm_100a C-ABI library ``lib/libfkc_sw.so``
(declared in ``include/fkc_sw.h``).

There is deliberately no CPU fallback: if the library is missing or fails to
load, every entry point raises :class:`NativeUnavailable` -- the hot path is
the CUDA kernel or nothing.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FKC_LIB") or os.path.join(PKG_DIR, "lib", "libfkc_sw.so")
CSRC = os.path.join(PKG_DIR, "csrc")

FKC_OK, FKC_EDOMAIN, FKC_EUSAGE, FKC_ECUDA = 0, 1, 2, 3
F32, F64 = 0, 1
BC_REFLECTIVE, BC_PERIODIC, BC_NONE = 0, 1, 2
MODE_EXACT, MODE_FAST = 0, 1
VARIANT_AUTO, VARIANT_GENERIC, VARIANT_TMA, VARIANT_RESIDENT, VARIANT_LOOP = 0, 1, 2, 3, 4
ERR_NONPOSITIVE_DEPTH, ERR_NONFINITE, ERR_WATCHDOG, ERR_NONPOSITIVE_FACE = 1, 2, 4, 8

EXPORTS = (
    "fkc_sw_step", "fkc_sw_advance_n", "fkc_sw_run_host", "fkc_sw_apply_boundary", "fkc_sw_reduce_state", "fkc_sw_reduce_reset",
    "fkc_region_cpy", "fkc_cshift", "fkc_copy2d", "fkc_halo_pack", "fkc_halo_unpack",
    "fkc_ipc_export", "fkc_ipc_open", "fkc_ipc_close",
    "fkc_tma_plan", "fkc_test_div_f32", "fkc_test_div_f64", "fkc_test_sqrt2_f32", "fkc_last_error",
    "fkc_abi_version",
)
ABI_VERSION = 4
SYNC_PDL = 1
MAX_RANKS = 8


class NativeUnavailable(RuntimeError):
    """The CUDA library is not built / not loadable."""


class FkcError(RuntimeError):
    """A non-zero C-ABI return code: 1 domain, 3 CUDA (2, usage, raises
    :class:`FkcUsageError`)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"[fkc rc={code}] {msg}")
        self.code = code


class FkcUsageError(FkcError, ValueError):
    """FKC_EUSAGE: the call was rejected before touching device memory (bad
    shape, pitch, alignment, pointer or enum).  ``swdemo.LaunchError``
    derives from it, so callers of the reference API that catch
    ``LaunchError`` / ``ValueError`` see these."""


class Grid(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int32), ("ny", ctypes.c_int32), ("pitch", ctypes.c_int64),
                ("dtype", ctypes.c_int32), ("_pad", ctypes.c_int32)]


class Reduce(ctypes.Structure):
    _fields_ = [("mass", ctypes.c_void_p), ("max_abs_u", ctypes.c_void_p),
                ("max_abs_v", ctypes.c_void_p), ("cfl_min", ctypes.c_void_p),
                ("err", ctypes.c_void_p)]


class PeerLine(ctypes.Structure):
    """fkc_peer_line: neighbour address of our cell (0,0) image per field + stride."""
    _fields_ = [("p", ctypes.c_void_p * 3), ("stride", ctypes.c_int64)]


class Sync(ctypes.Structure):
    """fkc_sync: per-side mailbox words, edge-writer counters, epoch, PDL flag, CFL board."""
    _fields_ = [("wait", ctypes.c_void_p * 4), ("signal", ctypes.c_void_p * 4),
                ("counter", ctypes.c_void_p), ("epoch", ctypes.c_uint32), ("flags", ctypes.c_uint32),
                ("cfl_board", ctypes.c_void_p), ("cfl_peers", ctypes.c_void_p * 8), ("cfl_counter", ctypes.c_void_p),
                ("cfl_rank", ctypes.c_int32), ("cfl_nranks", ctypes.c_int32)]


class Tune(ctypes.Structure):
    """fkc_sw_tune: per-call launch schedule (all zero = the defaults; results
    never depend on it)."""
    _fields_ = [("seg", ctypes.c_int32), ("tail_rows", ctypes.c_int32), ("tail_waves", ctypes.c_int32),
                ("order", ctypes.c_int32), ("parity", ctypes.c_int32), ("warps", ctypes.c_int32),
                ("no_pdl", ctypes.c_int32), ("no_alternate", ctypes.c_int32)]

    def __init__(self, **kw):
        super().__init__()
        for k, v in kw.items():
            setattr(self, k, int(v))

    def copy(self) -> "Tune":
        return Tune(**{k: getattr(self, k) for k, _ in self._fields_})


class StepArgs(ctypes.Structure):
    _fields_ = [("grid", Grid),
                ("H", ctypes.c_void_p), ("U", ctypes.c_void_p), ("V", ctypes.c_void_p),
                ("oH", ctypes.c_void_p), ("oU", ctypes.c_void_p), ("oV", ctypes.c_void_p),
                ("dx", ctypes.c_double), ("dy", ctypes.c_double), ("dt", ctypes.c_double),
                ("g", ctypes.c_double),
                ("dt_bound", ctypes.c_void_p), ("cfl", ctypes.c_double),
                ("bc", ctypes.c_int32 * 4), ("mode", ctypes.c_int32), ("variant", ctypes.c_int32),
                ("red", Reduce), ("peer", PeerLine * 4), ("sync", Sync), ("tune", Tune)]


class LoopArgs(ctypes.Structure):
    """fkc_sw_loop_args: the native time loop (fkc_sw_advance_n)."""
    _fields_ = [("step", StepArgs), ("first_step", ctypes.c_int64), ("steps", ctypes.c_int64),
                ("slots", ctypes.c_void_p), ("dt_from_slots", ctypes.c_int32), ("want_cfl", ctypes.c_int32),
                ("use_graph", ctypes.c_int32), ("_pad", ctypes.c_int32), ("host_slots", ctypes.c_void_p)]


_lib = None


def build(force: bool = False) -> str:
    """Compile the library in-tree with nvcc for sm_100a (see csrc/Makefile)."""
    if force and os.path.exists(LIB_PATH):
        os.remove(LIB_PATH)
    subprocess.run(["make", "-s", "-C", CSRC], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(f"{LIB_PATH} not built (run __graft_entry__.build() "
                                "or `make -C paper_1107_2157_b200/csrc`)")
    try:
        L = ctypes.CDLL(LIB_PATH)
    except OSError as e:  # pragma: no cover - depends on the box
        raise NativeUnavailable(f"cannot load {LIB_PATH}: {e}") from e
    vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
    sig = {
        "fkc_sw_step": [ctypes.POINTER(StepArgs), vp],
        "fkc_sw_advance_n": [ctypes.POINTER(LoopArgs), vp],
        "fkc_sw_run_host": [ctypes.POINTER(LoopArgs), ctypes.POINTER(vp), ctypes.POINTER(vp), i64, i32, vp],
        "fkc_sw_apply_boundary": [ctypes.POINTER(Grid), vp, vp, vp, ctypes.POINTER(i32), vp],
        "fkc_sw_reduce_state": [ctypes.POINTER(Grid), vp, vp, vp, dbl, dbl, dbl,
                                ctypes.POINTER(Reduce), vp],
        "fkc_sw_reduce_reset": [ctypes.POINTER(Reduce), vp],
        "fkc_region_cpy": [i32, vp, i32, i32, i64, ctypes.POINTER(i32), vp, i64, vp],
        "fkc_cshift": [i32, vp, i32, i32, i64, i32, i64, vp, i64, vp],
        "fkc_copy2d": [vp, i64, vp, i64, i64, i64, vp],
        "fkc_halo_pack": [ctypes.POINTER(Grid), vp, vp, vp, i32, vp, vp],
        "fkc_halo_unpack": [ctypes.POINTER(Grid), vp, vp, vp, i32, vp, vp],
        "fkc_ipc_export": [vp, ctypes.POINTER(ctypes.c_uint8), ctypes.POINTER(i64)],
        "fkc_ipc_open": [ctypes.POINTER(ctypes.c_uint8), ctypes.POINTER(vp)],
        "fkc_ipc_close": [vp],
        "fkc_tma_plan": [ctypes.POINTER(Grid), ctypes.c_int, ctypes.c_int, ctypes.POINTER(Tune),
                         ctypes.POINTER(ctypes.c_int)],
        "fkc_test_div_f32": [vp, vp, vp, vp, i64, vp],
        "fkc_test_div_f64": [vp, vp, vp, vp, i64, vp],
        "fkc_test_sqrt2_f32": [vp, vp, vp, i64, vp],
        "fkc_abi_version": [],
        "fkc_last_error": [],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_char_p if name == "fkc_last_error" else ctypes.c_int
    _lib = L
    return L


def ipc_export(ptr: int):
    """(64-byte handle, byte offset of ptr in its allocation)."""
    h = (ctypes.c_uint8 * 64)()
    off = ctypes.c_int64()
    check(lib().fkc_ipc_export(ptr, h, ctypes.byref(off)))
    return bytes(h), off.value


def ipc_open(handle: bytes) -> int:
    h = (ctypes.c_uint8 * 64).from_buffer_copy(handle)
    base = ctypes.c_void_p()
    check(lib().fkc_ipc_open(h, ctypes.byref(base)))
    return base.value


def ipc_close(base: int):
    check(lib().fkc_ipc_close(base))


def check(rc: int):
    if rc != FKC_OK:
        msg = lib().fkc_last_error().decode(errors="replace")
        if rc == FKC_EUSAGE:
            from .swdemo import LaunchError
            raise LaunchError(rc, msg)
        raise FkcError(rc, msg)


def bc_array(bc4) -> ctypes.Array:
    return (ctypes.c_int32 * 4)(*bc4)
