"""Region operators on device fields -- the ``region_cpy`` / ``region_ptr`` /
``cshift`` API of the reference's whole-array semantics (PAPER.md:404-410,
SPEC.md:289-306), executed by the C-ABI kernels.

* :func:`region_cpy` returns a fresh device array holding the interior of
  ``a`` selected by ``halo`` (refinterp.region_cpy_ref);
  the source is untouched.
* :func:`region_ptr` returns a writable strided view of that interior
  (the pointer binding of sema.py:290-307): stores write only the Rect.
* :func:`cshift` is the circular shift of SPEC.md:298-306:
  ``result(x, y) = a((x + offset) mod nx, y)`` for ``dim=1``.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .field import DeviceField
from .region import Extent, Halo, HaloTooLarge, interior_of


def _torch():
    import torch
    return torch


def _as_tensor2d(a):
    if isinstance(a, DeviceField):
        return a.data
    return a


def _is_host_field(a) -> bool:
    """A host Field of the reference's shape (``full`` / ``data`` numpy /
    ``precision``) -- ours or the reference's own ``fkc.field.Field``."""
    return hasattr(a, "full") and hasattr(a, "precision") and isinstance(getattr(a, "data", None), np.ndarray)


def _host_field_like(a, arr: np.ndarray):
    """A fresh host Field of ``a``'s own classes (Field and Extent) holding ``arr``."""
    ny, nx = arr.shape
    return type(a)(type(a.full)(nx, ny), arr, a.precision)


def region_cpy(a, halo):
    """Copy of ``interior_of(a.full, halo)``.

    A device field / tensor gives a contiguous device tensor; a host Field
    (ours or the reference's ``fkc.field.Field``) gives a fresh Field of the
    same class, like ``region_cpy_ref(a: Field, halo) -> Field``
     -- the copy itself runs on the device."""
    if _is_host_field(a):
        out = region_cpy(DeviceField.from_field(a), halo)
        return _host_field_like(a, out.cpu().numpy())
    torch = _torch()
    t = _as_tensor2d(a)
    h = Halo.of(halo)
    ny, nx = t.shape
    r = interior_of(Extent(nx, ny), h)            # raises HaloTooLarge
    if t.stride(1) != 1:
        raise ValueError("rows must be contiguous")
    code = 0 if t.dtype == torch.float32 else 1 if t.dtype == torch.float64 else None
    if code is None:
        raise ValueError(f"unsupported dtype {t.dtype}")
    out = torch.empty((r.ny, r.nx), dtype=t.dtype, device=t.device)
    halo4 = (ctypes.c_int32 * 4)(*h)
    N.check(N.lib().fkc_region_cpy(code, t.data_ptr(), nx, ny, t.stride(0), halo4, out.data_ptr(),
                                   out.stride(0), torch.cuda.current_stream(t.device).cuda_stream))
    return out


def region_ptr(a, halo):
    """Writable view of the interior selected by ``halo`` (no copy)."""
    t = _as_tensor2d(a)
    ny, nx = t.shape
    r = interior_of(Extent(nx, ny), Halo.of(halo))
    return t[r.y0:r.y0 + r.ny, r.x0:r.x0 + r.nx]


def cshift(a, dim: int, offset: int):
    """Circular shift along dim 1 (x, columns) or 2 (y, rows):
    ``result(x, y) = a((x + offset) mod nx, y)``.  A host
    Field gives a Field of the same class (``cshift_ref``), a device field /
    tensor a device tensor."""
    if _is_host_field(a):
        out = cshift(DeviceField.from_field(a), dim, offset)
        return _host_field_like(a, out.cpu().numpy())
    torch = _torch()
    t = _as_tensor2d(a)
    if t.stride(1) != 1:
        raise ValueError("rows must be contiguous")
    ny, nx = t.shape
    code = 0 if t.dtype == torch.float32 else 1 if t.dtype == torch.float64 else None
    if code is None:
        raise ValueError(f"unsupported dtype {t.dtype}")
    out = torch.empty((ny, nx), dtype=t.dtype, device=t.device)
    N.check(N.lib().fkc_cshift(code, t.data_ptr(), nx, ny, t.stride(0), dim, offset, out.data_ptr(),
                               out.stride(0), torch.cuda.current_stream(t.device).cuda_stream))
    return out


__all__ = ["region_cpy", "region_ptr", "cshift", "HaloTooLarge"]
