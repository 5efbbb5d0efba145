"""Grid containers: the host :class:`Field` (API of the reference
``fkc.field.Field``, field.py:25-60) and its device twin :class:`DeviceField`.

``Field`` is the numeric I/O unit of the reference: a full ``(ny, nx)``
numpy array (halo included) plus its :class:`~.region.Extent` and a
precision tag ``"f32" | "f64"``.  ``DeviceField`` holds the same array in
HBM in the layout the sm_100a kernels stream with TMA:

* rows of ``pitch`` elements, ``pitch`` a multiple of 128 bytes, so every
  row starts on the same alignment;
* the storage begins ``lead`` elements before cell (0, 0) so that the first
  interior column (x = 1) is 128-byte aligned: 128-bit loads/stores of
  interior cells and 16-byte-aligned TMA boxes start exactly on cell 1;
* ``data`` is a strided torch view ``(ny, nx)`` of that storage -- the
  reference only checks shape and dtype (field.py:31-37), so padded views
  are valid Fields.

PyTorch is used only as the device allocator / copy engine here.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .region import Extent, Halo, Rect, interior_of

PRECISIONS = {"f32": np.float32, "f64": np.float64}
_CODES = {"f32": 0, "f64": 1}
ALIGN_BYTES = 128


def dtype_of(precision: str) -> np.dtype:
    if precision not in PRECISIONS:
        raise ValueError(f"unknown precision {precision!r}")
    return np.dtype(PRECISIONS[precision])


def precision_of(dtype) -> str:
    d = np.dtype(dtype)
    for k, v in PRECISIONS.items():
        if np.dtype(v) == d:
            return k
    raise ValueError(f"unsupported dtype {d}")


@dataclass
class Field:
    """Host grid: ``data.shape == (full.ny, full.nx)``, dtype per precision."""

    full: Extent
    data: np.ndarray
    precision: str = "f64"

    def __post_init__(self):
        if tuple(self.data.shape) != (self.full.ny, self.full.nx):
            raise ValueError(f"data shape {self.data.shape} != {(self.full.ny, self.full.nx)}")
        if self.data.dtype != dtype_of(self.precision):
            raise ValueError(f"dtype {self.data.dtype} does not match precision {self.precision}")

    @classmethod
    def zeros(cls, full: Extent, precision: str = "f64") -> "Field":
        return cls(full, np.zeros((full.ny, full.nx), dtype_of(precision)), precision)

    @classmethod
    def from_array(cls, arr, precision: str = "f64") -> "Field":
        a = np.asarray(arr, dtype_of(precision))
        return cls(Extent(a.shape[1], a.shape[0]), a, precision)

    def copy(self) -> "Field":
        return Field(self.full, self.data.copy(), self.precision)

    def rect_view(self, rect: Rect) -> np.ndarray:
        return self.data[rect.y0:rect.y0 + rect.ny, rect.x0:rect.x0 + rect.nx]

    def interior(self, halo: Halo) -> np.ndarray:
        return self.rect_view(interior_of(self.full, halo))

    def content_hash(self) -> bytes:
        return np.ascontiguousarray(self.data).tobytes()


def _torch():
    import torch  # noqa: WPS433 (deferred: torch import is slow)
    return torch


def padded_pitch(nx_full: int, itemsize: int) -> int:
    per = ALIGN_BYTES // itemsize
    return ((nx_full + per - 1) // per) * per


class DeviceField:
    """A full (halo-included) grid resident in GPU memory.

    ``storage`` is a 1-D torch tensor; ``data`` a ``(ny, nx)`` view whose
    element (0, 0) sits ``lead`` elements into ``storage``.  ``ptr`` is the
    device address of element (0, 0) -- what the C-ABI takes.
    """

    def __init__(self, full: Extent, precision: str = "f32", device=None, pitch: int | None = None,
                 fill: float | None = None):
        torch = _torch()
        self.full = full
        self.precision = precision
        itemsize = dtype_of(precision).itemsize
        self.pitch = pitch or padded_pitch(full.nx, itemsize)
        if self.pitch < full.nx:
            raise ValueError("pitch smaller than the row length")
        per = ALIGN_BYTES // itemsize
        self.lead = per - 1                     # column 1 lands on a 128-B boundary
        n = self.lead + full.ny * self.pitch + per
        tdtype = torch.float32 if precision == "f32" else torch.float64
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if fill is None:
            self.storage = torch.empty(n, dtype=tdtype, device=dev)
        else:
            self.storage = torch.full((n,), fill, dtype=tdtype, device=dev)
        self.data = self.storage[self.lead:self.lead + full.ny * self.pitch].view(full.ny, self.pitch)[:, :full.nx]

    # -- reference-compatible surface ------------------------------------
    @property
    def ptr(self) -> int:
        return self.data.data_ptr()

    @property
    def dtype_code(self) -> int:
        return _CODES[self.precision]

    def rect_view(self, rect: Rect):
        return self.data[rect.y0:rect.y0 + rect.ny, rect.x0:rect.x0 + rect.nx]

    def interior(self, halo: Halo):
        return self.rect_view(interior_of(self.full, halo))

    # -- transfers --------------------------------------------------------
    @classmethod
    def from_field(cls, f: Field, device=None, non_blocking: bool = False) -> "DeviceField":
        d = cls(f.full, f.precision, device)
        d.copy_from_host(f.data, non_blocking=non_blocking)
        return d

    def _stream(self, stream=None) -> int:
        torch = _torch()
        s = stream if stream is not None else torch.cuda.current_stream(self.storage.device)
        return s.cuda_stream

    def copy_from_host(self, arr, non_blocking: bool = False, stream=None):
        """Host (ny, nx) array -> device, one pitched DMA (fkc_copy2d).
        Pinned host memory gives full PCIe bandwidth and, with
        non_blocking=True, an asynchronous copy on `stream`."""
        from . import _native as N
        torch = _torch()
        a = arr.numpy() if isinstance(arr, torch.Tensor) else np.asarray(arr)
        if a.shape != (self.full.ny, self.full.nx) or a.dtype != dtype_of(self.precision):
            raise ValueError(f"host array {a.shape}/{a.dtype} does not match {self!r}")
        if a.strides[1] != a.itemsize:
            a = np.ascontiguousarray(a)
        it = a.itemsize
        sp = self._stream(stream)
        N.check(N.lib().fkc_copy2d(self.ptr, self.pitch * it, a.ctypes.data, a.strides[0],
                                   self.full.nx * it, self.full.ny, sp))
        if not non_blocking:
            torch.cuda.current_stream(self.storage.device).synchronize() if stream is None else stream.synchronize()
        return self

    def copy_to_host(self, out: np.ndarray, non_blocking: bool = False, stream=None) -> np.ndarray:
        """Device -> host (ny, nx) array (pinned for full bandwidth)."""
        from . import _native as N
        torch = _torch()
        if out.shape != (self.full.ny, self.full.nx) or out.dtype != dtype_of(self.precision) \
                or out.strides[1] != out.itemsize:
            raise ValueError("output array does not match the field")
        it = out.itemsize
        N.check(N.lib().fkc_copy2d(out.ctypes.data, out.strides[0], self.ptr, self.pitch * it,
                                   self.full.nx * it, self.full.ny, self._stream(stream)))
        if not non_blocking:
            torch.cuda.current_stream(self.storage.device).synchronize() if stream is None else stream.synchronize()
        return out

    def to_numpy(self) -> np.ndarray:
        out = np.empty((self.full.ny, self.full.nx), dtype_of(self.precision))
        return self.copy_to_host(out)

    def to_field(self, out: Field | None = None) -> Field:
        if out is not None:
            self.copy_to_host(out.data)
            return out
        return Field(self.full, self.to_numpy(), self.precision)

    def empty_like(self) -> "DeviceField":
        return DeviceField(self.full, self.precision, self.storage.device, self.pitch)

    def copy(self) -> "DeviceField":
        d = self.empty_like()
        d.storage.copy_(self.storage)
        return d

    def content_hash(self) -> bytes:
        return self.to_numpy().tobytes()

    def __repr__(self):
        return (f"DeviceField(full=({self.full.nx}, {self.full.ny}), precision={self.precision!r}, "
                f"pitch={self.pitch}, device={self.storage.device})")
