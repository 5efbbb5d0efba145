"""B200-native (sm_100a) shallow-water hot path of arXiv 1107.2157 (ForOpenCL).

Drop-in for the reference package's solver path (``fkc.swdemo`` /
``fkc.refinterp`` region operators): same API, executed by
hand-written CUDA kernels behind the C-ABI in ``include/fkc_sw.h``.
"""

from .region import (Extent, Halo, HaloTooLarge, Rect, UNIT_HALO, ZERO_HALO, global_coord,  # noqa: F401
                     interior_of, local_linear_index, local_tile_extent, owned_cell)
from .field import DeviceField, Field  # noqa: F401

__version__ = "0.1.0"


def native():
    """The loaded C-ABI library (raises NativeUnavailable if not built)."""
    from . import _native
    return _native.lib()
