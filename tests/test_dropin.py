"""Drop-in with the reference's own types (VERDICT r01 "next" item 3).

CPU tier: ``paper_1107_2157_b200.region`` against the reference's
``fkc.region`` (region.py:13-114) exhaustively over small halos / extents /
groups -- same values, same errors -- and the C-ABI usage errors surfacing as
the reference's ``LaunchError`` (a ``ValueError``).

GPU tier: states built from ``fkc.field.Field`` (field.py:25-60) and
``fkc.region.Halo`` objects go through ``swdemo.advance / step_native /
run`` and ``refinterp.region_cpy / cshift`` unchanged, and come back as the
reference's own Field type, bit-identical to the oracle.
"""

import itertools

import numpy as np
import pytest

from conftest import reference_fkc
from paper_1107_2157_b200 import region as R

REF = reference_fkc()
needs_ref = pytest.mark.skipif(REF is None, reason="reference fkc package not installed (baseline/_ref)")


def _both(fn_ours, fn_ref):
    """(kind, value) of calling each: values compared, exception classes by name."""
    out = []
    for fn in (fn_ours, fn_ref):
        try:
            v = fn()
            out.append(("ok", tuple(v) if not isinstance(v, int) else v))
        except ValueError as e:
            out.append(("err", type(e).__name__))
    return out


def _t(x):
    """Normalise a Rect / Extent of either implementation to a tuple."""
    if hasattr(x, "x0"):
        return (x.x0, x.y0, x.nx, x.ny)
    if hasattr(x, "nx"):
        return (x.nx, x.ny)
    return x


@needs_ref
def test_region_differential_exhaustive():
    _, fr = REF
    n = 0
    for l, r, d, u in itertools.product(range(-1, 4), repeat=4):
        mk = [lambda: R.Halo(l, r, d, u), lambda: fr.Halo(l, r, d, u)]
        res = []
        for m in mk:
            try:
                res.append(("ok", tuple(m())))
            except ValueError as e:
                res.append(("err", type(e).__name__))
        assert res[0] == res[1], (l, r, d, u, res)
        if res[0][0] == "err":
            continue
        ho, hr = R.Halo(l, r, d, u), fr.Halo(l, r, d, u)
        assert (ho.deficit_x, ho.deficit_y) == (hr.deficit_x, hr.deficit_y)
        assert tuple(R.Halo.of([l, r, d, u])) == tuple(fr.Halo.of([l, r, d, u]))
        for nx in range(0, 13):
            for ny in range(0, 9, 2):
                got = []
                for X, H, io in ((R.Extent, ho, R.interior_of), (fr.Extent, hr, fr.interior_of)):
                    try:
                        got.append(("ok", _t(io(X(nx, ny), H))))
                    except ValueError as e:      # HaloTooLarge, or Extent < 1
                        got.append(("err", type(e).__name__))
                assert got[0] == got[1], (l, r, d, u, nx, ny, got)
                n += 1
        for gx, gy in ((16, 8), (4, 4), (1, 3)):
            to = R.local_tile_extent(R.Extent(gx, gy), ho)
            tr = fr.local_tile_extent(fr.Extent(gx, gy), hr)
            assert _t(to) == _t(tr) and to.cells == tr.cells
            for lx, ly in ((0, 0), (gx + l + r - 1, gy + d + u - 1), (1, 2)):
                assert R.local_linear_index(lx, ly, gx, ho) == fr.local_linear_index(lx, ly, gx, hr)
            for gid in ((0, 0), (2, 1), (5, 7)):
                for th in ((0, 0), (gx - 1, gy - 1)):
                    assert R.global_coord(gid, th, R.Extent(gx, gy)) == fr.global_coord(gid, th, fr.Extent(gx, gy))
                    assert R.owned_cell(gid, th, R.Extent(gx, gy), ho) == \
                        fr.owned_cell(gid, th, fr.Extent(gx, gy), hr)
    assert n > 5000
    # the product's errors ARE ValueErrors with the reference's class names
    assert issubclass(R.HaloTooLarge, ValueError)


@needs_ref
def test_product_accepts_reference_halo_objects():
    _, fr = REF
    rc = R.interior_of(R.Extent(6, 5), R.Halo.of(fr.Halo(0, 1, 1, 1)))
    assert _t(rc) == _t(fr.interior_of(fr.Extent(6, 5), fr.Halo(0, 1, 1, 1))) == (0, 1, 5, 3)


def test_usage_errors_are_launch_errors():
    """Every FKC_EUSAGE of the C-ABI surfaces as swdemo.LaunchError, a
    ValueError like the reference's -- no GPU needed."""
    from paper_1107_2157_b200 import _native as N
    from paper_1107_2157_b200 import swdemo
    L = N.lib()
    with pytest.raises(swdemo.LaunchError) as ei:
        N.check(L.fkc_sw_step(None, None))
    assert isinstance(ei.value, ValueError) and ei.value.code == N.FKC_EUSAGE and "null" in str(ei.value)
    with pytest.raises(ValueError):
        N.check(L.fkc_sw_advance_n(None, None))
    assert isinstance(swdemo.LaunchError("x"), ValueError)


def test_cshift_rejects_unsupported_dtypes():
    """cshift validates the dtype before any device call (an
    int32 / f16 tensor used to be read as 8-byte elements)."""
    import torch
    from paper_1107_2157_b200 import refinterp
    for dt in (torch.int32, torch.float16, torch.bfloat16, torch.int64):
        with pytest.raises(ValueError):
            refinterp.cshift(torch.zeros((4, 8), dtype=dt), 1, 1)
        with pytest.raises(ValueError):
            refinterp.region_cpy(torch.zeros((4, 8), dtype=dt), (1, 1, 1, 1))


# ---------------------------------------------------------------------------
# GPU tier
# ---------------------------------------------------------------------------

def _ref_state(ff, fr, H, U, V, prec, g=9.8, dx=1.0, dy=1.0):
    from paper_1107_2157_b200 import swdemo
    ny, nx = H.shape
    mk = lambda a: ff.Field(fr.Extent(nx, ny), a.copy(), prec)   # noqa: E731
    return swdemo.SWState(mk(H), mk(U), mk(V), g, dx, dy)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("variant", ["tma", "generic"])
def test_reference_fields_through_advance(prec, variant):
    from oracle import sw_oracle as so
    from paper_1107_2157_b200 import swdemo
    ff, fr = REF
    H, U, V = so.random_state(256, 96, prec, seed=77)
    st = _ref_state(ff, fr, H, U, V, prec, dx=1.0, dy=0.7)
    h0 = [f.content_hash() for f in (st.H, st.U, st.V)]
    out = swdemo.advance(st, 0.05, "reflective", "exact", variant)
    assert all(isinstance(f, ff.Field) for f in (out.H, out.U, out.V))   # the caller's own Field type
    assert isinstance(out.H.full, fr.Extent)
    want = so.step(H, U, V, 1.0, 0.7, 0.05)
    for f, w in zip((out.H, out.U, out.V), want):
        assert np.array_equal(f.data, w)
    assert [f.content_hash() for f in (st.H, st.U, st.V)] == h0            # inputs untouched
    # step_native on reference Fields, interior of the result via the reference's own helper
    out2 = swdemo.step_native(st, 0.05)
    inner = out2.H.interior(fr.Halo(1, 1, 1, 1))
    assert np.array_equal(inner, want[0][1:-1, 1:-1])


@pytest.mark.gpu
@needs_ref
def test_reference_fields_through_run():
    from oracle import sw_oracle as so
    from paper_1107_2157_b200 import swdemo
    ff, fr = REF
    H, U, V = so.init_state(128, 64, "f32")
    st = _ref_state(ff, fr, H, U, V, "f32")
    cfg = swdemo.SWConfig(nx=128, ny=64, steps=20, cfl_factor=0.9, precision="f32")
    res = swdemo.run(cfg, state=st, to_host=True)
    ref = so.run(H, U, V, 20, cfl=0.9)
    assert np.array_equal(res.state.H.data, ref.H) and np.array_equal(res.state.V.data, ref.V)
    assert [r[2] for r in res.rows] == [r[2] for r in ref.rows]              # dt series, bit for bit


@pytest.mark.gpu
@needs_ref
def test_reference_fields_through_region_ops():
    from oracle import sw_oracle as so
    from paper_1107_2157_b200 import refinterp
    ff, fr = REF
    a = np.arange(6 * 5, dtype=np.float64).reshape(5, 6)
    a = 10.0 * np.arange(5)[:, None] + np.arange(6)[None, :]                # data(x, y) = 10 y + x
    F = ff.Field(fr.Extent(6, 5), a, "f64")
    out = refinterp.region_cpy(F, fr.Halo(0, 1, 1, 1))
    assert isinstance(out, ff.Field) and isinstance(out.full, fr.Extent)
    assert (out.full.nx, out.full.ny) == (5, 3) and out.data[0, 0] == 10.0
    assert np.array_equal(out.data, so.region(a, (0, 1, 1, 1)))
    with pytest.raises(fr.HaloTooLarge.__base__):
        refinterp.region_cpy(F, fr.Halo(3, 3, 0, 0))
    one = ff.Field(fr.Extent(4, 1), np.array([[1, 2, 3, 4]], np.float32), "f32")
    sh = refinterp.cshift(one, 1, 1)
    assert isinstance(sh, ff.Field) and sh.data.tolist() == [[2, 3, 4, 1]]
    for off in (0, 4, -3, 9):
        assert np.array_equal(refinterp.cshift(F, 2, off).data, so.cshift(a, 2, off))
