"""GPU tier: the streamed host run (fkc_sw_run_host, swdemo.run with host
state and host output) -- the upload, the steps and the download overlap:
bands of rows are stepped as a wavefront while later bands are still
crossing PCIe.  Exact mode must equal the device-resident run bit for bit
(full arrays, halos included) and the per-step diagnostics rows must match;
fast mode value-identical to the per-step fast kernels."""

import numpy as np
import pytest

from oracle import c_oracle
from oracle import sw_oracle as so

pytestmark = pytest.mark.gpu

_PINNED = []   # pinned torch buffers behind the host arrays (kept alive for the module)


def host_state(H, U, V, dx=1.0, dy=0.8, pinned=True):
    import torch
    from paper_1107_2157_b200.field import Field, precision_of
    from paper_1107_2157_b200.swdemo import SWState
    p = precision_of(H.dtype)
    fs = []
    for a in (H, U, V):
        if pinned:
            t = torch.empty(a.shape, dtype=torch.float32 if p == "f32" else torch.float64, pin_memory=True)
            _PINNED.append(t)
            arr = t.numpy()
            arr[...] = a
        else:
            arr = a.copy()
        fs.append(Field.from_array(arr, p))
    return SWState(*fs, 9.8, dx, dy)


def empty_like_state(st, pinned=True):
    return host_state(*(np.zeros_like(getattr(st, n).data) for n in ("H", "U", "V")), st.dx, st.dy, pinned)


def device_run(cfg, st):
    from paper_1107_2157_b200 import swdemo
    sim = swdemo.Simulation(cfg, state=st.to_device(), diagnostics=True, stream_rows=True)
    sim.advance(cfg.steps)
    res = sim.rows()
    return res, tuple(getattr(res.state, n).to_numpy() for n in ("H", "U", "V"))


@pytest.mark.parametrize("steps", [0, 1, 5, 33, 70])
def test_streamed_exact_equals_device_run(steps):
    """Every phase of the schedule: upload-only (0 steps), a wavefront that
    also downloads (<= 32 steps), wavefront + wavefront (33), wavefront +
    whole-grid steps + wavefront (70); 35 bands of 32 rows (ny 1100 is not a
    multiple of the band; 16-row bands: 69 of them, 20 tasks per wave launch)."""
    from paper_1107_2157_b200 import swdemo
    H, U, V = so.random_state(512, 1100, "f32", seed=steps + 3)
    st = host_state(H, U, V)
    cfg = swdemo.SWConfig(nx=512, ny=1100, steps=steps, dt=0.04)
    out = empty_like_state(st)
    res = swdemo._run_streamed(cfg, st, out, band_rows=16)
    want_res, want = device_run(cfg, st)
    for x, w in zip((out.H.data, out.U.data, out.V.data), want):
        assert np.array_equal(x, w)
    assert np.array_equal(res.dts, want_res.dts)
    got_rows, want_rows = np.array(res.rows).reshape(-1, 6), np.array(want_res.rows).reshape(-1, 6)
    assert np.array_equal(got_rows[:, :3], want_rows[:, :3])
    assert np.array_equal(got_rows[:, 4:], want_rows[:, 4:])
    if steps:
        assert np.max(np.abs(got_rows[:, 3] - want_rows[:, 3]) / want_rows[:, 3]) <= 1e-12
    if steps == 5:
        ref = c_oracle.run_fixed(H, U, V, 5, 1.0, 0.8, 0.04)
        assert all(np.array_equal(x, w) for x, w in zip((out.H.data, out.U.data, out.V.data), ref))


@pytest.mark.parametrize("band_rows", [16, 32, 100, 1100, 5000])
@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_streamed_band_sizes(band_rows, prec):
    """Results never depend on the band height (one band = no overlap)."""
    from paper_1107_2157_b200 import swdemo
    H, U, V = so.random_state(256, 1100, prec, seed=band_rows)
    st = host_state(H, U, V)
    cfg = swdemo.SWConfig(nx=256, ny=1100, steps=9, dt=0.04, precision=prec)
    out = empty_like_state(st)
    swdemo._run_streamed(cfg, st, out, band_rows=band_rows)
    _, want = device_run(cfg, st)
    for x, w in zip((out.H.data, out.U.data, out.V.data), want):
        assert np.array_equal(x, w)


def test_streamed_fast_and_pageable():
    """Fast mode equals the per-step fast kernels' values; pageable (not
    pinned) host arrays are correct too (the copies just do not overlap)."""
    from paper_1107_2157_b200 import swdemo
    H, U, V = so.random_state(1024, 1024, "f32", seed=9)
    for pinned in (True, False):
        st = host_state(H, U, V, pinned=pinned)
        cfg = swdemo.SWConfig(nx=1024, ny=1024, steps=12, dt=0.04, mode="fast")
        out = empty_like_state(st, pinned=pinned)
        swdemo._run_streamed(cfg, st, out)
        _, want = device_run(cfg, st)
        for x, w in zip((out.H.data, out.U.data, out.V.data), want):
            assert np.array_equal(x, w)


def test_run_dispatches_large_host_runs():
    """swdemo.run with a host state, host output and a fixed dt on a grid of
    >= 2^20 cells takes the streamed path; CFL runs and periodic rows keep
    the device loop.  All equal the device run."""
    from paper_1107_2157_b200 import swdemo
    H, U, V = so.random_state(1024, 1024, "f32", seed=4)
    st = host_state(H, U, V)
    cfg = swdemo.SWConfig(nx=1024, ny=1024, steps=6, dt=0.04)
    assert swdemo._streamable(cfg, st, None)
    res = swdemo.run(cfg, state=st, to_host=True)
    _, want = device_run(cfg, st)
    assert all(np.array_equal(getattr(res.state, n).data, w) for n, w in zip(("H", "U", "V"), want))
    assert not swdemo._streamable(swdemo.SWConfig(nx=1024, ny=1024, steps=6), st, None)
    assert not swdemo._streamable(swdemo.SWConfig(nx=1024, ny=1024, steps=6, dt=0.04, boundary="periodic"), st, None)
    assert not swdemo._streamable(swdemo.SWConfig(nx=128, ny=128, steps=6, dt=0.04),
                                  host_state(*(a[:130, :130].copy() for a in (H, U, V))), None)


def test_streamed_errors():
    from paper_1107_2157_b200 import swdemo
    H, U, V = so.random_state(512, 600, "f32", seed=1)
    H[300, 200] = -1.0
    st = host_state(H, U, V)
    cfg = swdemo.SWConfig(nx=512, ny=600, steps=3, dt=0.04)
    with pytest.raises(swdemo.NonPositiveDepth):
        swdemo._run_streamed(cfg, st, empty_like_state(st))
    H, U, V = so.random_state(510, 64, "f32", seed=1)      # not the TMA layout
    st = host_state(H, U, V)
    with pytest.raises(swdemo.LaunchError):
        swdemo._run_streamed(swdemo.SWConfig(nx=510, ny=64, steps=3, dt=0.04), st, empty_like_state(st))


def test_run_host_c_abi_padded_host_pitch():
    """fkc_sw_run_host through the C-ABI with host rows padded beyond the
    row length (host pitch 37 elements past nx+2): same bits as the device
    run; the padding is never written."""
    import ctypes

    import torch

    from paper_1107_2157_b200 import _native as N
    from paper_1107_2157_b200 import swdemo
    nx, ny, pad = 384, 700, 37
    H, U, V = so.random_state(nx, ny, "f32", seed=12)
    hp = nx + 2 + pad
    bufs_in = [torch.full((ny + 2, hp), -7.0, dtype=torch.float32, pin_memory=True) for _ in range(3)]
    bufs_out = [torch.full((ny + 2, hp), -7.0, dtype=torch.float32, pin_memory=True) for _ in range(3)]
    for b, a in zip(bufs_in, (H, U, V)):
        b[:, :nx + 2] = torch.from_numpy(a)
    st = host_state(H, U, V)
    cfg = swdemo.SWConfig(nx=nx, ny=ny, steps=7, dt=0.04)
    dev = swdemo.SWState(*(swdemo.DeviceField(st.full, "f32") for _ in range(3)), 9.8, 1.0, 0.8)
    oth = swdemo.SWState(*(f.empty_like() for f in (dev.H, dev.U, dev.V)), 9.8, 1.0, 0.8)
    L = N.LoopArgs()
    L.step = swdemo._step_args(dev, oth, 0.04, "reflective", "exact", "auto")
    L.steps = 7
    src = (ctypes.c_void_p * 3)(*(b.data_ptr() for b in bufs_in))
    dst = (ctypes.c_void_p * 3)(*(b.data_ptr() for b in bufs_out))
    s = torch.cuda.current_stream()
    N.check(N.lib().fkc_sw_run_host(ctypes.byref(L), src, dst, hp * 4, 48, s.cuda_stream))
    s.synchronize()
    _, want = device_run(cfg, st)
    for b, w in zip(bufs_out, want):
        assert np.array_equal(b[:, :nx + 2].numpy(), w)
        assert bool((b[:, nx + 2:] == -7.0).all())


@pytest.mark.parametrize("nx,ny,steps,band", [(128, 5, 3, 0), (4, 40, 6, 16), (8, 1, 2, 0), (256, 33, 40, 16)])
def test_streamed_tiny_and_thin_grids(nx, ny, steps, band):
    """Grids thinner than one band, one-row grids, a 4-column grid, and a run
    longer than both wavefronts on a 3-band grid: same bits as the device run."""
    from paper_1107_2157_b200 import swdemo
    H, U, V = so.random_state(nx, ny, "f32", seed=nx + ny)
    st = host_state(H, U, V)
    cfg = swdemo.SWConfig(nx=nx, ny=ny, steps=steps, dt=0.04)
    out = empty_like_state(st)
    res = swdemo._run_streamed(cfg, st, out, band_rows=band)
    want_res, want = device_run(cfg, st)
    for x, w in zip((out.H.data, out.U.data, out.V.data), want):
        assert np.array_equal(x, w)
    assert np.array_equal(res.dts, want_res.dts)
