"""GPU tier: the chunked time loop of fkc_sw_advance_n (csrc/fkc_sw.cu
run_chunked) -- an eager SPEC-style loop (per-step reductions, CFL dt from
the device slots) of >= 128 steps on a mid-size grid replays ONE captured
graph of 32 steps whose reductions go to a private ring that a small kernel
appends to the caller's slots at a device step counter.  It must equal the
launch-per-step loop (FKC_NO_CHUNK=1) bit for bit: state (halos included),
dt series, every diagnostics row (host mirror too), errors."""

import os

import numpy as np
import pytest

from oracle import sw_oracle as so

pytestmark = pytest.mark.gpu


def dev_state(H, U, V, dx=1.0, dy=0.8, g=9.8):
    from paper_1107_2157_b200.field import DeviceField, Field, precision_of
    from paper_1107_2157_b200.swdemo import SWState
    p = precision_of(H.dtype)
    return SWState(*(DeviceField.from_field(Field.from_array(a, p)) for a in (H, U, V)), g, dx, dy)


def host(st):
    return tuple(f.to_numpy() for f in (st.H, st.U, st.V))


def run(H, U, V, splits, chunk, **kw):
    from paper_1107_2157_b200 import swdemo
    ny, nx = H.shape[0] - 2, H.shape[1] - 2
    prec = "f32" if H.dtype == np.float32 else "f64"
    steps = splits[-1]
    cfg = swdemo.SWConfig(nx=nx, ny=ny, steps=steps, precision=prec, **kw)
    if chunk:
        os.environ.pop("FKC_NO_CHUNK", None)
    else:
        os.environ["FKC_NO_CHUNK"] = "1"
    try:
        sim = swdemo.Simulation(cfg, state=dev_state(H, U, V), diagnostics=True, stream_rows=True)
        done = 0
        for k in splits:
            sim.advance(k - done)
            done = k
        res = sim.rows()
        host_rows = sim.host_rows[: steps + 1].numpy().copy()
    finally:
        os.environ.pop("FKC_NO_CHUNK", None)
    return res, host_rows


def same(a, b):
    """Bit-equal except the mass (an atomic double sum: its order, and so
    its last bits, vary from launch to launch -- 1e-12 relative)."""
    (ra, ha), (rb, hb) = a, b
    assert np.array_equal(ra.dts, rb.dts)
    assert all(np.array_equal(x, y) for x, y in zip(host(ra.state), host(rb.state)))
    xa, xb = np.array(ra.rows), np.array(rb.rows)
    assert np.array_equal(np.delete(xa, 3, axis=1), np.delete(xb, 3, axis=1))
    assert np.max(np.abs(xa[:, 3] - xb[:, 3]) / np.abs(xb[:, 3])) <= 1e-12
    assert np.array_equal(ha[:, 1:], hb[:, 1:])


@pytest.mark.parametrize("n,prec,mode,bc", [(512, "f32", "exact", "reflective"),
                                            (400, "f32", "fast", "periodic"),
                                            (320, "f64", "exact", "reflective"),
                                            (1024, "f32", "exact", "periodic")])
def test_chunked_cfl_run_equals_per_step_loop(n, prec, mode, bc):
    """The SPEC run (CFL 0.9 every step): 3 steps, then 200 from an odd step
    (one eager step to reach an even one, 6 chunks, 5 eager steps), then 140
    more (the cached graph replayed at a new position)."""
    H, U, V = so.init_state(n, n, prec)
    so.apply_boundary(H, U, V, bc)
    a = run(H, U, V, (3, 203, 343), True, cfl_factor=0.9, mode=mode, boundary=bc)
    b = run(H, U, V, (3, 203, 343), False, cfl_factor=0.9, mode=mode, boundary=bc)
    same(a, b)


def test_chunked_fixed_dt_diagnostics_run():
    """Fixed dt with per-step diagnostics (mass, maxima): chunked equals
    per-step; the dt series is the constant."""
    H, U, V = so.random_state(600, 360, "f32", seed=3)
    a = run(H, U, V, (256,), True, dt=0.04)
    b = run(H, U, V, (256,), False, dt=0.04)
    same(a, b)


def test_chunked_run_error_rows():
    """A negative depth mid-grid: the error word lands in the same rows and
    run() raises the same error as the per-step loop."""
    from paper_1107_2157_b200 import swdemo
    H, U, V = so.init_state(512, 512, "f32")
    H[200, 300] = -1.0
    errs = []
    for chunk in (True, False):
        cfg = swdemo.SWConfig(nx=512, ny=512, steps=160, cfl_factor=0.9)
        if not chunk:
            os.environ["FKC_NO_CHUNK"] = "1"
        try:
            sim = swdemo.Simulation(cfg, state=dev_state(H, U, V, 1.0, 1.0), diagnostics=True)
            sim.advance(160)
            errs.append(sim.diagnostics()["err"].copy())
        finally:
            os.environ.pop("FKC_NO_CHUNK", None)
    assert np.array_equal(errs[0], errs[1])
    assert np.any(errs[0] != 0)
    with pytest.raises(swdemo.NonPositiveDepth):
        swdemo.run(swdemo.SWConfig(nx=512, ny=512, steps=160, cfl_factor=0.9), state=dev_state(H, U, V, 1.0, 1.0))


def test_chunked_run_many_simulations():
    """More live simulations than cached chunk graphs (8): every run still
    equals its per-step twin (graphs are evicted and rebuilt)."""
    H, U, V = so.init_state(288, 256, "f32")
    want = run(H, U, V, (130,), False, cfl_factor=0.9)
    for _ in range(10):
        same(run(H, U, V, (130,), True, cfl_factor=0.9), want)


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_chunked_fixed_dt_without_reductions(mode):
    """An eager fixed-dt loop without diagnostics (no slots): 1 step, then
    300 from an odd step, then 130; chunked equals per-step bit for bit."""
    from paper_1107_2157_b200 import swdemo
    H, U, V = so.random_state(480, 300, "f32", seed=11)
    outs = []
    for chunk in (True, False):
        if not chunk:
            os.environ["FKC_NO_CHUNK"] = "1"
        try:
            cfg = swdemo.SWConfig(nx=480, ny=300, dt=0.02, mode=mode)
            sim = swdemo.Simulation(cfg, state=dev_state(H, U, V), diagnostics=False)
            for k in (1, 300, 130):
                sim.advance(k)
            outs.append(host(sim.state()))
        finally:
            os.environ.pop("FKC_NO_CHUNK", None)
    assert all(np.array_equal(x, y) for x, y in zip(*outs))


def test_chunked_loop_inside_a_callers_capture():
    """A caller capturing its own CUDA graph around advance(): the native
    loop sees the capturing stream, skips the chunk graph and enqueues the
    steps into the caller's capture; replaying it equals the eager run."""
    import torch

    from paper_1107_2157_b200 import swdemo
    H, U, V = so.random_state(480, 300, "f32", seed=12)
    cfg = swdemo.SWConfig(nx=480, ny=300, dt=0.02)
    want = swdemo.Simulation(cfg, state=dev_state(H, U, V), diagnostics=False)
    want.advance(256)
    s = torch.cuda.Stream()
    sim = swdemo.Simulation(cfg, state=dev_state(H, U, V), diagnostics=False, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        sim.advance(128)
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    assert sim.n == 128          # the host counter moved once, at capture
    got = host(sim.a)            # 256 steps: even, back in buffer A
    assert all(np.array_equal(x, y) for x, y in zip(got, host(want.state())))
