"""2-D domain decomposition.

CPU tier: process-grid logic, and a world_size 2 / 4 run over torch.distributed
(gloo) in which every rank advances its tile with the CPU oracle and
exchanges halos with the package's HaloExchanger/DistTransport -- the gathered
interiors must be bit-identical to the undecomposed oracle run.
GPU tier: the same decomposition with the CUDA kernel (per-side BC, native
pack/unpack) on one device through LocalTransport.
"""

import os
import socket

import numpy as np
import pytest

from oracle import sw_oracle as so
from paper_1107_2157_b200.decomp import (DOWN, LEFT, RIGHT, UP, CartGrid, choose_grid, gather_interior,
                                         gaussian_tile)


def test_choose_grid():
    assert choose_grid(1) == (1, 1)
    assert choose_grid(2) == (1, 2)
    assert choose_grid(4) == (2, 2)
    assert choose_grid(8) == (2, 4)


@pytest.mark.parametrize("px,py", [(1, 2), (2, 2), (2, 4), (3, 1)])
def test_tiles_partition_and_neighbors(px, py):
    g = CartGrid(px, py, 37, 29, "reflective")
    seen = np.zeros((29, 37), int)
    for r in range(g.size):
        t = g.tile(r)
        seen[t.y0:t.y0 + t.ny, t.x0:t.x0 + t.nx] += 1
        for s, o in ((LEFT, RIGHT), (RIGHT, LEFT), (DOWN, UP), (UP, DOWN)):
            n = g.neighbor(r, s)
            if n is not None:
                assert g.neighbor(n, o) == r
    assert (seen == 1).all()
    # physical walls keep the boundary condition, internal sides are exchanged
    assert g.local_bc(0)[LEFT] == "reflective" and g.local_bc(0)[DOWN] == "reflective"


def test_periodic_wraps():
    g = CartGrid(2, 2, 8, 8, "periodic")
    assert g.neighbor(0, LEFT) == 1 and g.neighbor(0, DOWN) == 2
    assert g.local_bc(0) == ("none",) * 4
    g1 = CartGrid(1, 2, 8, 8, "periodic")
    assert g1.local_bc(0) == ("periodic", "periodic", "none", "none")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, px, py, nx, ny, steps, bc, q):
    import torch
    import torch.distributed as dist

    from paper_1107_2157_b200.decomp import DistTransport, HaloExchanger, TorchLines
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        grid = CartGrid(px, py, nx, ny, bc)
        t = grid.tile(rank)
        sides = grid.local_bc(rank)
        H = np.zeros((t.ny + 2, t.nx + 2), np.float32)
        U = np.zeros_like(H)
        V = np.zeros_like(H)
        H[1:-1, 1:-1] = gaussian_tile(grid, rank, "f32")
        # add a deterministic momentum field so cross terms are exercised
        yy, xx = np.meshgrid(np.arange(t.y0, t.y0 + t.ny), np.arange(t.x0, t.x0 + t.nx), indexing="ij")
        U[1:-1, 1:-1] = (0.01 * np.sin(0.3 * xx + 0.1 * yy)).astype(np.float32)
        V[1:-1, 1:-1] = (0.01 * np.cos(0.2 * xx - 0.4 * yy)).astype(np.float32)

        class St:
            pass
        st = St()
        st.H, st.U, st.V = (torch.from_numpy(a) for a in (H, U, V))
        ex = HaloExchanger(grid, rank, DistTransport(), TorchLines(), "cpu", torch.float32)
        so.apply_boundary_sides(H, U, V, sides)
        ex.exchange(st)
        for _ in range(steps):
            h, u, v = so.wave_advance(1.0, 1.0, 0.05, H, U, V)
            H[1:-1, 1:-1], U[1:-1, 1:-1], V[1:-1, 1:-1] = h, u, v
            so.apply_boundary_sides(H, U, V, sides)
            ex.exchange(st)
        q.put((rank, H[1:-1, 1:-1].copy(), U[1:-1, 1:-1].copy(), V[1:-1, 1:-1].copy()))
    finally:
        dist.destroy_process_group()


def _global_reference(nx, ny, steps, bc):
    grid = CartGrid(1, 1, nx, ny, bc)
    H = np.zeros((ny + 2, nx + 2), np.float32)
    U = np.zeros_like(H)
    V = np.zeros_like(H)
    H[1:-1, 1:-1] = gaussian_tile(grid, 0, "f32")
    yy, xx = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    U[1:-1, 1:-1] = (0.01 * np.sin(0.3 * xx + 0.1 * yy)).astype(np.float32)
    V[1:-1, 1:-1] = (0.01 * np.cos(0.2 * xx - 0.4 * yy)).astype(np.float32)
    so.apply_boundary(H, U, V, bc)
    for _ in range(steps):
        H, U, V = so.step(H, U, V, 1.0, 1.0, 0.05, boundary=bc)
    return H[1:-1, 1:-1], U[1:-1, 1:-1], V[1:-1, 1:-1]


@pytest.mark.parametrize("px,py", [(1, 2), (2, 2)])
@pytest.mark.parametrize("bc", ["reflective", "periodic"])
def test_gloo_decomposed_bit_identical(px, py, bc):
    import torch.multiprocessing as mp
    world = px * py
    nx, ny, steps = 40, 34, 6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, px, py, nx, ny, steps, bc, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, h, u, v = q.get(timeout=180)
        res[r] = (h, u, v)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    grid = CartGrid(px, py, nx, ny, bc)
    want = _global_reference(nx, ny, steps, bc)
    for k in range(3):
        got = gather_interior(grid, [res[r][k] for r in range(world)])
        assert np.array_equal(got, want[k])


@pytest.mark.gpu
@pytest.mark.parametrize("px,py", [(1, 2), (2, 2), (2, 4)])
@pytest.mark.parametrize("bc", ["reflective", "periodic"])
@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_local_decomposed_gpu_bit_identical(px, py, bc, mode):
    """px*py tiles on one GPU (native kernels, per-side BC, native line
    pack/unpack) == the single-domain GPU run, bit for bit (fast mode
    included: the decomposition does not change per-cell arithmetic)."""
    from paper_1107_2157_b200 import swdemo
    from paper_1107_2157_b200.decomp import run_local_decomposed
    nx, ny, steps = 960, 512, 8
    cfg = swdemo.SWConfig(nx=nx, ny=ny, dt=0.05, boundary=bc, mode=mode)
    grid, states = run_local_decomposed(cfg, px, py, steps)
    sim = swdemo.Simulation(cfg, diagnostics=False)
    sim.advance(steps)
    ref = sim.state()
    for f in ("H", "U", "V"):
        got = gather_interior(grid, [getattr(s, f).to_numpy()[1:-1, 1:-1] for s in states])
        assert np.array_equal(got, getattr(ref, f).to_numpy()[1:-1, 1:-1]), f
