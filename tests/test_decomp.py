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
@pytest.mark.parametrize("exchange", ["pack", "fused", "fused-concurrent"])
def test_local_decomposed_gpu_bit_identical(px, py, bc, mode, exchange):
    """px*py tiles on one GPU (native kernels, per-side BC) == the
    single-domain GPU run, bit for bit (fast mode included: the
    decomposition does not change per-cell arithmetic).  pack: native line
    pack / copy / unpack; fused: the step kernel stores its boundary lines
    into the neighbours' halos; fused-concurrent: every tile on its own
    stream, ordered only by the in-kernel mailbox protocol."""
    from paper_1107_2157_b200 import swdemo
    from paper_1107_2157_b200.decomp import run_local_decomposed
    nx, ny, steps = 960, 512, 8
    cfg = swdemo.SWConfig(nx=nx, ny=ny, dt=0.05, boundary=bc, mode=mode, variant="tma")
    grid, states = run_local_decomposed(cfg, px, py, steps, exchange=exchange.split("-")[0],
                                        concurrent=exchange.endswith("concurrent"))
    sim = swdemo.Simulation(cfg, diagnostics=False)
    sim.advance(steps)
    ref = sim.state()
    for f in ("H", "U", "V"):
        got = gather_interior(grid, [getattr(s, f).to_numpy()[1:-1, 1:-1] for s in states])
        assert np.array_equal(got, getattr(ref, f).to_numpy()[1:-1, 1:-1]), f


# ---------------------------------------------------------------------------
# fused exchange (the step kernel writes the neighbours' halos)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("px,py", [(1, 2), (2, 2), (2, 4)])
@pytest.mark.parametrize("bc", ["reflective", "periodic"])
def test_peer_line_addressing(px, py, bc):
    """CPU tier: the peer-line addresses map every boundary cell of a tile
    onto exactly the neighbour halo cell the pack/unpack exchange fills.
    Fake 'device memory': each tile's field f lives at base(r, f) with
    pitch nx+7; decode the kernel's store address back to (tile, field, x, y)."""
    from paper_1107_2157_b200 import _native as N
    from paper_1107_2157_b200.decomp import OPPOSITE, set_peer_line
    g = CartGrid(px, py, 44, 36, bc)
    it = 4
    span = 1 << 24

    def base(r, f):
        return (1 + 3 * r + f) * span

    def pitch(r):
        return g.tile(r).nx + 7

    def decode(addr):
        k, off = divmod(addr, span)
        r, f = divmod(k - 1, 3)
        y, x = divmod(off // it, pitch(r))
        return r, f, x, y

    for r in range(g.size):
        t = g.tile(r)
        for s in (LEFT, RIGHT, DOWN, UP):
            n = g.neighbor(r, s)
            if n is None:
                continue
            nt = g.tile(n)
            line = N.PeerLine()
            set_peer_line(line, s, [base(n, f) for f in range(3)], pitch(n), nt.nx, nt.ny, it)
            # the cells the kernel stores for this side, and where they must land
            if s in (DOWN, UP):
                y = 1 if s == DOWN else t.ny
                cells = [(x, y) for x in range(1, t.nx + 1)]
                want = [(x, nt.ny + 1 if s == DOWN else 0) for x, _ in cells]
                idx = [x for x, _ in cells]
            else:
                x = 1 if s == LEFT else t.nx
                cells = [(x, y) for y in range(1, t.ny + 1)]
                want = [(nt.nx + 1 if s == LEFT else 0, y) for _, y in cells]
                idx = [y for _, y in cells]
            for f in range(3):
                got = [decode(line.p[f] + i * line.stride * it) for i in idx]
                assert all(gr == n and gf == f for gr, gf, _, _ in got)
                assert [(gx, gy) for _, _, gx, gy in got] == want
            # and the neighbour fills its OPPOSITE halo side from us
            assert g.neighbor(n, OPPOSITE[s]) == r


def _peer_worker(rank, world, port, px, py, nx, ny, steps, bc, mode, q):
    import torch
    import torch.distributed as dist

    from paper_1107_2157_b200 import swdemo
    from paper_1107_2157_b200.decomp import DistributedSimulation
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        grid = CartGrid(px, py, nx, ny, bc)
        cfg = swdemo.SWConfig(nx=nx, ny=ny, dt=0.05, boundary=bc, mode=mode, variant="tma")
        sim = DistributedSimulation(cfg, grid, rank, torch.device("cuda", 0), transport="peer")
        sim.advance(steps)
        torch.cuda.synchronize()
        st = sim.state()
        q.put((rank, *(getattr(st, f).to_numpy()[1:-1, 1:-1] for f in ("H", "U", "V"))))
        sim.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("px,py,bc", [(1, 2, "reflective"), (2, 2, "periodic")])
def test_ipc_peer_processes_bit_identical(px, py, bc):
    """One process per tile, all on cuda:0: CUDA-IPC peer memory, the fused
    in-kernel exchange and the mailbox ordering across processes (what runs
    across GPUs over NVLink) == the single-domain run, bit for bit."""
    import torch.multiprocessing as mp

    from paper_1107_2157_b200 import swdemo
    world = px * py
    nx, ny, steps = 960, 512, 10
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, px, py, nx, ny, steps, bc, "exact", q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, h, u, v = q.get(timeout=300)
        res[r] = (h, u, v)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    grid = CartGrid(px, py, nx, ny, bc)
    cfg = swdemo.SWConfig(nx=nx, ny=ny, dt=0.05, boundary=bc, mode="exact")
    sim = swdemo.Simulation(cfg, diagnostics=False)
    sim.advance(steps)
    ref = sim.state()
    for k, f in enumerate(("H", "U", "V")):
        got = gather_interior(grid, [res[r][k] for r in range(world)])
        assert np.array_equal(got, getattr(ref, f).to_numpy()[1:-1, 1:-1]), f


@pytest.mark.gpu
@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_local_fused_generic_kernel(precision):
    """The generic (one thread per cell) kernel's fused exchange and CTA-level
    mailbox protocol: odd tile widths (no TMA) and f64, concurrent streams."""
    from paper_1107_2157_b200 import swdemo
    from paper_1107_2157_b200.decomp import run_local_decomposed
    nx, ny, steps = 331, 203, 7
    cfg = swdemo.SWConfig(nx=nx, ny=ny, dt=0.05, boundary="periodic", mode="exact", precision=precision)
    grid, states = run_local_decomposed(cfg, 2, 2, steps, exchange="fused", concurrent=True)
    sim = swdemo.Simulation(cfg, diagnostics=False)
    sim.advance(steps)
    ref = sim.state()
    for f in ("H", "U", "V"):
        got = gather_interior(grid, [getattr(s, f).to_numpy()[1:-1, 1:-1] for s in states])
        assert np.array_equal(got, getattr(ref, f).to_numpy()[1:-1, 1:-1]), f


_WATCHDOG_SCRIPT = r"""
import ctypes, sys, torch
sys.path.insert(0, sys.argv[1])
from paper_1107_2157_b200 import _native as N, swdemo
from paper_1107_2157_b200.decomp import Mailbox, fill_sync, LEFT
cfg = swdemo.SWConfig(nx=int(sys.argv[2]), ny=64, dt=0.05, variant=sys.argv[3])
a = swdemo.init_state(cfg)
b = swdemo.SWState(a.H.empty_like(), a.U.empty_like(), a.V.empty_like())
mail, other = Mailbox(a.H.storage.device), Mailbox(a.H.storage.device)
args = swdemo._step_args(a, b, 0.05, ("none", "reflective", "reflective", "reflective"), "fast", cfg.variant)
fill_sync(args.sync, mail, {LEFT: other.word(1)}, 1)     # wait for epoch 1: nobody ever signals
N.check(N.lib().fkc_sw_step(ctypes.byref(args), torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print("UNEXPECTED: step completed")
"""


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["tma", "generic"])
def test_missing_neighbour_fails_loudly(variant):
    """A neighbour that never signals its mailbox must not hang the GPU: the
    waiting warps trip the watchdog (~2 s) and trap, the process sees a CUDA
    error and exits non-zero."""
    import subprocess
    import sys
    import time
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    t0 = time.time()
    r = subprocess.run([sys.executable, "-c", _WATCHDOG_SCRIPT, root, "480", variant], capture_output=True,
                       text=True, timeout=120)
    assert r.returncode != 0 and "UNEXPECTED" not in r.stdout, (r.stdout, r.stderr[-2000:])
    assert time.time() - t0 < 100


def _peer_error_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from paper_1107_2157_b200.decomp import CartGrid, PeerExchange, PeerSetupError
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        class F:
            def __init__(self):
                self.storage = torch.zeros(64)
                self.pitch = 8

            @property
            def ptr(self):      # host memory: CUDA IPC export must fail
                return self.storage.data_ptr()

        class S:
            def __init__(self):
                self.H, self.U, self.V = F(), F(), F()
        try:
            PeerExchange(CartGrid(1, world, 8, 8), rank, (S(), S()))
            q.put((rank, "no error"))
        except PeerSetupError as e:
            q.put((rank, "PeerSetupError" + (" with rank 0 and 1" if "rank 0" in str(e) and "rank 1" in str(e)
                                              else "")))
    finally:
        dist.destroy_process_group()


def test_peer_setup_error_is_collective():
    """CPU tier: when CUDA-IPC setup fails, every rank raises PeerSetupError
    (agreed over the process group), so 'auto' falls back consistently
    instead of leaving ranks stuck in a collective."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_error_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got == {0: "PeerSetupError with rank 0 and 1", 1: "PeerSetupError with rank 0 and 1"}, got


def _cfl_worker(rank, world, port, px, py, nx, ny, steps, bc, q, cfl_exchange="auto"):
    import torch
    import torch.distributed as dist

    from paper_1107_2157_b200 import swdemo
    from paper_1107_2157_b200.decomp import DistributedSimulation
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        grid = CartGrid(px, py, nx, ny, bc)
        cfg = swdemo.SWConfig(nx=nx, ny=ny, steps=steps, cfl_factor=0.9, boundary=bc, mode="exact",
                              variant="tma")
        sim = DistributedSimulation(cfg, grid, rank, torch.device("cuda", 0), transport="peer",
                                    cfl_exchange=cfl_exchange)
        assert sim.cfl_exchange == ("allreduce" if cfl_exchange == "allreduce" else "board")
        assert not sim.peer.pdl                       # all ranks share GPU 0
        sim.advance(steps)
        rows = sim.rows()
        st = sim.state()
        q.put((rank, rows, *(getattr(st, f).to_numpy()[1:-1, 1:-1] for f in ("H", "U", "V"))))
        sim.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("cfl_exchange", ["board", "allreduce"])
@pytest.mark.parametrize("px,py,bc", [(1, 2, "reflective"), (2, 2, "periodic")])
def test_distributed_cfl_run_matches_single_domain(px, py, bc, cfl_exchange):
    """The SPEC run across processes: CFL dt recomputed every step from the
    tiles' fused bounds -- combined on the device through the rank boards
    (the step kernels publish and read them over peer memory) or all-reduced
    (MIN) per step -- same dt series, state bit-identical and mass within
    1e-12 of the single-domain swdemo.run."""
    import torch.multiprocessing as mp

    from paper_1107_2157_b200 import swdemo
    world = px * py
    nx, ny, steps = 960, 512, 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cfl_worker, args=(r, world, port, px, py, nx, ny, steps, bc, q, cfl_exchange))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, rows, h, u, v = q.get(timeout=300)
        res[r] = (rows, h, u, v)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = swdemo.SWConfig(nx=nx, ny=ny, steps=steps, cfl_factor=0.9, boundary=bc, mode="exact", variant="tma")
    ref = swdemo.run(cfg)
    grid = CartGrid(px, py, nx, ny, bc)
    for k, f in enumerate(("H", "U", "V")):
        got = gather_interior(grid, [res[r][k + 1] for r in range(world)])
        assert np.array_equal(got, getattr(ref.state, f).to_numpy()[1:-1, 1:-1]), f
    rows = np.array(res[0][0])
    want = np.array(ref.rows)
    assert np.array_equal(rows[:, :3], want[:, :3])                       # step, t, dt
    assert np.array_equal(rows[:, 4:], want[:, 4:])                       # maxima
    assert np.max(np.abs(rows[:, 3] - want[:, 3]) / want[:, 3]) <= 1e-12   # mass


@pytest.mark.gpu
@pytest.mark.parametrize("seed", list(range(12)))
def test_fuzz_fused_exchange(seed):
    """Randomised decompositions with the fused exchange and concurrent
    per-tile streams (mailbox ordering only): process grid, extent, kernel
    (TMA warp-level / generic CTA-level protocol), boundary, mode, precision,
    steps -- bit-identical to the single-domain run with the same kernel."""
    from paper_1107_2157_b200 import swdemo
    from paper_1107_2157_b200.decomp import run_local_decomposed
    rng = np.random.default_rng(500 + seed)
    px, py = [(1, 2), (2, 1), (2, 2), (3, 2), (2, 3), (4, 2)][int(rng.integers(6))]
    prec = "f32" if rng.random() < 0.75 else "f64"
    variant = ["tma", "generic"][int(rng.integers(2))]
    cpl = 4 if prec == "f32" else 2
    if variant == "tma":          # every tile's width a multiple of the cells per lane
        nx = px * cpl * int(rng.integers(2, 700 // (px * cpl)))
    else:
        nx = int(rng.integers(8 * px, 700))
    ny = int(rng.integers(4 * py, 400))
    bc = ["reflective", "periodic"][int(rng.integers(2))]
    mode = ["exact", "fast"][int(rng.integers(2))]
    steps = int(rng.integers(2, 7))
    cfg = swdemo.SWConfig(nx=nx, ny=ny, dt=0.05, boundary=bc, mode=mode, precision=prec, variant=variant)
    grid, states = run_local_decomposed(cfg, px, py, steps, exchange="fused", concurrent=True)
    sim = swdemo.Simulation(cfg, diagnostics=False)
    sim.advance(steps)
    ref = sim.state()
    for f in ("H", "U", "V"):
        got = gather_interior(grid, [getattr(s, f).to_numpy()[1:-1, 1:-1] for s in states])
        assert np.array_equal(got, getattr(ref, f).to_numpy()[1:-1, 1:-1]), (f, px, py, nx, ny, bc, mode, prec,
                                                                               variant)
