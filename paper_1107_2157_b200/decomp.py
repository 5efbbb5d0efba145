"""2-D domain decomposition of the shallow-water grid over GPUs (one process
per GPU) with a one-cell halo exchange per step -- SURVEY.md 8(e).

The reference runs on one device (the paper leaves MPI generation as future
work).  Every cell update needs only the 1-cell ring of
H, U, V (a 3x3 cross stencil; corners are never read), so a Cartesian split
needs exactly one exchange of boundary lines per step:

* rank (rx, ry) of a px x py grid owns a rectangle of the global interior;
* the step kernel applies the physical boundary condition on the sides that
  touch the global boundary and leaves the other halo sides alone
  (``FKC_BC_NONE``);
* after the step, each rank sends the outermost interior row/column of the
  new H, U, V to the neighbour on that side, which writes it into its halo
  (periodic boundaries wrap around the process grid; an axis with one rank
  wraps locally in the kernel).

Per-cell arithmetic is unchanged by the decomposition, so the decomposed
state is bit-identical to the single-domain state (tested).  Transports:
``DistTransport`` (torch.distributed P2P: NCCL on GPUs, gloo in the CPU
tests) and ``LocalTransport`` (several sub-domains in one process, used to
validate the GPU path on a single device).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from .region import Extent

LEFT, RIGHT, DOWN, UP = 0, 1, 2, 3
OPPOSITE = {LEFT: RIGHT, RIGHT: LEFT, DOWN: UP, UP: DOWN}
# transfer order: every rank issues the same sequence, so P2P messages
# between any pair of ranks match in order (NCCL) and by tag (gloo)
EXCHANGE_ORDER = (RIGHT, LEFT, UP, DOWN)


def choose_grid(n: int) -> Tuple[int, int]:
    """px x py with py >= px (more of the halo in contiguous rows)."""
    best = (1, n)
    for px in range(1, int(n ** 0.5) + 1):
        if n % px == 0:
            best = (px, n // px)
    return best


@dataclass(frozen=True)
class Tile:
    rank: int
    rx: int
    ry: int
    x0: int       # global interior column offset (0-based) of the first owned column
    y0: int
    nx: int
    ny: int


class CartGrid:
    """px x py Cartesian split of an NX x NY interior; rank = ry*px + rx."""

    def __init__(self, px: int, py: int, NX: int, NY: int, boundary: str = "reflective"):
        if px < 1 or py < 1 or NX < px or NY < py:
            raise ValueError("bad process grid")
        self.px, self.py, self.NX, self.NY = px, py, NX, NY
        self.boundary = boundary
        self.periodic = boundary == "periodic"

    @property
    def size(self) -> int:
        return self.px * self.py

    @staticmethod
    def _split(n: int, parts: int, i: int) -> Tuple[int, int]:
        base, extra = divmod(n, parts)
        start = i * base + min(i, extra)
        return start, base + (1 if i < extra else 0)

    def tile(self, rank: int) -> Tile:
        rx, ry = rank % self.px, rank // self.px
        x0, nx = self._split(self.NX, self.px, rx)
        y0, ny = self._split(self.NY, self.py, ry)
        return Tile(rank, rx, ry, x0, y0, nx, ny)

    def neighbor(self, rank: int, side: int) -> Optional[int]:
        """Rank across `side`, None at a physical (non-periodic) boundary or
        when the axis has a single rank (the kernel wraps locally)."""
        t = self.tile(rank)
        rx, ry = t.rx, t.ry
        if side in (LEFT, RIGHT):
            if self.px == 1:
                return None
            rx += -1 if side == LEFT else 1
            if not 0 <= rx < self.px:
                if not self.periodic:
                    return None
                rx %= self.px
        else:
            if self.py == 1:
                return None
            ry += -1 if side == DOWN else 1
            if not 0 <= ry < self.py:
                if not self.periodic:
                    return None
                ry %= self.py
        return ry * self.px + rx

    def local_bc(self, rank: int) -> Tuple[str, str, str, str]:
        """Per-side boundary handling for the step kernel of `rank`."""
        out = []
        for side in (LEFT, RIGHT, DOWN, UP):
            single = self.px == 1 if side in (LEFT, RIGHT) else self.py == 1
            if self.neighbor(rank, side) is not None:
                out.append("none")                  # filled by the exchange
            elif self.periodic and single:
                out.append("periodic")              # local wrap
            else:
                out.append(self.boundary)           # physical wall
        return tuple(out)


# ---------------------------------------------------------------------------
# line pack / unpack
# ---------------------------------------------------------------------------

def _line_len(side: int, nx: int, ny: int) -> int:
    return ny if side in (LEFT, RIGHT) else nx


class NativeLines:
    """Pack / unpack boundary lines with the C-ABI kernels (device fields)."""

    def __init__(self, stream=None):
        self.stream = stream

    def _sp(self):
        import torch
        s = self.stream if self.stream is not None else torch.cuda.current_stream()
        return s.cuda_stream

    def pack(self, st, side: int, buf):
        from .swdemo import _grid
        g = _grid(st.H)
        N.check(N.lib().fkc_halo_pack(ctypes.byref(g), st.H.ptr, st.U.ptr, st.V.ptr, side, buf.data_ptr(),
                                      self._sp()))

    def unpack(self, st, side: int, buf):
        from .swdemo import _grid
        g = _grid(st.H)
        N.check(N.lib().fkc_halo_unpack(ctypes.byref(g), st.H.ptr, st.U.ptr, st.V.ptr, side, buf.data_ptr(),
                                        self._sp()))


class TorchLines:
    """Pack / unpack with tensor slicing -- for CPU states in the gloo tests
    (state fields are (ny+2, nx+2) torch tensors or objects with ``.data``)."""

    @staticmethod
    def _arrays(st):
        return [getattr(f, "data", f) for f in (st.H, st.U, st.V)]

    def pack(self, st, side: int, buf):
        arrs = self._arrays(st)
        for k, a in enumerate(arrs):
            line = {LEFT: a[1:-1, 1], RIGHT: a[1:-1, -2], DOWN: a[1, 1:-1], UP: a[-2, 1:-1]}[side]
            n = line.shape[0]
            buf[k * n:(k + 1) * n].copy_(line)

    def unpack(self, st, side: int, buf):
        arrs = self._arrays(st)
        for k, a in enumerate(arrs):
            line = {LEFT: a[1:-1, 0], RIGHT: a[1:-1, -1], DOWN: a[0, 1:-1], UP: a[-1, 1:-1]}[side]
            n = line.shape[0]
            line.copy_(buf[k * n:(k + 1) * n])


# ---------------------------------------------------------------------------
# transports
# ---------------------------------------------------------------------------

class DistTransport:
    """Neighbour P2P over torch.distributed (NCCL across GPUs, gloo on CPU).
    All ops of one exchange go into one batch_isend_irecv group."""

    TAG = {RIGHT: 11, LEFT: 12, UP: 13, DOWN: 14}

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def exchange(self, sends: Dict[int, Tuple[int, object]], recvs: Dict[int, Tuple[int, object]]):
        """sends/recvs: side -> (peer rank, buffer).  A line sent towards
        `side` lands in the peer's halo on OPPOSITE[side]."""
        dist = self.dist
        ops = []
        for side in EXCHANGE_ORDER:
            if side in sends:
                peer, buf = sends[side]
                ops.append(dist.P2POp(dist.isend, buf, peer, self.group, self.TAG[side]))
            opp = OPPOSITE[side]
            if opp in recvs:      # the message travelling towards `side` arrives on our OPPOSITE side
                peer, buf = recvs[opp]
                ops.append(dist.P2POp(dist.irecv, buf, peer, self.group, self.TAG[side]))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()


class HaloExchanger:
    """Send the outermost interior lines of a state to the neighbours and
    fill its halo lines from theirs."""

    def __init__(self, grid: CartGrid, rank: int, transport, lines, device=None, dtype=None):
        import torch
        self.grid, self.rank, self.transport, self.lines = grid, rank, transport, lines
        t = grid.tile(rank)
        self.nbr = {s: grid.neighbor(rank, s) for s in (LEFT, RIGHT, DOWN, UP)}
        dtype = dtype or torch.float32
        self.send = {s: torch.empty(3 * _line_len(s, t.nx, t.ny), dtype=dtype, device=device)
                     for s, p in self.nbr.items() if p is not None}
        self.recv = {s: torch.empty_like(b) for s, b in self.send.items()}

    def exchange(self, st):
        for s in self.send:
            self.lines.pack(st, s, self.send[s])
        self.transport.exchange({s: (self.nbr[s], b) for s, b in self.send.items()},
                                {s: (self.nbr[s], b) for s, b in self.recv.items()})
        for s in self.recv:
            self.lines.unpack(st, s, self.recv[s])


class LocalTransport:
    """All sub-domains in one process: exchange = buffer copies."""

    def __init__(self, grid: CartGrid):
        self.grid = grid

    def exchange_all(self, exchangers: List[HaloExchanger], states):
        for ex, st in zip(exchangers, states):
            for s in ex.send:
                ex.lines.pack(st, s, ex.send[s])
        for ex in exchangers:
            for s, buf in ex.recv.items():
                src = exchangers[ex.nbr[s]]
                buf.copy_(src.send[OPPOSITE[s]])
        for ex, st in zip(exchangers, states):
            for s in ex.recv:
                ex.lines.unpack(st, s, ex.recv[s])


# ---------------------------------------------------------------------------
# fused exchange: the step kernel stores boundary lines into the neighbours'
# halos (peer memory) and orders steps with mailbox words -- no separate
# pack / transfer / unpack phase (include/fkc_sw.h fkc_peer_line, fkc_sync)
# ---------------------------------------------------------------------------

def set_peer_line(line: "N.PeerLine", side: int, ptrs: Sequence[int], pitch: int, nbr_nx: int, nbr_ny: int,
                  itemsize: int):
    """Fill `line` so that our boundary cells land in the halo of the
    neighbour across `side`, whose fields (element (0,0) at ptrs[f]) have row
    pitch `pitch` and interior nbr_nx x nbr_ny: our row 1 -> its row ny+1
    (down), row ny -> row 0 (up), column 1 -> column nx+1 (left), column
    nx -> column 0 (right)."""
    if side == DOWN:
        off, stride = (nbr_ny + 1) * pitch, 1
    elif side == UP:
        off, stride = 0, 1
    elif side == LEFT:
        off, stride = nbr_nx + 1, pitch
    else:
        off, stride = 0, pitch
    for f in range(3):
        line.p[f] = ptrs[f] + off * itemsize
    line.stride = stride


def _field_ptrs(st) -> Tuple[int, int, int]:
    return st.H.ptr, st.U.ptr, st.V.ptr


class Mailbox:
    """Per-tile sync words: [0..3] mailbox per side (written by that side's
    neighbour), [4..7] edge-writer counters (used by the kernel)."""

    def __init__(self, device):
        import torch
        self.buf = torch.zeros(8, dtype=torch.int32, device=device)

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr()

    def word(self, side: int) -> int:
        return self.ptr + 4 * side

    @property
    def counters(self) -> int:
        return self.ptr + 16


def fill_sync(sync: "N.Sync", mail: Mailbox, signal: Dict[int, int], epoch: int, pdl: bool = False):
    """wait on our own mailbox words, signal the neighbours' words for us;
    ``pdl``: every neighbour tile runs on another GPU (programmatic launch
    stays on with the fused exchange)."""
    for s in (LEFT, RIGHT, DOWN, UP):
        if s in signal:
            sync.wait[s] = mail.word(s)
            sync.signal[s] = signal[s]
        else:
            sync.wait[s] = None
            sync.signal[s] = None
    sync.counter = mail.counters
    sync.epoch = epoch & 0xFFFFFFFF
    sync.flags = N.SYNC_PDL if pdl else 0


def initial_peer_exchange(grid: CartGrid, rank: int, st, lines: Dict[int, "N.PeerLine"], stream=None):
    """One-time fill of the neighbours' halos of their INITIAL buffers from
    our initial boundary lines (pitched DMA through peer memory, fkc_copy2d)."""
    import torch
    t = grid.tile(rank)
    it = st.H.storage.element_size()
    sp = (stream if stream is not None else torch.cuda.current_stream()).cuda_stream
    L = N.lib()
    for side, line in lines.items():
        for f, fld in enumerate((st.H, st.U, st.V)):
            p = fld.pitch
            if side in (DOWN, UP):
                y = 1 if side == DOWN else t.ny
                src = fld.ptr + (y * p + 1) * it
                N.check(L.fkc_copy2d(line.p[f] + it, t.nx * it, src, t.nx * it, t.nx * it, 1, sp))
            else:
                x = 1 if side == LEFT else t.nx
                src = fld.ptr + (p + x) * it
                N.check(L.fkc_copy2d(line.p[f] + line.stride * it, line.stride * it, src, p * it, it, t.ny, sp))


class PeerSetupError(RuntimeError):
    """CUDA-IPC peer setup failed on some rank (raised on every rank)."""


class PeerExchange:
    """Fused exchange between the processes of a decomposed run (one per
    GPU): every rank exports its two state buffers (H,U,V of each parity) and
    its mailbox with CUDA IPC, opens its neighbours' (NVLink / NVSwitch peer
    memory), and from then on the step kernel itself writes the neighbours'
    halos and signals their mailboxes."""

    def __init__(self, grid: CartGrid, rank: int, bufs, group=None):
        import torch.distributed as dist
        self.grid, self.rank = grid, rank
        dev = bufs[0].H.storage.device
        self.mail = Mailbox(dev)
        self._opened: Dict[bytes, int] = {}
        world = dist.get_world_size(group)
        # every failure is agreed on collectively, so all ranks raise together
        # (PeerSetupError) and a caller can fall back to another transport
        # the CFL board of the decomposed SPEC run (include/fkc_sw.h fkc_sync):
        # [2 parities][world] entries of {bound bits, tag}, written by every rank
        import torch
        self.world = world
        self.board = torch.zeros(4 * world, dtype=torch.int64, device=dev)
        self.board_count = torch.zeros(1, dtype=torch.int32, device=dev)
        try:
            uuid = str(torch.cuda.get_device_properties(dev).uuid)
        except Exception:  # noqa: BLE001 - older torch: treat as shared (no PDL)
            uuid = None
        try:
            mine, err = {"bufs": [[N.ipc_export(p) for p in _field_ptrs(b)] for b in bufs],
                         "mail": N.ipc_export(self.mail.ptr), "board": N.ipc_export(self.board.data_ptr()),
                         "uuid": uuid,
                         "pitch": bufs[0].H.pitch, "itemsize": bufs[0].H.storage.element_size()}, None
        except Exception as e:  # noqa: BLE001 - reported collectively
            mine, err = None, f"rank {rank} export: {e}"
        everyone = [None] * world
        dist.all_gather_object(everyone, {"info": mine, "err": err}, group=group)
        errs = [e["err"] for e in everyone if e["err"]]
        if errs:
            raise PeerSetupError("; ".join(errs))
        self.nbr = {s: grid.neighbor(rank, s) for s in (LEFT, RIGHT, DOWN, UP)}
        self.nbr = {s: n for s, n in self.nbr.items() if n is not None}
        # lines[p][side]: targets for a step whose OUTPUT parity is p
        self.lines = [{}, {}]
        self.signal: Dict[int, int] = {}
        err = None
        try:
            for s, n in self.nbr.items():
                info = everyone[n]["info"]
                nt = grid.tile(n)
                for p in (0, 1):
                    ptrs = [self._open(h) + off for h, off in info["bufs"][p]]
                    line = N.PeerLine()
                    set_peer_line(line, s, ptrs, info["pitch"], nt.nx, nt.ny, info["itemsize"])
                    self.lines[p][s] = line
                h, off = info["mail"]
                self.signal[s] = self._open(h) + off + 4 * OPPOSITE[s]
            # every rank's board (own: local memory)
            self.boards = []
            for r in range(world):
                if r == rank:
                    self.boards.append(self.board.data_ptr())
                else:
                    h, off = everyone[r]["info"]["board"]
                    self.boards.append(self._open(h) + off)
        except Exception as e:  # noqa: BLE001 - reported collectively
            err = f"rank {rank} open: {e}"
        # programmatic launch with the fused exchange only if no neighbour
        # tile shares this GPU
        my_uuid = everyone[rank]["info"]["uuid"]
        self.pdl = my_uuid is not None and all(everyone[n]["info"]["uuid"] not in (None, my_uuid)
                                               for n in self.nbr.values())
        errs = [None] * world
        dist.all_gather_object(errs, err, group=group)
        errs = [e for e in errs if e]
        if errs:
            self.close()
            raise PeerSetupError("; ".join(errs))

    def _open(self, handle: bytes) -> int:
        if handle not in self._opened:
            self._opened[handle] = N.ipc_open(handle)
        return self._opened[handle]

    def fill_board(self, sync: "N.Sync", rank: int):
        """The CFL board fields of fkc_sync (global CFL minimum without a
        collective)."""
        if self.world > N.MAX_RANKS:
            raise ValueError(f"the CFL board serves up to {N.MAX_RANKS} ranks")
        sync.cfl_board = self.board.data_ptr()
        for r, p in enumerate(self.boards):
            sync.cfl_peers[r] = p
        sync.cfl_counter = self.board_count.data_ptr()
        sync.cfl_rank = rank
        sync.cfl_nranks = self.world

    def close(self):
        for base in self._opened.values():
            N.ipc_close(base)
        self._opened.clear()


# ---------------------------------------------------------------------------
# initial state of a tile (same f64 formula as swdemo.init_state)
# ---------------------------------------------------------------------------

def gaussian_tile(grid: CartGrid, rank: int, precision="f32", dx=1.0, dy=1.0, base=1.0, amplitude=0.4,
                  center=None, width=None) -> np.ndarray:
    """Interior (ny, nx) of the global Gaussian hump restricted to the tile,
    evaluated exactly as swdemo.init_state / oracle.init_state do."""
    t = grid.tile(rank)
    NX, NY = grid.NX, grid.NY
    cx, cy = center if center is not None else (NX * dx / 2.0, NY * dy / 2.0)
    w = width if width is not None else NX * dx / 8.0
    xc = (np.arange(t.x0, t.x0 + t.nx, dtype=np.float64) + 0.5) * dx - cx
    yc = (np.arange(t.y0, t.y0 + t.ny, dtype=np.float64) + 0.5) * dy - cy
    h = base + amplitude * np.exp(-(xc[None, :] ** 2 + yc[:, None] ** 2) / (w * w))
    return h.astype({"f32": np.float32, "f64": np.float64}[precision])


# ---------------------------------------------------------------------------
# distributed simulation (one process per GPU)
# ---------------------------------------------------------------------------

class DistributedSimulation:
    """One rank's tile of a decomposed run: step kernel with per-side BC and
    the halo exchange (fused peer stores, or NCCL), double-buffer swap.

    ``cfg.dt`` fixed: the weak-scaling benchmark.  ``cfg.dt is None``: the
    SPEC ``run`` across GPUs -- every step's fused
    reduction produces this tile's CFL bound; with ``cfl_exchange="board"``
    (default with the peer transport) the last warp of the step kernel
    writes it into every rank's board (NVLink peer stores) and the next step
    kernel takes the minimum of the board entries on the device -- no
    collective, no extra launch; ``"allreduce"``: one 8-byte all-reduce (MIN,
    stream-ordered) into a device slot per step.  ``diagnostics=True`` (implied by CFL mode) also keeps the per-step
    mass / maxima / error words; :meth:`rows` combines them over the ranks.
    """

    def __init__(self, cfg, grid: CartGrid, rank: int, device=None, group=None, stream=None,
                 transport: str = "peer", state=None, diagnostics: bool = False, capacity=None,
                 cfl_exchange: str = "auto"):
        import torch
        import torch.distributed as dist
        from . import swdemo
        from .field import Field
        if transport not in ("peer", "nccl", "auto"):
            raise ValueError(f"unknown transport {transport!r}")
        if cfl_exchange not in ("auto", "board", "allreduce"):
            raise ValueError(f"unknown cfl_exchange {cfl_exchange!r}")
        self.fallback_reason = None
        self.transport = transport
        self.cfg, self.grid, self.rank = cfg, grid, rank
        self.tile = grid.tile(rank)
        self.bc = grid.local_bc(rank)
        self.stream = stream
        t = self.tile
        full = Extent(t.nx + 2, t.ny + 2)
        if state is None:       # the tile of swdemo.init_state's Gaussian hump
            h = gaussian_tile(grid, rank, cfg.precision, cfg.dx, cfg.dy, cfg.base, cfg.amplitude, cfg.center,
                              cfg.width)
            H = Field.zeros(full, cfg.precision)
            H.data[1:-1, 1:-1] = h
            state = swdemo.SWState(H, Field.zeros(full, cfg.precision), Field.zeros(full, cfg.precision),
                                   cfg.g, cfg.dx, cfg.dy)
        elif tuple(state.full) != tuple(full):
            raise ValueError(f"state extent {tuple(state.full)} != tile extent {tuple(full)}")
        st = state.to_device(device)
        self.a = st
        self.b = swdemo.SWState(st.H.empty_like(), st.U.empty_like(), st.V.empty_like(), st.g, st.dx, st.dy)
        tdt = torch.float32 if cfg.precision == "f32" else torch.float64
        swdemo.apply_boundary(self.a, self.bc, stream)
        self.n = 0
        self.ex = self.peer = None
        if transport == "nccl":
            self.ex = HaloExchanger(grid, rank, DistTransport(group), NativeLines(stream), st.H.storage.device,
                                    tdt)
            self.ex.exchange(self.a)
        else:
            try:
                self.peer = PeerExchange(grid, rank, (self.a, self.b), group)
            except PeerSetupError as e:
                if transport == "peer":
                    raise
                # auto: every rank got the same error -> all fall back together
                self.transport, self.fallback_reason = "nccl", str(e)
                self.ex = HaloExchanger(grid, rank, DistTransport(group), NativeLines(stream),
                                        st.H.storage.device, tdt)
                self.ex.exchange(self.a)
        if self.peer is not None:
            self.transport = "peer"
            initial_peer_exchange(grid, rank, self.a, self.peer.lines[0], stream)
            (stream or torch.cuda.current_stream()).synchronize()
            dist.barrier(group)
        self._group = group
        self.cfl = cfg.dt is None
        # per-step global CFL minimum: through the rank boards inside the step
        # kernels (peer transport, <= 8 ranks), else a stream-ordered all-reduce
        board_ok = self.peer is not None and dist.get_world_size(group) <= N.MAX_RANKS
        if cfl_exchange == "board" and not board_ok:
            raise ValueError("cfl_exchange='board' needs the peer transport and <= 8 ranks")
        self.cfl_exchange = "board" if (cfl_exchange != "allreduce" and board_ok) else "allreduce"
        self.diag = diagnostics or self.cfl
        self.slots = None
        if self.diag:
            cap = (capacity if capacity is not None else cfg.steps) + 1
            self.slots = swdemo.ReductionSlots(cap, st.H.storage.device)
            red = self.slots.reduce_struct(0)
            g = swdemo._grid(st.H)
            with torch.cuda.stream(stream or torch.cuda.current_stream()):
                N.check(N.lib().fkc_sw_reduce_state(ctypes.byref(g), st.H.ptr, st.U.ptr, st.V.ptr, st.dx, st.dy,
                                                    st.g, ctypes.byref(red), swdemo._stream_ptr(stream)))
                if self.cfl:
                    self._allreduce_bound(0)

    def _allreduce_bound(self, row: int):
        """Global CFL bound of state `row`: MIN over the ranks of the tiles'
        bounds (positive doubles stored as int64 bits: integer order = value
        order), in place in the device slot."""
        import torch.distributed as dist
        slot = self.slots.buf[row, 3:4]
        if dist.get_backend(self._group) == "nccl":
            dist.all_reduce(slot, op=dist.ReduceOp.MIN, group=self._group)      # stream-ordered on the device
        else:                                                                    # gloo (tests): via the host
            h = slot.cpu()
            dist.all_reduce(h, op=dist.ReduceOp.MIN, group=self._group)
            slot.copy_(h)

    def _launches_per_step(self) -> int:
        return 1 if self.transport == "peer" else 1 + 2 * len(self.ex.send)

    def advance(self, steps: int):
        import torch
        from . import swdemo
        L = N.lib()
        sp = swdemo._stream_ptr(self.stream)
        cfg = self.cfg
        if self.diag and self.n + steps >= self.slots.n:
            raise ValueError("reduction slot capacity exceeded")
        with torch.cuda.stream(self.stream or torch.cuda.current_stream()):
            for _ in range(steps):
                src, dst = (self.a, self.b) if self.n % 2 == 0 else (self.b, self.a)
                red = self.slots.reduce_struct(self.n + 1, cfl=self.cfl) if self.diag else None
                bound = self.slots.addr(self.n, 3) if self.cfl else None
                a = swdemo._step_args(src, dst, cfg.dt if cfg.dt is not None else 0.0, self.bc, cfg.mode,
                                      cfg.variant, red, bound, cfg.cfl_factor)
                a.tune.parity = self.n & 1          # alternating segment order (L2 reuse)
                if self.transport == "peer":
                    out_parity = (self.n + 1) % 2
                    for s, line in self.peer.lines[out_parity].items():
                        a.peer[s] = line
                    fill_sync(a.sync, self.peer.mail, self.peer.signal, self.n, pdl=self.peer.pdl)
                    if self.cfl and self.cfl_exchange == "board":
                        self.peer.fill_board(a.sync, self.rank)
                    N.check(L.fkc_sw_step(ctypes.byref(a), sp))
                else:
                    N.check(L.fkc_sw_step(ctypes.byref(a), sp))
                    self.ex.exchange(dst)
                if cfg.dt is not None:
                    dst.t = src.t + float(cfg.dt)
                self.n += 1
                if self.cfl and self.cfl_exchange == "allreduce":
                    self._allreduce_bound(self.n)
        return self

    def rows(self):
        """Global diagnostics rows (step, t, dt, mass, max_hu, max_hv) of the
        steps so far (collective: sums the tiles' masses, maxima over ranks,
        error words OR-ed); raises the reference's errors like swdemo.run."""
        import torch
        import torch.distributed as dist
        from . import swdemo
        if not self.diag:
            return []
        (self.stream or torch.cuda.current_stream()).synchronize()
        d = swdemo.ReductionSlots.decode(self.slots.buf[: self.n + 1].cpu().numpy())
        mass = torch.tensor(d["mass"], dtype=torch.float64)
        mx = torch.tensor(np.stack([d["max_hu"], d["max_hv"]]), dtype=torch.float64)
        e = d["err"].astype(np.int64)
        err = torch.tensor(np.stack([e & 1, (e >> 1) & 1, (e >> 2) & 1]))   # OR of bits = MAX per bit
        dev = self.slots.buf.device if dist.get_backend(self._group) == "nccl" else "cpu"
        mass, mx, err = mass.to(dev), mx.to(dev), err.to(dev)
        # the tiles' CFL bounds (bits of positive doubles: integer MIN = value
        # MIN); with the board exchange each slot holds only its tile's bound
        cb = torch.tensor(self.slots.buf[: self.n + 1, 3].cpu().numpy()).to(dev)
        dist.all_reduce(cb, op=dist.ReduceOp.MIN, group=self._group)
        d["cfl_min"] = cb.cpu().numpy().view(np.float64)
        dist.all_reduce(mass, op=dist.ReduceOp.SUM, group=self._group)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=self._group)
        dist.all_reduce(err, op=dist.ReduceOp.MAX, group=self._group)
        mass, mx = mass.cpu().numpy(), mx.cpu().numpy()
        eb = err.cpu().numpy()
        err = eb[0] | (eb[1] << 1) | (eb[2] << 2)
        cfg = self.cfg
        f = np.float32 if cfg.precision == "f32" else np.float64
        out, t = [], 0.0
        if err[0]:
            swdemo.raise_for_error(int(err[0]), "in the initial state")
        for k in range(self.n):
            if err[k + 1]:
                swdemo.raise_for_error(int(err[k + 1]), f"at step {k + 1}")
            dt = float(cfg.dt) if cfg.dt is not None else float(f(cfg.cfl_factor) * f(d["cfl_min"][k]))
            t += dt
            out.append((k + 1, t, dt, float(mass[k + 1]) * cfg.dx * cfg.dy, float(mx[0, k + 1]),
                        float(mx[1, k + 1])))
        return out

    def close(self):
        """Drain, then unmap the neighbours' memory (collective)."""
        import torch
        import torch.distributed as dist
        torch.cuda.synchronize()
        dist.barrier(self._group)
        if self.peer is not None:
            self.peer.close()
            self.peer = None
        dist.barrier(self._group)

    def state(self):
        return self.a if self.n % 2 == 0 else self.b


def run_local_decomposed(cfg, px: int, py: int, steps: int, device=None, exchange: str = "pack",
                         concurrent: bool = False, warmup: int = 0, timing: Optional[list] = None):
    """All px*py tiles in one process on one device: the GPU-side validation
    of the decomposed path.  Returns (grid, the tiles' states).

    exchange="pack": step kernel, then native line pack / copy / unpack
    (LocalTransport).  exchange="fused": the step kernel writes the
    neighbours' halos itself (peer lines into the other tiles' buffers); with
    concurrent=True every tile runs on its own stream and steps are ordered
    only by the in-kernel mailbox protocol -- the multi-GPU synchronisation,
    exercised on one device."""
    import torch
    from . import swdemo
    from .field import Field
    if exchange not in ("pack", "fused"):
        raise ValueError(f"unknown exchange {exchange!r}")
    grid = CartGrid(px, py, cfg.nx, cfg.ny, cfg.boundary)
    bufs = []        # bufs[r] = (parity-0 state, parity-1 state)
    for r in range(grid.size):
        t = grid.tile(r)
        full = Extent(t.nx + 2, t.ny + 2)
        H = Field.zeros(full, cfg.precision)
        H.data[1:-1, 1:-1] = gaussian_tile(grid, r, cfg.precision, cfg.dx, cfg.dy, cfg.base, cfg.amplitude,
                                           cfg.center, cfg.width)
        st = swdemo.SWState(H, Field.zeros(full, cfg.precision), Field.zeros(full, cfg.precision),
                            cfg.g, cfg.dx, cfg.dy).to_device(device)
        swdemo.apply_boundary(st, grid.local_bc(r))
        bufs.append((st, swdemo.SWState(st.H.empty_like(), st.U.empty_like(), st.V.empty_like(), st.g, st.dx,
                                        st.dy)))
    tdt = torch.float32 if cfg.precision == "f32" else torch.float64
    if exchange == "pack":
        states, others = [b[0] for b in bufs], [b[1] for b in bufs]
        exs = [HaloExchanger(grid, r, None, NativeLines(), states[r].H.storage.device, tdt)
               for r in range(grid.size)]
        lt = LocalTransport(grid)
        lt.exchange_all(exs, states)
        ev = None
        for k in range(warmup + steps):
            if k == warmup and timing is not None:
                torch.cuda.synchronize()
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                ev[0].record()
            for r in range(grid.size):
                swdemo.advance(states[r], cfg.dt, grid.local_bc(r), cfg.mode, cfg.variant, out=others[r])
            states, others = others, states
            lt.exchange_all(exs, states)
        if ev is not None:
            ev[1].record()
            torch.cuda.synchronize()
            timing.append(ev[0].elapsed_time(ev[1]))
        return grid, states

    dev = bufs[0][0].H.storage.device
    lines = []       # lines[r][p][side]
    for r in range(grid.size):
        per = [{}, {}]
        for s in (LEFT, RIGHT, DOWN, UP):
            n = grid.neighbor(r, s)
            if n is None:
                continue
            nt = grid.tile(n)
            for p in (0, 1):
                nb = bufs[n][p]
                line = N.PeerLine()
                set_peer_line(line, s, _field_ptrs(nb), nb.H.pitch, nt.nx, nt.ny, nb.H.storage.element_size())
                per[p][s] = line
        lines.append(per)
    for r in range(grid.size):
        initial_peer_exchange(grid, r, bufs[r][0], lines[r][0])
    torch.cuda.synchronize()
    mails = [Mailbox(dev) for _ in range(grid.size)] if concurrent else None
    streams = [torch.cuda.Stream(dev) for _ in range(grid.size)] if concurrent else None
    L = N.lib()
    ev = None
    for k in range(warmup + steps):
        if k == warmup and timing is not None:     # time the last `steps` steps: all tiles, all streams
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(1 + grid.size)]
            ev[0].record()
            if concurrent:
                for st in streams:
                    st.wait_event(ev[0])
        for r in range(grid.size):
            src, dst = bufs[r][k % 2], bufs[r][(k + 1) % 2]
            a = swdemo._step_args(src, dst, cfg.dt, grid.local_bc(r), cfg.mode, cfg.variant)
            a.tune.parity = k & 1
            for s, line in lines[r][(k + 1) % 2].items():
                a.peer[s] = line
            if concurrent:
                sig = {s: mails[grid.neighbor(r, s)].word(OPPOSITE[s]) for s in lines[r][0]}
                fill_sync(a.sync, mails[r], sig, k)
                sp = streams[r].cuda_stream
            else:
                sp = torch.cuda.current_stream(dev).cuda_stream
            N.check(L.fkc_sw_step(ctypes.byref(a), sp))
    if ev is not None:
        cur = torch.cuda.current_stream(dev)
        for r in range(grid.size):
            ev[1 + r].record(streams[r] if concurrent else cur)
        torch.cuda.synchronize()
        timing.append(max(ev[0].elapsed_time(e) for e in ev[1:]))
    torch.cuda.synchronize()
    return grid, [b[(warmup + steps) % 2] for b in bufs]


def gather_interior(grid: CartGrid, tiles: Sequence[np.ndarray]) -> np.ndarray:
    """Assemble per-rank interiors (ny, nx) into the global interior."""
    out = np.empty((grid.NY, grid.NX), dtype=tiles[0].dtype)
    for r, a in enumerate(tiles):
        t = grid.tile(r)
        out[t.y0:t.y0 + t.ny, t.x0:t.x0 + t.nx] = a
    return out
