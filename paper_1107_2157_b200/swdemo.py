"""Shallow-water driver API on the B200 -- a drop-in for the reference's
``swdemo`` module (specified in SPEC.md:472-569, absent from the shipped
package).

Same names and meaning as the reference: :class:`SWConfig`,
:class:`SWState`, :func:`init_state`, :func:`apply_boundary`,
:func:`stable_dt`, :func:`step_native` / :func:`advance`, :func:`run`,
:func:`total_mass`, and the errors :class:`NonPositiveDepth` /
:class:`NonfiniteValue`.  The engine selector of ``run``
gains the engine ``"cuda"``; it is the only engine this package ships --
the reference's CPU engines (``native``/``ref``/``sim``) are not
re-implemented here, and nothing in this module computes a step on the CPU.

Every numeric operation on a state runs through the C-ABI library
(``_native``): the fused Lax-Wendroff step kernel (which also fills the
output halo, i.e. ``apply_boundary`` of the new state, and can reduce
CFL bound / mass / maxima of the new state in the same pass), the boundary
kernel and the reduction kernel.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field as dc_field
from typing import List, Optional, Sequence, Tuple, Union

import numpy as np

from . import _native as N
from .field import DeviceField, Field, dtype_of
from .region import Extent

BC_CODES = {"reflective": N.BC_REFLECTIVE, "periodic": N.BC_PERIODIC, "none": N.BC_NONE}
MODES = {"exact": N.MODE_EXACT, "fast": N.MODE_FAST}
VARIANTS = {"auto": N.VARIANT_AUTO, "generic": N.VARIANT_GENERIC, "tma": N.VARIANT_TMA,
            "resident": N.VARIANT_RESIDENT, "loop": N.VARIANT_LOOP}
ENGINES = ("cuda",)


class NonPositiveDepth(ValueError):
    """h <= 0."""


class NonfiniteValue(ArithmeticError):
    """NaN/Inf in the state."""


class LaunchError(N.FkcUsageError):
    """Invalid launch configuration: raised for every
    usage error the C-ABI reports (FKC_EUSAGE -- bad extent, pitch,
    alignment, enum, aliasing), before any device memory is touched.  A
    ``ValueError``, like the reference's."""

    def __init__(self, code_or_msg, msg=None):
        if msg is None:
            code_or_msg, msg = N.FKC_EUSAGE, str(code_or_msg)
        super().__init__(code_or_msg, msg)


@dataclass
class SWConfig:
    """SPEC.md:483-488 fields, plus the B200 engine knobs.

    ``dt=None`` recomputes ``dt = stable_dt(state)`` every step (on device,
    fused into the previous step); a number fixes dt.
    """

    nx: int = 64
    ny: int = 64
    dx: float = 1.0
    dy: float = 1.0
    g: float = 9.8
    cfl_factor: float = 0.9
    steps: int = 100
    boundary: str = "reflective"
    base: float = 1.0
    amplitude: float = 0.4
    center: Optional[Tuple[float, float]] = None
    width: Optional[float] = None
    precision: str = "f32"
    group: Tuple[int, int] = (16, 8)
    dt: Optional[float] = None
    mode: str = "exact"
    variant: str = "auto"

    def __post_init__(self):
        if not (0 < self.cfl_factor <= 1):
            raise ValueError("cfl_factor must be in (0, 1]")
        if self.boundary not in ("reflective", "periodic"):
            raise ValueError(f"unknown boundary {self.boundary!r}")
        if self.mode not in MODES:
            raise ValueError(f"unknown mode {self.mode!r}")
        dtype_of(self.precision)
        Extent(self.nx, self.ny)

    @property
    def interior(self) -> Extent:
        return Extent(self.nx, self.ny)


AnyField = Union[Field, DeviceField]


@dataclass
class SWState:
    """H (h), U (hu), V (hv) sharing one full extent, halo [1,1,1,1]."""

    H: AnyField
    U: AnyField
    V: AnyField
    g: float = 9.8
    dx: float = 1.0
    dy: float = 1.0
    t: float = 0.0

    @property
    def on_device(self) -> bool:
        return isinstance(self.H, DeviceField)

    @property
    def full(self) -> Extent:
        return self.H.full

    @property
    def precision(self) -> str:
        return self.H.precision

    def to_device(self, device=None) -> "SWState":
        if self.on_device:
            return self
        return SWState(*(DeviceField.from_field(f, device) for f in (self.H, self.U, self.V)),
                       self.g, self.dx, self.dy, self.t)

    def to_host(self, out: Optional["SWState"] = None, like: Optional["SWState"] = None) -> "SWState":
        """Device -> host Fields (into `out`'s arrays when given, e.g. pinned).
        With ``like`` (a host state), the new Fields are of ``like``'s Field
        class -- e.g. the reference's own ``fkc.field.Field`` -- so a caller
        of the reference API gets its own types back."""
        if not self.on_device:
            return self
        if out is not None:
            for name in ("H", "U", "V"):
                getattr(self, name).to_field(getattr(out, name))
            out.g, out.dx, out.dy, out.t = self.g, self.dx, self.dy, self.t
            return out
        if like is not None and not isinstance(like.H, Field):
            mk = lambda dev, tmpl: type(tmpl)(tmpl.full, dev.to_numpy(), dev.precision)  # noqa: E731
            return SWState(mk(self.H, like.H), mk(self.U, like.U), mk(self.V, like.V),
                           self.g, self.dx, self.dy, self.t)
        return SWState(self.H.to_field(), self.U.to_field(), self.V.to_field(),
                       self.g, self.dx, self.dy, self.t)


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------

def _torch():
    import torch
    return torch


def _stream_ptr(stream=None) -> int:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _grid(f: DeviceField) -> N.Grid:
    return N.Grid(f.full.nx - 2, f.full.ny - 2, f.pitch, f.dtype_code, 0)


def _bc4(boundary: Union[str, Sequence[str]]) -> Tuple[int, int, int, int]:
    if isinstance(boundary, str):
        return (BC_CODES[boundary],) * 4
    return tuple(BC_CODES[b] for b in boundary)


def _as_device(state: SWState) -> SWState:
    if not state.on_device:
        return state.to_device()
    return state


class ReductionSlots:
    """Device slots for the fused reductions: one row of 5 x 64-bit words
    per state: [mass (f64), max|hu| (f64 bits), max|hv| (f64 bits),
    min CFL bound (f64 bits), error word]."""

    INF_BITS = 0x7FF0000000000000

    def __init__(self, n: int, device):
        torch = _torch()
        self.n = n
        self.buf = torch.zeros((n, 5), dtype=torch.int64, device=device)
        self.template = torch.tensor([0, 0, 0, self.INF_BITS, 0], dtype=torch.int64, device=device)
        self.reset()

    def reset(self, lo: int = 0, hi: Optional[int] = None):
        hi = self.n if hi is None else hi
        self.buf[lo:hi].copy_(self.template.expand(hi - lo, 5))

    def addr(self, i: int, k: int) -> int:
        return self.buf.data_ptr() + (i * 5 + k) * 8

    def reduce_struct(self, i: int, mass=True, maxima=True, cfl=True, err=True) -> N.Reduce:
        return N.Reduce(self.addr(i, 0) if mass else None,
                        self.addr(i, 1) if maxima else None,
                        self.addr(i, 2) if maxima else None,
                        self.addr(i, 3) if cfl else None,
                        self.addr(i, 4) if err else None)

    @staticmethod
    def decode(rows_i64: np.ndarray):
        r = np.ascontiguousarray(rows_i64)
        as_f = r.view(np.float64)
        return {"mass": as_f[:, 0].copy(), "max_hu": as_f[:, 1].copy(), "max_hv": as_f[:, 2].copy(),
                "cfl_min": as_f[:, 3].copy(), "err": r[:, 4].astype(np.uint32)}


def raise_for_error(err_word: int, where: str = ""):
    if err_word & N.ERR_WATCHDOG:
        raise RuntimeError(f"device watchdog fired {where}")
    if err_word & N.ERR_NONFINITE:
        raise NonfiniteValue(f"non-finite state {where}")
    if err_word & N.ERR_NONPOSITIVE_FACE:
        raise NonPositiveDepth(f"face depth <= 0 {where}")
    if err_word & N.ERR_NONPOSITIVE_DEPTH:
        raise NonPositiveDepth(f"depth <= 0 {where}")


# ---------------------------------------------------------------------------
# reference API
# ---------------------------------------------------------------------------

def init_state(cfg: SWConfig, device=None) -> SWState:
    """Gaussian hump ``h = base + amp*exp(-r^2/width^2)`` at cell centres,
    hu = hv = 0, evaluated in f64 and rounded to the
    precision, uploaded, halos filled on device.  ``device=None`` keeps
    the state on the current CUDA device."""
    nx, ny = cfg.nx, cfg.ny
    cx, cy = cfg.center if cfg.center is not None else (nx * cfg.dx / 2.0, ny * cfg.dy / 2.0)
    w = cfg.width if cfg.width is not None else nx * cfg.dx / 8.0
    xc = (np.arange(nx, dtype=np.float64) + 0.5) * cfg.dx - cx
    yc = (np.arange(ny, dtype=np.float64) + 0.5) * cfg.dy - cy
    h = cfg.base + cfg.amplitude * np.exp(-(xc[None, :] ** 2 + yc[:, None] ** 2) / (w * w))
    full = Extent(nx + 2, ny + 2)
    dt_ = dtype_of(cfg.precision)
    H = Field.zeros(full, cfg.precision)
    H.data[1:-1, 1:-1] = h.astype(dt_)
    st = SWState(H, Field.zeros(full, cfg.precision), Field.zeros(full, cfg.precision),
                 cfg.g, cfg.dx, cfg.dy, 0.0).to_device(device)
    apply_boundary(st, cfg.boundary)
    return st


def apply_boundary(state: SWState, mode: Union[str, Sequence[str]] = "reflective", stream=None) -> SWState:
    """Fill the one-cell halo in place, on device."""
    if not state.on_device:
        dev = _as_device(state)
        apply_boundary(dev, mode, stream)
        for name in ("H", "U", "V"):
            getattr(state, name).data[...] = getattr(dev, name).to_numpy()
        return state
    g = _grid(state.H)
    bc = N.bc_array(_bc4(mode))
    N.check(N.lib().fkc_sw_apply_boundary(ctypes.byref(g), state.H.ptr, state.U.ptr, state.V.ptr, bc,
                                          _stream_ptr(stream)))
    return state


def reduce_state(state: SWState, stream=None) -> dict:
    """mass, max|hu|, max|hv|, min CFL bound and error word of a state
    (one fused device reduction)."""
    st = _as_device(state)
    slots = ReductionSlots(1, st.H.storage.device)
    red = slots.reduce_struct(0)
    g = _grid(st.H)
    N.check(N.lib().fkc_sw_reduce_state(ctypes.byref(g), st.H.ptr, st.U.ptr, st.V.ptr, st.dx, st.dy, st.g,
                                        ctypes.byref(red), _stream_ptr(stream)))
    d = ReductionSlots.decode(slots.buf.cpu().numpy())
    return {k: v[0] for k, v in d.items()}


def stable_dt(state: SWState, cfl_factor: float = 1.0) -> float:
    """dt = cfl * min over interior of min(dx,dy)/(sqrt(g h) + max(|hu|,|hv|)/h)
    (SPEC.md:508-516), computed in field precision on device."""
    r = reduce_state(state)
    raise_for_error(int(r["err"]), "in stable_dt")
    f = dtype_of(state.precision).type
    return float(f(cfl_factor) * f(r["cfl_min"]))


def total_mass(state: SWState) -> float:
    """Sum of interior h * dx * dy."""
    return float(reduce_state(state)["mass"]) * state.dx * state.dy


def _step_args(src: SWState, dst: SWState, dt: float, boundary, mode: str, variant: str,
               red: Optional[N.Reduce] = None, dt_bound: Optional[int] = None, cfl: float = 1.0,
               tune: Optional[N.Tune] = None) -> N.StepArgs:
    a = N.StepArgs()
    a.grid = _grid(src.H)
    a.H, a.U, a.V = src.H.ptr, src.U.ptr, src.V.ptr
    a.oH, a.oU, a.oV = dst.H.ptr, dst.U.ptr, dst.V.ptr
    a.dx, a.dy, a.dt, a.g = src.dx, src.dy, float(dt), src.g
    a.dt_bound = dt_bound
    a.cfl = cfl
    a.bc = N.bc_array(_bc4(boundary))
    a.mode = MODES[mode]
    a.variant = VARIANTS[variant]
    if red is not None:
        a.red = red
    if tune is not None:
        a.tune = tune
    return a


def advance(state: SWState, dt: float, boundary="reflective", mode: str = "exact",
            variant: str = "auto", out: Optional[SWState] = None, stream=None,
            tune: Optional[N.Tune] = None, check: bool = False) -> SWState:
    """Engine contract ``advance(state, dt) -> state``: one
    Lax-Wendroff step into fresh (or given) buffers; the input state is never
    mutated.  The output halo is filled per ``boundary``
    in the same kernel (== apply_boundary of the new state).

    ``check=True`` adds step_native's domain check: the input
    depths are reduced on device and the step kernel reports its half-step
    face depths; :class:`NonPositiveDepth` is raised if any face or input
    cell depth is <= 0 (one synchronisation).  ``tune`` is the per-call
    launch schedule (``_native.Tune``; results never depend on it)."""
    host = not state.on_device
    src = _as_device(state)
    if out is None:
        out = SWState(src.H.empty_like(), src.U.empty_like(), src.V.empty_like(), src.g, src.dx, src.dy, src.t)
    slots = None
    red = None
    if check:
        slots = ReductionSlots(2, src.H.storage.device)
        g = _grid(src.H)
        red0 = slots.reduce_struct(0, mass=False, maxima=False, cfl=False)
        N.check(N.lib().fkc_sw_reduce_state(ctypes.byref(g), src.H.ptr, src.U.ptr, src.V.ptr, src.dx, src.dy,
                                            src.g, ctypes.byref(red0), _stream_ptr(stream)))
        red = slots.reduce_struct(1, mass=False, maxima=False, cfl=False)
    a = _step_args(src, out, dt, boundary, mode, variant, red=red, tune=tune)
    N.check(N.lib().fkc_sw_step(ctypes.byref(a), _stream_ptr(stream)))
    if slots is not None:
        err = ReductionSlots.decode(slots.buf.cpu().numpy())["err"]
        if (err[0] & N.ERR_NONPOSITIVE_DEPTH) or (err[1] & N.ERR_NONPOSITIVE_FACE):
            raise NonPositiveDepth("face or cell depth <= 0")
    out.t = src.t + float(dt)
    return out.to_host(like=state) if host else out


def step_native(state: SWState, dt: float, boundary="reflective", mode: str = "exact") -> SWState:
    """Name-compatible alias of the reference's ``step_native``
    -- executed by the CUDA kernel, with its NonPositiveDepth check
    (SPEC.md:524)."""
    return advance(state, dt, boundary, mode, check=True)


# ---------------------------------------------------------------------------
# device-resident time loop
# ---------------------------------------------------------------------------

@dataclass
class RunResult:
    rows: List[Tuple[int, float, float, float, float, float]]  # step,t,dt,mass,max_hu,max_hv
    state: SWState
    dts: np.ndarray = dc_field(default_factory=lambda: np.zeros(0))


class Simulation:
    """Double-buffered device state + per-step fused reductions.

    ``advance(n)`` enqueues n steps on the stream without any host
    synchronisation: with ``cfg.dt is None`` each step reads its dt bound
    from the reduction slot the previous step (or the initial reduction)
    wrote, exactly like ``run`` recomputes ``stable_dt`` every step
    (SPEC.md:529-537).
    """

    def __init__(self, cfg: SWConfig, state: Optional[SWState] = None, diagnostics: bool = True,
                 capacity: Optional[int] = None, stream=None, boundary=None, stream_rows: bool = False,
                 tune: Optional[N.Tune] = None):
        torch = _torch()
        self.cfg = cfg
        self.tune = tune
        self.stream = stream
        self.boundary = boundary if boundary is not None else cfg.boundary
        st = state if state is not None else init_state(cfg)
        st = _as_device(st)
        self.t0 = st.t          # a resumed state keeps its clock (rows() continues from it)
        self.a = st
        self.b = SWState(st.H.empty_like(), st.U.empty_like(), st.V.empty_like(), st.g, st.dx, st.dy, st.t)
        self.diag = diagnostics or cfg.dt is None
        self.n = 0
        cap = (capacity if capacity is not None else cfg.steps) + 1
        self.slots = ReductionSlots(cap, st.H.storage.device) if self.diag else None
        # stream_rows: every step's diagnostics row is copied back into pinned
        # host memory right after the step (stream-ordered, no host sync)
        self.host_rows = None
        if self.diag:
            red = self.slots.reduce_struct(0)
            g = _grid(st.H)
            N.check(N.lib().fkc_sw_reduce_state(ctypes.byref(g), st.H.ptr, st.U.ptr, st.V.ptr, st.dx, st.dy,
                                                st.g, ctypes.byref(red), _stream_ptr(stream)))
            if stream_rows:
                self.host_rows = torch.zeros((cap, 5), dtype=torch.int64, pin_memory=True)
                self.host_rows[0:1].copy_(self.slots.buf[0:1], non_blocking=True)
        self._args = [None, None]
        self.torch = torch

    def _loop_args(self, first: int, steps: int, use_graph: bool = False) -> N.LoopArgs:
        """Argument block of the native time loop (fkc_sw_advance_n): buffer
        A = self.a, B = self.b, global step index `first`, per-step
        reduction rows in self.slots (row i+1 = state after step i)."""
        cfg = self.cfg
        L = N.LoopArgs()
        L.step = _step_args(self.a, self.b, cfg.dt if cfg.dt is not None else 0.0, self.boundary, cfg.mode,
                            cfg.variant, None, None, cfg.cfl_factor, self.tune)
        L.first_step = first
        L.steps = steps
        if self.diag:
            L.slots = self.slots.buf.data_ptr()
            L.dt_from_slots = int(cfg.dt is None)
            L.want_cfl = int(cfg.dt is None)
            if self.host_rows is not None:
                L.host_slots = self.host_rows.data_ptr()
        L.use_graph = int(use_graph)
        return L

    def advance(self, steps: int):
        """Enqueue `steps` steps with ONE native call (the loop runs in C,
        fkc_sw_advance_n); no host synchronisation."""
        if self.diag and self.n + steps >= self.slots.n:
            raise ValueError("reduction slot capacity exceeded")
        if steps <= 0:
            return self
        L = self._loop_args(self.n, steps)
        N.check(N.lib().fkc_sw_advance_n(ctypes.byref(L), _stream_ptr(self.stream)))
        self.n += steps
        return self

    def capture(self, steps: int):
        """CUDA-graph the next `steps` steps (fixed dt, no diagnostics) for
        launch-bound small grids: returns a callable that replays them.
        `steps` must be even so the double buffers end where they started;
        each replay advances the state by `steps` steps.  The graph is built
        and cached natively (fkc_sw_advance_n with use_graph)."""
        torch = self.torch
        if steps % 2 or self.diag:
            raise ValueError("capture needs an even step count and diagnostics off")
        stream = self.stream if self.stream is not None else torch.cuda.Stream()
        self.advance(2)                      # warm-up outside capture (tensor maps, attributes)
        torch.cuda.synchronize()
        parity = self.n % 2
        L = self._loop_args(parity, steps, use_graph=True)
        sp = stream.cuda_stream
        own = self.stream is None            # a private capture stream: order it with the caller's

        def launch():
            if own:
                stream.wait_stream(torch.cuda.current_stream())
            N.check(N.lib().fkc_sw_advance_n(ctypes.byref(L), sp))
            if own:
                torch.cuda.current_stream().wait_stream(stream)
            self.n += steps

        launch()                             # capture + first launch

        def replay():
            launch()
        replay.args = L
        return replay

    def state(self) -> SWState:
        s = self.a if self.n % 2 == 0 else self.b
        return s

    def diagnostics(self) -> dict:
        """All reduction rows so far: from the pinned host mirror the steps
        streamed back (stream_rows=True), else one device->host copy."""
        if not self.diag:
            return {}
        if self.host_rows is not None:
            torch = self.torch
            (self.stream if self.stream is not None else torch.cuda.current_stream()).synchronize()
            return ReductionSlots.decode(self.host_rows[: self.n + 1].numpy())
        return ReductionSlots.decode(self.slots.buf[: self.n + 1].cpu().numpy())

    def rows(self) -> RunResult:
        # the steps run with the state's own spacing (SWState.dx / dy), so the
        # mass does too
        return _run_result(self.cfg, self.diagnostics(), self.n, self.t0, self.a.dx * self.a.dy, self.state())


def _run_result(cfg: SWConfig, d: dict, n: int, t0: float, cell_area: float, st: SWState) -> RunResult:
    """The per-step rows (step, t, dt, mass, max|hu|, max|hv|) of a run from
    its decoded reduction rows; raises the SPEC errors a row reports."""
    f = dtype_of(cfg.precision).type
    rows = []
    dts = []
    t = t0
    if d["err"][0]:
        raise_for_error(int(d["err"][0]), "in the initial state")
    for k in range(n):
        if d["err"][k + 1]:
            raise_for_error(int(d["err"][k + 1]), f"at step {k + 1}")
        dt = float(cfg.dt) if cfg.dt is not None else float(f(cfg.cfl_factor) * f(d["cfl_min"][k]))
        t += dt
        dts.append(dt)
        rows.append((k + 1, t, dt, float(d["mass"][k + 1]) * cell_area,
                     float(d["max_hu"][k + 1]), float(d["max_hv"][k + 1])))
    st.t = t
    return RunResult(rows, st, np.array(dts))


# grids from this size up take the streamed host path (below it a run is
# short next to its copies' latency, and the resident / per-step paths apply)
STREAM_MIN_CELLS = 1 << 20


def _host_arrays(st: SWState):
    return [getattr(st, n).data for n in ("H", "U", "V")]


def _streamable(cfg: SWConfig, state: SWState, out: Optional[SWState]) -> bool:
    """fkc_sw_run_host's domain: fixed dt, no periodic rows, the TMA layout,
    C-contiguous host arrays of one row pitch (in and out)."""
    if cfg.dt is None or state.on_device:
        return False
    bc = _bc4(cfg.boundary)
    if bc[2] == N.BC_PERIODIC or cfg.variant not in ("auto", "tma"):
        return False
    nx, ny = state.full.nx - 2, state.full.ny - 2
    cpl = 4 if state.precision == "f32" else 2
    if nx % cpl or nx * ny < STREAM_MIN_CELLS:
        return False
    arrs = _host_arrays(state) + (_host_arrays(out) if out is not None else [])
    for a in arrs:
        if not isinstance(a, np.ndarray) or not a.flags.c_contiguous or a.dtype != dtype_of(state.precision) \
                or a.shape != (ny + 2, nx + 2):
            return False
    return True


def _run_streamed(cfg: SWConfig, state: SWState, out: Optional[SWState], tune: Optional[N.Tune] = None,
                  band_rows: int = 0) -> RunResult:
    """run() from and to host memory with the copies overlapping the steps
    (fkc_sw_run_host): the bands of the state are stepped while later ones
    are still uploading and downloaded as soon as their last step is done."""
    torch = _torch()
    full, prec = state.full, state.precision
    a = SWState(DeviceField(full, prec), DeviceField(full, prec), DeviceField(full, prec),
                state.g, state.dx, state.dy, state.t)
    b = SWState(a.H.empty_like(), a.U.empty_like(), a.V.empty_like(), state.g, state.dx, state.dy, state.t)
    if out is None:
        out = SWState(*(Field(full, np.empty((full.ny, full.nx), dtype_of(prec)), prec) for _ in range(3)),
                      state.g, state.dx, state.dy, state.t)
    slots = ReductionSlots(cfg.steps + 1, a.H.storage.device)
    host_rows = torch.zeros((cfg.steps + 1, 5), dtype=torch.int64, pin_memory=True)
    L = N.LoopArgs()
    L.step = _step_args(a, b, cfg.dt, cfg.boundary, cfg.mode, cfg.variant, None, None, cfg.cfl_factor, tune)
    L.first_step = 0
    L.steps = cfg.steps
    L.slots = slots.buf.data_ptr()
    L.host_slots = host_rows.data_ptr()
    src = (ctypes.c_void_p * 3)(*(x.ctypes.data for x in _host_arrays(state)))
    dst = (ctypes.c_void_p * 3)(*(x.ctypes.data for x in _host_arrays(out)))
    stream = torch.cuda.current_stream()
    N.check(N.lib().fkc_sw_run_host(ctypes.byref(L), src, dst, _host_arrays(state)[0].strides[0], band_rows,
                                    stream.cuda_stream))
    stream.synchronize()
    # row 0 (the uploaded state) was reduced band by band inside the call
    host_rows[0].copy_(slots.buf[0])
    d = ReductionSlots.decode(host_rows.numpy())
    out.g, out.dx, out.dy = state.g, state.dx, state.dy
    return _run_result(cfg, d, cfg.steps, state.t, state.dx * state.dy, out)


def run(cfg: SWConfig, engine: str = "cuda", state: Optional[SWState] = None,
        to_host: bool = False, out: Optional[SWState] = None) -> RunResult:
    """Time loop: apply_boundary -> dt -> advance -> swap ->
    diagnostics (mass, max|hu|, max|hv|, dt), aborting on non-finite values.

    The whole loop is enqueued on the GPU by one native call; per-step
    diagnostics come from the reductions fused into each step and each
    step's row is copied back to pinned host memory as soon as the step is
    done (stream-ordered, no host synchronisation until the end).
    A host ``state`` is uploaded first; ``to_host=True`` returns the final
    state as host Fields (written into ``out``'s arrays when given).  With a
    host state, host output and a fixed dt on a large grid the upload, the
    steps and the download overlap (fkc_sw_run_host: bands of rows stepped
    as a wavefront while later bands are still crossing PCIe).
    """
    if engine not in ENGINES:
        raise ValueError(f"engine {engine!r} is not provided by the B200 package "
                         f"(available: {ENGINES}); the CPU engines live in the reference")
    if state is not None and (to_host or out is not None) and _streamable(cfg, state, out):
        return _run_streamed(cfg, state, out)
    sim = Simulation(cfg, state=state, diagnostics=True, stream_rows=True)
    sim.advance(cfg.steps)
    res = sim.rows()
    if to_host or out is not None:
        res.state = res.state.to_host(out)
    return res
