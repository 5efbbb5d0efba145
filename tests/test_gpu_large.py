"""GPU tier: BASELINE config 4 field sizes, where per-field byte offsets pass
2^31 and 2^32 (VERDICT r01 "next" item 1).

* 32768^2 f32 on one GPU (the strong-scaling base: 6 x 4.30 GB) -- row y of a
  field starts y * 131200 bytes past its first row, so rows above ~16368 lie
  beyond 2 GiB and the top rows beyond 4 GiB;
* 32768 x 16384, the per-GPU tile of the 1x2 split of 32768^2 (2.15 GB per
  field: its top rows lie beyond 2 GiB).

The whole grid is advanced K steps on the device from a seeded random state
with momentum everywhere.  The CPU oracle (C restatement, DSL op order)
cannot step 25.8 GB in a test, so it advances row WINDOWS instead: a slab of
the initial state reaching K+1 rows past the window on each side, full width
(so the x-boundaries are the real ones).  The slab's cut edges get
boundary-filled garbage, which travels one row per step -- after K steps
every window row is untouched by it (the domain of dependence), so exact
mode must match the oracle bit for bit there and fast mode within its
tolerance.  Windows: the bottom rows (true boundary), rows straddling the
2 GiB offset, and the top rows (true boundary, past 4 GiB at 32768^2).
"""

import numpy as np
import pytest

from oracle import c_oracle

pytestmark = pytest.mark.gpu

K = 3
DT = 0.05
FAST_RTOL = 2e-5


def _random_state_on_device(nx, ny, seed):
    """h ~ U[0.9, 1.1], hu, hv ~ U[-0.05, 0.05] (SURVEY.md 8(d) parity input),
    generated on the device in row chunks, then the reflective halo."""
    import torch
    from paper_1107_2157_b200 import swdemo
    from paper_1107_2157_b200.field import DeviceField
    from paper_1107_2157_b200.region import Extent
    full = Extent(nx + 2, ny + 2)
    fields = [DeviceField(full, "f32", fill=0.0) for _ in range(3)]
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    for r0 in range(1, ny + 1, 4096):
        r1 = min(ny + 1, r0 + 4096)
        for k, f in enumerate(fields):
            t = torch.rand((r1 - r0, nx), generator=gen, device="cuda", dtype=torch.float32)
            f.data[r0:r1, 1:-1] = (0.9 + 0.2 * t) if k == 0 else (0.1 * t - 0.05)
    st = swdemo.SWState(*fields)
    swdemo.apply_boundary(st, "reflective")
    return st


def _rows(st, y0, y1):
    """Rows y0 .. y1-1 (full width) of H, U, V, copied to the host."""
    return tuple(np.ascontiguousarray(f.data[y0:y1].cpu().numpy()) for f in (st.H, st.U, st.V))


def _check_windows(nx, ny, windows, mode):
    import torch
    from paper_1107_2157_b200 import swdemo
    st = _random_state_on_device(nx, ny, seed=nx ^ ny)
    slabs = []
    for a, b in windows:                       # interior rows a .. b-1 (full-array row index)
        s0, s1 = max(0, a - K - 1), min(ny + 2, b + K + 1)
        slabs.append((a, b, s0, s1, _rows(st, s0, s1)))
    cfg = swdemo.SWConfig(nx=nx, ny=ny, steps=K, dt=DT, mode=mode, variant="tma")
    sim = swdemo.Simulation(cfg, state=st, diagnostics=False)
    sim.advance(K)
    torch.cuda.synchronize()
    fin = sim.state()
    assert fin.H.pitch * 4 * (ny + 1) > 2 ** 31          # the top rows lie past 2 GiB
    for a, b, s0, s1, slab in slabs:
        want = c_oracle.run_fixed(*slab, K, 1.0, 1.0, DT)
        got = _rows(fin, a, b)
        sub = [w[a - s0:b - s0] for w in want]
        for k, (g, w) in enumerate(zip(got, sub)):
            if mode == "exact":
                bad = np.argwhere(g != w)
                assert bad.size == 0, (k, a, b, bad[:3].tolist())
            else:
                assert np.max(np.abs(g.astype(np.float64) - w)) <= FAST_RTOL * np.max(np.abs(w)), (k, a, b)
    del sim, st, fin
    torch.cuda.empty_cache()


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_config4_single_gpu_32768sq(mode):
    n = 32768
    # row y starts y * 131200 B into a field: 2 GiB at y ~ 16368, 4 GiB at y ~ 32736
    _check_windows(n, n, [(1, 12), (16360, 16380), (32750, 32769)], mode)


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_config4_tile_32768x16384(mode):
    _check_windows(32768, 16384, [(1, 8), (8190, 8200), (16370, 16385)], mode)
