"""GPU tier: the 2-D decomposition at the headline size, where every tile
(8192 x 16384 cells) takes the large-grid eager schedule of the step kernel
(uniform 14-row segments, csrc/fkc_sw.cu SEG_HBM): the fused peer exchange
on concurrent streams and the pack / unpack exchange must equal the
undecomposed run over full interiors (fast mode: same arithmetic per cell)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("exchange,concurrent", [("fused", True), ("pack", False)])
def test_headline_size_decomposed_equals_single_domain(exchange, concurrent):
    import torch

    from paper_1107_2157_b200 import swdemo
    from paper_1107_2157_b200.decomp import run_local_decomposed
    n = 16384
    cfg = swdemo.SWConfig(nx=n, ny=n, dt=0.02, mode="fast", boundary="reflective")
    sim = swdemo.Simulation(cfg, state=swdemo.init_state(cfg).to_device(), diagnostics=False)
    sim.advance(3)
    ref = [f.to_numpy() for f in (sim.state().H, sim.state().U, sim.state().V)]
    del sim
    torch.cuda.empty_cache()
    grid, tiles = run_local_decomposed(cfg, 2, 1, 3, exchange=exchange, concurrent=concurrent)
    for r, t in enumerate(tiles):
        tl = grid.tile(r)
        for k, f in enumerate((t.H, t.U, t.V)):
            a = f.to_numpy()[1:-1, 1:-1]
            b = ref[k][tl.y0 + 1: tl.y0 + 1 + tl.ny, tl.x0 + 1: tl.x0 + 1 + tl.nx]
            assert np.array_equal(a, b), (exchange, r, k)
    del tiles
    torch.cuda.empty_cache()
