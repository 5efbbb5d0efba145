"""CPU tier: region module examples and exhaustive halo
properties for halos <= 3 and extents <= 32."""

import itertools

import pytest

from paper_1107_2157_b200.region import (Extent, Halo, HaloTooLarge, Rect, global_coord, interior_of,
                                         local_linear_index, local_tile_extent, owned_cell)


def test_spec_examples():
    assert interior_of(Extent(6, 5), Halo(1, 1, 1, 1)) == Rect(1, 1, 4, 3)
    assert interior_of(Extent(6, 5), Halo(0, 0, 0, 0)) == Rect(0, 0, 6, 5)
    assert interior_of(Extent(6, 5), Halo(0, 1, 1, 1)) == Rect(0, 1, 5, 3)
    t = local_tile_extent(Extent(16, 8), Halo(1, 1, 1, 1))
    assert t == Extent(18, 10) and t.cells == 180
    assert local_tile_extent(Extent(4, 4), Halo(2, 0, 0, 3)) == Extent(6, 7)
    assert local_linear_index(3, 2, 16, Halo(1, 1, 0, 0)) == 39
    assert local_linear_index(17, 9, 16, Halo(1, 1, 1, 1)) == 179
    assert global_coord((1, 0), (0, 0), Extent(16, 8)) == (16, 0)
    assert global_coord((1, 1), (17, 9), Extent(16, 8)) == (33, 17)
    with pytest.raises(HaloTooLarge):
        interior_of(Extent(3, 3), Halo(2, 2, 0, 0))
    with pytest.raises(ValueError):
        Halo(-1, 0, 0, 0)
    with pytest.raises(ValueError):
        Extent(0, 3)
    # section 3.1: one more face than cells
    full = Extent(10, 10)
    assert interior_of(full, Halo(0, 1, 1, 1)).nx == interior_of(full, Halo(1, 1, 1, 1)).nx + 1


def test_exhaustive_halo_properties():
    for l, r, d, u in itertools.product(range(4), repeat=4):
        h = Halo(l, r, d, u)
        for nx in range(1, 33, 3):
            for ny in range(1, 33, 5):
                full = Extent(nx, ny)
                if nx - l - r < 1 or ny - d - u < 1:
                    with pytest.raises(HaloTooLarge):
                        interior_of(full, h)
                    continue
                rc = interior_of(full, h)
                assert rc.x0 == l and rc.y0 == d
                assert rc.x0 + rc.nx + r == nx and rc.y0 + rc.ny + u == ny


def test_tile_index_bijection_and_ownership_partition():
    group, halo = Extent(16, 8), Halo(1, 1, 1, 1)
    tile = local_tile_extent(group, halo)
    idx = {local_linear_index(x, y, group.nx, halo) for x in range(tile.nx) for y in range(tile.ny)}
    assert idx == set(range(tile.cells))
    owned = [owned_cell((gx, gy), (tx, ty), group, halo)
             for gx in range(2) for gy in range(2) for tx in range(16) for ty in range(8)]
    assert len(owned) == len(set(owned)) == 32 * 16
    assert set(owned) == {(x, y) for x in range(1, 33) for y in range(1, 17)}
