"""CPU checks of the distributed rank-2k tile ownership: the tile
schedule of the skew rank-2k kernel (skew_tile_schedule runs the kernel's own host/device tile
decoder, tma_tile_coords, for 128-row x 64-column tiles) visits exactly the tiles that meet
the strictly lower triangle, and over the ranks of a 1D block-cyclic column distribution the
per-rank sets partition them with rank r owning exactly the column tiles q = r (mod P)."""
import ctypes

import numpy as np
import pytest


def _sched(L, ntm, P, r):
    cnt = L.skew_tile_schedule(ntm, P, r, None, None, 0)
    assert cnt >= 0
    tm = np.zeros(max(cnt, 1), dtype=np.int64)
    tn = np.zeros(max(cnt, 1), dtype=np.int64)
    got = L.skew_tile_schedule(ntm, P, r, tm.ctypes.data_as(ctypes.c_void_p), tn.ctypes.data_as(ctypes.c_void_p), cnt)
    assert got == cnt
    return tm[:cnt], tn[:cnt]


@pytest.fixture(scope="module")
def L():
    from paper_1912_04062_b200 import build
    import paper_1912_04062_b200 as m
    build.build()
    return m.lib()


@pytest.mark.parametrize("ntm", [0, 1, 2, 3, 7, 64, 511, 1023])
def test_single_device_schedule_is_the_lower_triangle(L, ntm):
    tm, tn = _sched(L, ntm, 1, 0)
    want = {(a, b) for a in range(ntm) for b in range(2 * ntm) if 128 * a + 127 > 64 * b}
    assert len(tm) == len(want) == ntm * (ntm + 1)
    assert set(zip(tm.tolist(), tn.tolist())) == want


@pytest.mark.parametrize("ntm", [1, 2, 5, 8, 9, 64, 255, 512])
@pytest.mark.parametrize("P", [2, 3, 4, 8])
def test_ranks_partition_the_lower_triangle(L, ntm, P):
    seen = {}
    for r in range(P):
        tm, tn = _sched(L, ntm, P, r)
        assert np.all(tn % P == r), "rank r owns the column tiles q = r mod P"
        assert np.all(128 * tm + 127 > 64 * tn) and np.all(tm < ntm) and np.all(tn < 2 * ntm)
        for a, b in zip(tm.tolist(), tn.tolist()):
            assert (a, b) not in seen, f"tile {(a, b)} visited by ranks {seen[(a, b)]} and {r}"
            seen[(a, b)] = r
    assert len(seen) == ntm * (ntm + 1)
