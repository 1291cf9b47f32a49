"""The chunk map of the chunked later sweeps (sweep_march2.cu: dyn_chunk / dyn_chunk_count):
every band-row of a launch belongs to exactly one chunk, whatever the lattice and grid, so
which CTA takes a chunk cannot change a result.  Host-only (no GPU)."""
import ctypes as C

import pytest

from paper_2003_04345_b200 import _lib


def _hook():
    L = _lib.lib()
    f = L.mb4cu_debug_chunk
    f.restype = C.c_longlong
    f.argtypes = [C.c_longlong, C.c_longlong, C.c_longlong, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]
    return f


@pytest.mark.parametrize("total,grid", [
    (67 * 8192, 444),      # cfg5 later sweeps: 67 bands of 8192 rows, 3 CTAs on each of 148 SMs
    (34 * 4096, 444),      # cfg4
    (9 * 1024, 444),       # cfg3 (below the chunking threshold, the map still has to be exact)
    (133 * 32768, 444),    # the 8-GPU cfg5 lattice on one GPU
    (8192 * 67 - 5, 296), (1, 1), (31, 7), (32, 1), (33, 2), (4096, 4096), (100000, 3),
])
def test_chunks_cover_every_band_row_once(total, grid):
    f = _hook()
    n = f(-1, total, grid, None, None)
    assert n >= 1
    p0, p1 = C.c_longlong(), C.c_longlong()
    pos = 0
    sizes = []
    for c in range(n):
        assert f(c, total, grid, C.byref(p0), C.byref(p1)) == 1
        assert p0.value == pos and p0.value < p1.value <= total  # contiguous, in order, non-empty
        sizes.append(p1.value - p0.value)
        pos = p1.value
    assert pos == total
    # past the last chunk: every CTA's final grab ends its loop
    for c in (n, n + 1, n + grid):
        assert f(c, total, grid, C.byref(p0), C.byref(p1)) == 0
    # guided: chunk sizes never grow (the tail balances the CTAs' uneven rates)
    assert all(a >= b for a, b in zip(sizes[:-2], sizes[1:-1]))


def test_chunk_hook_rejects_bad_arguments():
    f = _hook()
    assert f(-1, 0, 4, None, None) == -1
    assert f(0, 10, 0, None, None) == -1
    assert f(0, 10, 2, None, None) == -1
