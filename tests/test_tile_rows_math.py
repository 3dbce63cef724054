"""Host check of the closed forms `k_tile_rows` (csrc/binsort.cu)
uses to derive every tile row's ranges without communication between CTAs:
with d the tile-rect difference array, per column x'
  col_y(x') = sum_{y'' <= y} d(x', y''),   counts c(x, y) = sum_{x' <= x} col_y(x'),
  S(y) = sum_{y' < y} sum_x c(x, y') = sum_x' (TX - x') sum_{y'' < y} (y - y'') d(x', y''),
  P = S(TY),
against the plain 2-D prefix and row-major scan on random rect sets."""
import numpy as np


def _rects(rng, n, TX, TY):
    x0 = rng.integers(0, TX, n)
    y0 = rng.integers(0, TY, n)
    x1 = np.minimum(TX - 1, x0 + rng.integers(0, 6, n))
    y1 = np.minimum(TY - 1, y0 + rng.integers(0, 6, n))
    return x0, y0, x1, y1


def test_row_offsets_closed_form():
    rng = np.random.default_rng(3)
    for TX, TY, n in ((7, 5, 40), (75, 43, 3000), (163, 3, 500), (1, 1, 3)):
        x0, y0, x1, y1 = _rects(rng, n, TX, TY)
        d = np.zeros((TY + 1, TX + 1), np.int64)  # the kernels' 2-D difference array
        for a, b, c, e in zip(x0, y0, x1, y1):
            d[b, a] += 1
            d[b, c + 1] -= 1
            d[e + 1, a] -= 1
            d[e + 1, c + 1] += 1
        counts = np.cumsum(np.cumsum(d, 0), 1)[:TY, :TX]  # plain 2-D prefix
        brute = np.zeros((TY, TX), np.int64)
        for a, b, c, e in zip(x0, y0, x1, y1):
            brute[b:e + 1, a:c + 1] += 1
        assert np.array_equal(counts, brute)
        starts = np.concatenate([[0], np.cumsum(counts.ravel())[:-1]]).reshape(TY, TX)  # row-major scan
        dd = d[:TY, :TX]
        xs = np.arange(TX)
        for y in range(TY):
            col = dd[:y + 1].sum(0)
            c = np.cumsum(col)
            S = int(((TX - xs) * ((y - np.arange(y))[:, None] * dd[:y]).sum(0)).sum()) if y else 0
            assert np.array_equal(c, counts[y])
            assert np.array_equal(S + np.concatenate([[0], np.cumsum(c)[:-1]]), starts[y])
        P = int(((TX - xs) * ((TY - np.arange(TY))[:, None] * dd).sum(0)).sum())
        assert P == int(counts.sum()) == int(sum((c - a + 1) * (e - b + 1) for a, b, c, e in zip(x0, y0, x1, y1)))
