"""Small seeded test matrices (edge cases the reference tests exercise:
empty rows, ragged rows, explicit zeros, single row/column, edge blocks)."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def matrix_a():
    with open(os.path.join(GOLDEN, "matrix_a.json")) as f:
        return json.load(f)


def random_coo(seed, m, n, density=0.3, zeros=0.0, shuffle=True, dups=0, fp32=True):
    """Unique coordinates with values on an fp32-exact grid (never 0 unless
    `zeros` > 0, which turns that fraction into explicit zeros)."""
    rng = np.random.default_rng(seed)
    mask = rng.random((m, n)) < density
    r, c = np.nonzero(mask)
    k = len(r)
    v = (0.5 + rng.integers(0, 1 << 23, k) / float(1 << 23)) * np.where(rng.random(k) < 0.5, -1, 1)
    if zeros > 0 and k:
        v[rng.random(k) < zeros] = 0.0
    if fp32:
        v = v.astype(np.float32).astype(np.float64)
    if dups and k:
        pick = rng.integers(0, k, dups)
        r = np.concatenate([r, r[pick]])
        c = np.concatenate([c, c[pick]])
        v = np.concatenate([v, v[pick] * 0.5])
    if shuffle:
        p = rng.permutation(len(r))
        r, c, v = r[p], c[p], v[p]
    return r.astype(np.int64), c.astype(np.int64), v


def power_law_coo(seed, m, n, avg=6.0, alpha=1.6):
    """Skewed row lengths (a few heavy rows), unique sorted coordinates."""
    rng = np.random.default_rng(seed)
    lens = np.minimum(n, (rng.pareto(alpha, m) * avg * 0.5).astype(np.int64))
    rows, cols = [], []
    for i, L in enumerate(lens):
        if L:
            cols.append(np.sort(rng.choice(n, int(L), replace=False)))
            rows.append(np.full(int(L), i))
    if not rows:
        return np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0)
    r = np.concatenate(rows).astype(np.int64)
    c = np.concatenate(cols).astype(np.int64)
    k = len(r)
    v = (0.5 + rng.integers(0, 1 << 23, k) / float(1 << 23)) * np.where(rng.random(k) < 0.5, -1, 1)
    return r, c, v.astype(np.float32).astype(np.float64)


# Shapes that stress edge handling: single row / column, blocks wider than
# the matrix, ragged edge blocks, tall and wide.
EDGE_SHAPES = [(1, 1), (1, 7), (7, 1), (3, 3), (5, 4), (16, 16), (17, 33), (40, 9), (64, 64)]
