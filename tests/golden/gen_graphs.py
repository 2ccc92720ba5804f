"""Seeded numpy graph generators shared by the golden-vector script and the CPU tests.

Test infrastructure only.  These are small, deterministic numpy generators
(Chung-Lu power law, planted communities) so fixtures can store generator
parameters instead of whole adjacency arrays.
"""

from __future__ import annotations

import numpy as np


def chung_lu_edges(n: int, n_pairs: int, gamma: float = 2.3, i0: float | None = None, seed: int = 0):
    """Undirected Chung-Lu pairs: endpoints drawn proportional to w_i = (1 + i/i0)^(-1/(gamma-1)),
    ids shuffled, self-loops dropped, symmetrised + deduplicated.  Returns (rows, cols) of the
    symmetric adjacency sorted by (row, col)."""
    rng = np.random.default_rng(seed)
    if i0 is None:
        i0 = max(1.0, n / 664.0)
    w = (1.0 + np.arange(n) / i0) ** (-1.0 / (gamma - 1.0))
    p = w / w.sum()
    u = rng.choice(n, size=n_pairs, p=p)
    v = rng.choice(n, size=n_pairs, p=p)
    perm = rng.permutation(n)
    u, v = perm[u], perm[v]
    keep = u != v
    u, v = u[keep], v[keep]
    r = np.concatenate([u, v]).astype(np.int64)
    c = np.concatenate([v, u]).astype(np.int64)
    key = np.unique(r * n + c)
    return key // n, key % n


def csr_from_pairs(n: int, rows, cols):
    counts = np.bincount(rows, minlength=n)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    return row_ptr, np.asarray(cols, dtype=np.int64), np.ones(len(cols))


def cora_shaped(seed: int = 0):
    """n = 2708, ~5.3K undirected edges (~10.5K directed nnz), power law."""
    n = 2708
    r, c = chung_lu_edges(n, 5600, gamma=2.3, seed=seed)
    return n, r, c


def power_law(n: int, avg_deg: float, seed: int = 0, gamma: float = 2.3):
    r, c = chung_lu_edges(n, int(n * avg_deg / 2 * 1.1), gamma=gamma, seed=seed)
    return n, r, c


def block_pairs(num_blocks: int, block_size: int, p_intra: float, p_inter: float, seed: int, scramble_seed=None):
    """Planted partition (restates rowwin.graphgen.block_community semantics with numpy sampling)."""
    n = num_blocks * block_size
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, k=1)
    same = (iu // block_size) == (ju // block_size)
    keep = rng.random(iu.size) < np.where(same, p_intra, p_inter)
    u, v = iu[keep], ju[keep]
    if scramble_seed is not None:
        perm = np.random.default_rng(scramble_seed).permutation(n)
        u, v = perm[u], perm[v]
    r = np.concatenate([u, v]).astype(np.int64)
    c = np.concatenate([v, u]).astype(np.int64)
    key = np.unique(r * n + c)
    return n, key // n, key % n
