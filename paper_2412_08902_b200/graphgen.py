"""Seeded synthetic graph generators on the GPU (benchmark inputs).

The reference's generators (graphgen.py) use triu_indices and are O(n^2); the
BASELINE configs need 233K-vertex / 115M-edge and 16.8M-vertex / 1B-edge
graphs, so these are vectorised on the device with a seeded torch.Generator
(Philox; deterministic for a given seed and size).

  reddit_shaped(): capped Chung-Lu power law, gamma 2.3, n = 232,965, ~114.6M
                   directed nnz before gcn self-loops (C2/C3/C4)
  reddit_community(): the same shape with 41 planted communities, scrambled ids
                   (secondary C2/C4 input: the locality LOA is meant to recover)
  cora_shaped():   n = 2,708, ~10.5K directed nnz (C1)
  rmat():          R-MAT (a,b,c,d) = (0.57, 0.19, 0.19, 0.05) (C5)
All graphs: self-loops dropped, symmetrised, deduplicated, unit values.
"""

from __future__ import annotations

import torch

from .matrices import DeviceCsr

REDDIT_N = 232_965
REDDIT_TARGET_NNZ = 114_615_892


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def csr_from_keys(n: int, keys: torch.Tensor, values: torch.Tensor | None = None) -> DeviceCsr:
    """keys = row*n + col, sorted ascending and unique -> DeviceCsr."""
    dev = keys.device
    rows = torch.div(keys, n, rounding_mode="floor")
    cols = (keys - rows * n).to(torch.int32)
    counts = torch.bincount(rows, minlength=n)
    row_ptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    torch.cumsum(counts, 0, out=row_ptr[1:])
    vals = torch.ones(keys.numel(), dtype=torch.float32, device=dev) if values is None else values
    return DeviceCsr(n, n, row_ptr, cols, vals.to(torch.float32),
                     host_values_f64=None if values is not None else None)


def symmetric_from_pairs(n: int, u: torch.Tensor, v: torch.Tensor) -> DeviceCsr:
    keep = u != v
    u, v = u[keep], v[keep]
    keys = torch.cat([u * n + v, v * n + u])
    del u, v, keep
    keys = torch.unique(keys, sorted=True)
    return csr_from_keys(n, keys)


def chung_lu_device(n: int, avg_deg: float, seed: int = 0, gamma: float = 2.3, i0: float | None = None,
                    oversample: float = 1.12, device="cuda") -> DeviceCsr:
    """Chung-Lu with weights w_i = (1 + i/i0)^(-1/(gamma-1)), endpoints drawn by inverse
    CDF, ids shuffled.  ~oversample compensates dedup/self-loop losses."""
    g = _gen(seed, device)
    if i0 is None:
        i0 = max(1.0, n * 350.7 / REDDIT_N)
    i = torch.arange(n, device=device, dtype=torch.float64)
    w = (1.0 + i / i0) ** (-1.0 / (gamma - 1.0))
    cdf = torch.cumsum(w, 0)
    cdf = cdf / cdf[-1]
    pairs = int(n * avg_deg / 2 * oversample)
    perm = torch.randperm(n, generator=g, device=device)
    out_u, out_v = [], []
    chunk = 1 << 25
    for s in range(0, pairs, chunk):
        m = min(chunk, pairs - s)
        ru = torch.rand(m, generator=g, device=device, dtype=torch.float64)
        rv = torch.rand(m, generator=g, device=device, dtype=torch.float64)
        u = torch.clamp(torch.searchsorted(cdf, ru), max=n - 1)
        v = torch.clamp(torch.searchsorted(cdf, rv), max=n - 1)
        out_u.append(perm[u])
        out_v.append(perm[v])
    return symmetric_from_pairs(n, torch.cat(out_u), torch.cat(out_v))


def reddit_shaped(seed: int = 0, device="cuda") -> DeviceCsr:
    """C2: n = 232,965, capped power law (max weight ratio as in SURVEY §8d), target
    ~114.6M directed nnz before self-loops."""
    return chung_lu_device(REDDIT_N, REDDIT_TARGET_NNZ / REDDIT_N, seed=seed, oversample=1.03,
                           device=device)


def community_power_law(n: int, avg_deg: float, communities: int, p_in: float = 0.8, seed: int = 0,
                        gamma: float = 2.3, i0: float | None = None, oversample: float = 1.03,
                        device="cuda") -> DeviceCsr:
    """Degree-corrected planted partition: Chung-Lu weights as chung_lu_device, every vertex
    in one of `communities` groups (uniform), a fraction p_in of the edges drawn with both
    endpoints inside one community (community chosen by weight mass, endpoints by weight
    within it), the rest drawn globally.  Vertex ids are a random permutation, so rows carry
    no locality until a layout pass (LOA, C4) recovers it."""
    g = _gen(seed, device)
    if i0 is None:
        i0 = max(1.0, n * 350.7 / REDDIT_N)
    i = torch.arange(n, device=device, dtype=torch.float64)
    w = (1.0 + i / i0) ** (-1.0 / (gamma - 1.0))
    comm = torch.randint(0, communities, (n,), generator=g, device=device)
    order = torch.argsort(comm * n + torch.arange(n, device=device))  # vertices grouped by community
    cw = torch.cumsum(w[order], 0)
    total = cw[-1]
    cnt = torch.bincount(comm, minlength=communities)
    cend = torch.cumsum(cnt, 0)  # community c owns order[cend[c]-cnt[c] : cend[c]]
    mass_end = cw[cend - 1]
    mass_start = mass_end - torch.bincount(comm, weights=w, minlength=communities)
    ccdf = torch.cumsum(mass_end - mass_start, 0) / total
    gcdf = torch.cumsum(w, 0) / total
    perm = torch.randperm(n, generator=g, device=device)
    pairs = int(n * avg_deg / 2 * oversample)
    out_u, out_v = [], []
    chunk = 1 << 25
    for s in range(0, pairs, chunk):
        m = min(chunk, pairs - s)
        intra = torch.rand(m, generator=g, device=device) < p_in
        c = torch.clamp(torch.searchsorted(ccdf, torch.rand(m, generator=g, device=device, dtype=torch.float64)),
                        max=communities - 1)
        lo, span = mass_start[c], mass_end[c] - mass_start[c]
        ru = lo + torch.rand(m, generator=g, device=device, dtype=torch.float64) * span
        rv = lo + torch.rand(m, generator=g, device=device, dtype=torch.float64) * span
        ui = order[torch.clamp(torch.searchsorted(cw, ru), max=n - 1)]
        vi = order[torch.clamp(torch.searchsorted(cw, rv), max=n - 1)]
        gu = torch.clamp(torch.searchsorted(gcdf, torch.rand(m, generator=g, device=device, dtype=torch.float64)),
                         max=n - 1)
        gv = torch.clamp(torch.searchsorted(gcdf, torch.rand(m, generator=g, device=device, dtype=torch.float64)),
                         max=n - 1)
        out_u.append(perm[torch.where(intra, ui, gu)])
        out_v.append(perm[torch.where(intra, vi, gv)])
    return symmetric_from_pairs(n, torch.cat(out_u), torch.cat(out_v))


def reddit_community(seed: int = 0, device="cuda") -> DeviceCsr:
    """C2/C4 secondary input: Reddit-shaped (n = 232,965, ~114.6M directed nnz) with 41
    planted communities (Reddit's class count), 80% intra-community edges, scrambled ids."""
    return community_power_law(REDDIT_N, REDDIT_TARGET_NNZ / REDDIT_N, 41, seed=seed, oversample=1.25,
                               device=device)


def cora_shaped(seed: int = 0, device="cuda") -> DeviceCsr:
    """C1: n = 2,708, ~10.5K directed nnz."""
    return chung_lu_device(2708, 10556 / 2708, seed=seed, oversample=1.06, device=device)


def rmat(scale: int, edge_factor: float, seed: int = 0, abcd=(0.57, 0.19, 0.19, 0.05), device="cuda") -> DeviceCsr:
    """R-MAT quadrant recursion; self-loops dropped, symmetrised, deduplicated."""
    g = _gen(seed, device)
    n = 1 << scale
    m = int(edge_factor * n)
    a, b, c, _ = abcd
    us, vs = [], []
    chunk = 1 << 24
    for s in range(0, m, chunk):
        k = min(chunk, m - s)
        u = torch.zeros(k, dtype=torch.int64, device=device)
        v = torch.zeros(k, dtype=torch.int64, device=device)
        for lvl in range(scale):
            r = torch.rand(k, generator=g, device=device)
            bit_u = (r >= a + b).to(torch.int64)  # quadrants c, d -> lower half
            bit_v = (((r >= a) & (r < a + b)) | (r >= a + b + c)).to(torch.int64)  # b or d -> right half
            u |= bit_u << lvl
            v |= bit_v << lvl
        us.append(u)
        vs.append(v)
    return symmetric_from_pairs(n, torch.cat(us), torch.cat(vs))


def gcn_normalize_device(adj: DeviceCsr) -> DeviceCsr:
    """gnn.normalize_adj(kind='gcn') on the device (see gnn.normalize_adj)."""
    from .gnn import normalize_adj

    return normalize_adj(adj, "gcn")


def dense_features(n: int, dim: int, seed: int, dtype=torch.bfloat16, device="cuda") -> torch.Tensor:
    """U[-1, 1) features (synthetic X), generated on the device."""
    g = _gen(seed, device)
    return (torch.rand(n, dim, generator=g, device=device) * 2 - 1).to(dtype)
