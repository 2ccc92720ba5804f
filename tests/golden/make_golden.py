"""Generate golden vectors by running the REFERENCE package (rowwin) in this container.

Usage (dev container only; /root/reference does not exist on the GPU box):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes tests/golden/*.npz.  The GPU box only reads these fixtures; it never
imports the reference.  Each fixture stores the inputs (or the generator
parameters for larger graphs) and the reference outputs:

  windows_*.npz : partition (windows.py:81-106) + features (109-123) +
                  classify_windows(default_model()) (selector.py:63, 284)
                  + spmm_hybrid(precision f32/f64) Z (executors.py:234) + ExecStats
  gnn_*.npz     : normalize_adj (gnn.py:68) + forward/backward fused & unfused (gnn.py:121-205)
  loa_*.npz     : build_windows_optimized groups (layout.py:186) + reorder perm (266)
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")
sys.path.insert(0, HERE)

from rowwin import executors as rex  # noqa: E402
from rowwin import gnn as rgnn  # noqa: E402
from rowwin import layout as rlay  # noqa: E402
from rowwin import selector as rsel  # noqa: E402
from rowwin import windows as rwin  # noqa: E402
from rowwin.matrices import DenseMatrix, Graph, SparseCsr  # noqa: E402

import gen_graphs as gg  # noqa: E402


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def graph_of(n, rows, cols) -> Graph:
    adj = SparseCsr.from_coo(n, n, rows, cols, np.ones(len(rows)))
    return Graph(n, adj, True)


def window_outputs(csr: SparseCsr, dim: int, xseed: int, store_full: bool, with_f64: bool = True):
    ws = rwin.partition(csr)
    feats = [rwin.features(w) for w in ws]
    model = rsel.default_model()
    asg = rsel.classify_windows(model, ws)
    ncols = np.array([f.ncols for f in feats], dtype=np.int64)
    dens = np.array([f.density for f in feats], dtype=np.float64)
    ci = np.array([f.computing_intensity for f in feats], dtype=np.float64)
    nzc = np.concatenate([w.nonzero_cols for w in ws]) if ws else np.zeros(0, np.int64)
    cond = np.concatenate([w.cond_cols for w in ws]) if ws else np.zeros(0, np.int64)
    x = DenseMatrix.random(csr.num_cols, dim, seed=xseed)
    out = dict(
        ncols=ncols, density=dens, ci=ci, codes=asg.codes,
        nonzero_cols_sha=np.array(digest(nzc.astype(np.int64))),
        cond_cols_sha=np.array(digest(cond.astype(np.int64))),
        dim=np.array(dim), xseed=np.array(xseed),
    )
    if store_full:
        out["nonzero_cols"] = nzc.astype(np.int64)
        out["cond_cols"] = cond.astype(np.int64)
    r32 = rex.spmm_hybrid(ws, asg, x, precision="f32")
    out["z_f32"] = r32.z.data
    for k, v in r32.stats.as_dict().items():
        out["stats_" + k] = np.array(v)
    if with_f64:
        out["z_f64"] = rex.spmm_hybrid(ws, asg, x, precision="f64").z.data
        out["z_scalar_f64"] = rex.spmm_scalar(csr, x).z.data
        out["z_tile_f64"] = rex.spmm_tile(ws, x).z.data
    return out


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {name}.npz ({os.path.getsize(path) / 1e3:.1f} kB)")


def csr_arrays(csr: SparseCsr, prefix=""):
    return {prefix + "n_rows": np.array(csr.num_rows), prefix + "n_cols": np.array(csr.num_cols),
            prefix + "row_ptr": csr.row_ptr, prefix + "col_idx": csr.col_idx, prefix + "values": csr.values}


def main():
    from conftest import build_corpus, random_csr  # reference test helpers

    # ---- KAT: tests/test_windows.py:23-32
    kat = SparseCsr.from_coo(2, 16, np.array([0, 0, 1]), np.array([9, 5, 9]), np.array([1.0, 2.0, 3.0]))
    save("windows_kat_condense", **csr_arrays(kat), **window_outputs(kat, 4, 0, True))

    # ---- random matrices (tests/conftest.py:31-39 generator), full arrays stored
    rand_cases = [(33, 20, 0.2, 0), (50, 40, 0.1, 11), (100, 100, 0.05, 15), (70, 50, 0.15, 7),
                  (64, 64, 0.08, 18), (48, 8, 0.3, 5), (500, 300, 0.02, 3), (257, 1000, 0.01, 9),
                  (16, 600, 0.08, 21), (16, 900, 0.06, 22), (32, 2000, 0.04, 23)]
    for i, (r, c, d, s) in enumerate(rand_cases):
        csr = random_csr(r, c, d, s)
        save(f"windows_rand{i}", **csr_arrays(csr), **window_outputs(csr, [1, 3, 8, 17, 32][i % 5], s + 1, True))

    # ---- corpus graphs (tests/conftest.py:50-95), gcn-normalised
    for name, g in build_corpus():
        a = rgnn.normalize_adj(g, "gcn")
        save(f"windows_corpus_{name}", **csr_arrays(a), **window_outputs(a, 32, 1, True))

    # ---- Cora-shaped: generator params stored, reference outputs full
    n, rr, cc = gg.cora_shaped(seed=0)
    g = graph_of(n, rr, cc)
    a = rgnn.normalize_adj(g, "gcn")
    save("windows_cora", gen=np.array("cora_shaped"), seed=np.array(0), **csr_arrays(a),
         **window_outputs(a, 32, 1, True))

    # ---- power-law 8192 / avg deg 40 (mixed TILE/SCALAR) -- arrays hashed, Z stored
    n, rr, cc = gg.power_law(8192, 40.0, seed=7)
    g = graph_of(n, rr, cc)
    a = rgnn.normalize_adj(g, "gcn")
    save("windows_plaw8k", gen=np.array("power_law"), n=np.array(8192), avg_deg=np.array(40.0), seed=np.array(7),
         nnz=np.array(a.nnz), values_sha=np.array(digest(a.values)),
         **window_outputs(a, 32, 1, False, with_f64=False))

    # ---- GNN layer (gnn.py:121-205) on gnp-like graphs, every normalisation, f64
    for kind in ("gcn", "row", "gin", "raw"):
        n, rr, cc = gg.power_law(300, 8.0, seed=11)
        g = graph_of(n, rr, cc)
        a = rgnn.normalize_adj(g, kind)
        layer = rgnn.GnnLayer.random(16, 8, seed=4)
        x = DenseMatrix.random(n, 16, seed=5)
        ws = rwin.partition(a)
        asg = rex.Assignment.from_paths(rex.Path.TILE if i % 2 else rex.Path.SCALAR for i in range(len(ws)))
        xn, z, tf = rgnn.forward(layer, a, x, mode="fused", assignment=asg, windows=ws)
        xu, zu, tu = rgnn.forward(layer, a, x, mode="unfused", assignment=asg, windows=ws)
        gout = DenseMatrix.random(n, 8, seed=9)
        gw, gx, tb = rgnn.backward(layer, a, z, gout, mode="fused", assignment=asg)
        gwu, gxu, tbu = rgnn.backward(layer, a, z, gout, mode="unfused", assignment=asg)
        save(f"gnn_{kind}", adj_row_ptr=g.adjacency.row_ptr, adj_col_idx=g.adjacency.col_idx,
             **csr_arrays(a, "a_"), w=layer.weight.data, x=x.data, gout=gout.data,
             x_next=xn.data, z=z.data, x_next_unfused=xu.data, grad_w=gw.data, grad_x=gx.data,
             grad_w_unfused=gwu.data, grad_x_unfused=gxu.data, codes=asg.codes,
             traffic_fwd_fused=np.array(list(tf.as_dict().values())),
             traffic_fwd_unfused=np.array(list(tu.as_dict().values())),
             traffic_bwd_fused=np.array(list(tb.as_dict().values())),
             traffic_bwd_unfused=np.array(list(tbu.as_dict().values())))

    # ---- LOA (layout.py:186-263): corpus + communities + power law
    loa_cases = [(name, g, 128) for name, g in build_corpus()]
    for name, g, vw in loa_cases:
        grouping = rlay.build_windows_optimized(g, vw=vw)
        _, perm = rlay.reorder(g, grouping)
        flat = np.array([v for grp in grouping.groups for v in grp], dtype=np.int64)
        gptr = np.cumsum([0] + [len(grp) for grp in grouping.groups]).astype(np.int64)
        save(f"loa_corpus_{name}", n=np.array(g.num_vertices), row_ptr=g.adjacency.row_ptr,
             col_idx=g.adjacency.col_idx, vw=np.array(vw), order=rlay.sort_by_min_neighbor(g),
             flat=flat, gptr=gptr, perm=perm)
    extra = [("block64s", gg.block_pairs(64, 16, 0.6, 0.02, seed=9, scramble_seed=10), 128),
             ("block128s", gg.block_pairs(128, 16, 0.55, 0.004, seed=204, scramble_seed=4), 128),
             ("plaw3k", gg.power_law(3000, 12.0, seed=3), 128),
             ("plaw3k_vw16", gg.power_law(3000, 12.0, seed=3), 16),
             ("cora", gg.cora_shaped(seed=0), 128)]
    for name, (n, rr, cc), vw in extra:
        g = graph_of(n, rr, cc)
        grouping = rlay.build_windows_optimized(g, vw=vw)
        flat = np.array([v for grp in grouping.groups for v in grp], dtype=np.int64)
        gptr = np.cumsum([0] + [len(grp) for grp in grouping.groups]).astype(np.int64)
        _, perm = rlay.reorder(g, grouping)
        save(f"loa_{name}", n=np.array(n), row_ptr=g.adjacency.row_ptr, col_idx=g.adjacency.col_idx,
             vw=np.array(vw), order=rlay.sort_by_min_neighbor(g), flat=flat, gptr=gptr, perm=perm)


if __name__ == "__main__":
    main()
