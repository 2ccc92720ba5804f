"""GPU SpMM parity (K2/K3/K4) against the oracle and the reference's golden results.

Tolerances (BASELINE.json north_star): max_rel_err (tests/conftest.py:42-47 of the
reference: max|a-o| / max|o|) <= 1e-2 for bf16 inputs, against the exact fp64
product of the same inputs.  Integer outputs (stats) are exact.
"""

import numpy as np
import pytest
import torch

from conftest import golden_csr, golden_names, load_golden, plaw8k_csr
from oracle import rowwin_oracle as orc

import paper_2412_08902_b200 as hc
from paper_2412_08902_b200.executors import Assignment, Path

pytestmark = pytest.mark.gpu
BF16_TOL = 1e-2


def to_hc(csr):
    return hc.SparseCsr(csr.num_rows, csr.num_cols, csr.row_ptr, csr.col_idx, csr.values)


@pytest.mark.parametrize("name", [n for n in golden_names("windows_") if n != "windows_plaw8k"])
def test_hybrid_matches_reference(cuda_ok, name):
    g = load_golden(name)
    csr = golden_csr(g)
    x = orc.random_dense(csr.num_cols, int(g["dim"]), int(g["xseed"]))
    ws = hc.partition(to_hc(csr))
    asg = hc.classify_windows(hc.default_model(), ws)
    res = hc.spmm_hybrid(ws, asg, hc.DenseMatrix(x), precision="bf16")
    assert res.z.data.shape == (csr.num_rows, int(g["dim"]))
    assert orc.max_rel_err(res.z.data, g["z_f64"]) <= BF16_TOL
    assert orc.max_rel_err(res.z.data, g["z_f32"]) <= BF16_TOL
    for k, v in res.stats.as_dict().items():
        assert v == int(g["stats_" + k]), k


@pytest.mark.parametrize("name", ["windows_cora", "windows_corpus_block125", "windows_corpus_clique64",
                                  "windows_rand6", "windows_rand9"])
def test_all_tile_and_all_scalar(cuda_ok, name):
    g = load_golden(name)
    csr = golden_csr(g)
    x = orc.random_dense(csr.num_cols, int(g["dim"]), int(g["xseed"]))
    ws = hc.partition(to_hc(csr))
    t = hc.spmm_tile(ws, hc.DenseMatrix(x))
    assert orc.max_rel_err(t.z.data, g["z_f64"]) <= BF16_TOL
    s = hc.spmm_scalar(to_hc(csr), hc.DenseMatrix(x))
    assert orc.max_rel_err(s.z.data, g["z_f64"]) <= BF16_TOL
    live = int((ws.nnz_per_window() > 0).sum())
    assert t.stats.windows_tile == live and t.stats.entries_tile == csr.nnz
    assert s.stats.windows_scalar == live and s.stats.entries_scalar == csr.nnz
    # all-scalar hybrid == spmm_scalar (same kernel, same order): bitwise
    h = hc.spmm_hybrid(ws, Assignment.uniform(len(ws), Path.SCALAR), hc.DenseMatrix(x))
    assert np.array_equal(h.z.data, s.z.data)
    assert h.stats.as_dict() == s.stats.as_dict()


def test_plaw8k_mixed_paths(cuda_ok):
    g = load_golden("windows_plaw8k")
    a = plaw8k_csr()
    x = orc.random_dense(a.num_cols, 32, 1)
    ws = hc.partition(to_hc(a))
    asg = hc.classify_windows(hc.default_model(), ws)
    assert 0 < asg.count(Path.TILE) < len(asg)
    res = hc.spmm_hybrid(ws, asg, hc.DenseMatrix(x))
    assert orc.max_rel_err(res.z.data, g["z_f32"]) <= BF16_TOL
    for k, v in res.stats.as_dict().items():
        assert v == int(g["stats_" + k]), k


@pytest.mark.parametrize("dim", [1, 3, 8, 17, 32, 40, 64, 96, 128, 136, 256, 300])
def test_feature_dims(cuda_ok, dim):
    a = orc.random_csr(300, 700, 0.08, seed=dim)
    x = orc.random_dense(700, dim, seed=dim + 1)
    ws = hc.partition(to_hc(a))
    codes = np.random.default_rng(dim).integers(0, 2, size=len(ws)).astype(np.uint8)
    res = hc.spmm_hybrid(ws, Assignment(codes), hc.DenseMatrix(x))
    assert orc.max_rel_err(res.z.data, orc.spmm_exact(a, x)) <= BF16_TOL
    t = hc.spmm_tile(ws, hc.DenseMatrix(x))
    assert orc.max_rel_err(t.z.data, orc.spmm_exact(a, x)) <= BF16_TOL


def test_empty_windows_zero_and_uncounted(cuda_ok):
    # reference tests/test_executors.py:136-146
    csr = hc.SparseCsr.from_coo(48, 8, np.array([0, 35]), np.array([2, 3]), np.array([1.0, 1.0]))
    ws = hc.partition(csr)
    assert [w.nnz for w in ws] == [1, 0, 1]
    x = hc.DenseMatrix.random(8, 3, seed=1)
    res = hc.spmm_hybrid(ws, Assignment.uniform(3, Path.TILE), x)
    assert res.stats.windows_tile == 2
    assert np.array_equal(res.z.data[16:32], np.zeros((16, 3)))


def test_stats_tiles(cuda_ok):
    # reference tests/test_executors.py:110-120: 9 cols -> 2 tiles, 4 cols -> 1 tile
    rows = np.concatenate([np.zeros(9, dtype=np.int64), np.full(4, 16, dtype=np.int64)])
    cols = np.concatenate([np.arange(9), np.arange(4)]).astype(np.int64)
    csr = hc.SparseCsr.from_coo(32, 16, rows, cols, np.ones(13))
    res = hc.spmm_tile(hc.partition(csr), hc.DenseMatrix.random(16, 4, seed=0))
    assert res.stats.windows_tile == 2 and res.stats.entries_tile == 13 and res.stats.tiles_processed == 3


def test_validation_messages(cuda_ok):
    csr = to_hc(orc.random_csr(8, 10, 0.5, seed=0))
    ws = hc.partition(csr)
    with pytest.raises(ValueError, match="X has"):
        hc.spmm_tile(ws, hc.DenseMatrix.random(3, 2, seed=0))
    ws2 = hc.partition(to_hc(orc.random_csr(40, 10, 0.2, seed=1)))
    with pytest.raises(ValueError, match="assignment covers"):
        hc.spmm_hybrid(ws2, Assignment.uniform(1, Path.SCALAR), hc.DenseMatrix.random(10, 2, seed=0))


def test_deterministic_repeat(cuda_ok):
    a = plaw8k_csr()
    x = torch.rand(a.num_cols, 64, device="cuda").to(torch.bfloat16)
    ws = hc.partition(to_hc(a))
    asg = hc.classify_windows(hc.default_model(), ws)
    z1 = hc.spmm_hybrid(ws, asg, x).z.data.clone()
    z2 = hc.spmm_hybrid(ws, asg, x).z.data
    assert torch.equal(z1, z2)
    zt1 = hc.spmm_tile(ws, x).z.data.clone()
    assert torch.equal(zt1, hc.spmm_tile(ws, x).z.data)


def test_power_of_two_scaling_exact(cuda_ok):
    a = orc.random_csr(40, 30, 0.2, seed=20)
    d = orc.Csr(a.num_rows, a.num_cols, a.row_ptr, a.col_idx, a.values * 2.0)
    x = hc.DenseMatrix.random(30, 7, seed=21)
    z1 = hc.spmm_tile(hc.partition(to_hc(a)), x).z.data
    z2 = hc.spmm_tile(hc.partition(to_hc(d)), x).z.data
    assert np.array_equal(z1 * 2.0, z2)


def test_device_operands_and_auto(cuda_ok):
    a = orc.random_csr(500, 500, 0.05, seed=5)
    xd = torch.randn(500, 32, device="cuda", dtype=torch.bfloat16)
    res = hc.spmm_auto(to_hc(a), xd, lambda ws: hc.classify_windows(hc.default_model(), ws))
    assert isinstance(res.z.data, torch.Tensor) and res.z.data.is_cuda
    want = orc.spmm_exact(a, xd.float().cpu().numpy())
    assert orc.max_rel_err(res.z.data.cpu().numpy(), want) <= BF16_TOL


def test_large_powerlaw_tile_path_checksum(cuda_ok):
    """Size-independent property at ~6M nnz: Z summed over rows == (A^T 1)^T X in fp64."""
    from paper_2412_08902_b200 import graphgen

    g = graphgen.chung_lu_device(60000, 200.0, seed=3)
    a = graphgen.gcn_normalize_device(g)
    ws = hc.partition(a)
    x = torch.rand(a.num_rows, 128, device="cuda", generator=torch.Generator("cuda").manual_seed(1)) * 2 - 1
    xb = x.to(torch.bfloat16)
    res = hc.spmm_hybrid(ws, hc.classify_windows(hc.default_model(), ws), xb)
    colsum = torch.zeros(a.num_cols, dtype=torch.float64, device="cuda")
    colsum.index_add_(0, a.col_idx.long(), a.values.double())
    want = colsum @ xb.double()
    got = res.z.data.double().sum(0)
    assert float((got - want).abs().max() / want.abs().max()) <= 1e-3
    # row spot-check against exact fp64 on 200 random rows
    rows = torch.randint(0, a.num_rows, (200,), generator=torch.Generator().manual_seed(0))
    rp = a.row_ptr.cpu()
    for r in rows.tolist()[:50]:
        lo, hi = int(rp[r]), int(rp[r + 1])
        cols = a.col_idx[lo:hi].long()
        exact = (a.values[lo:hi].double()[:, None] * xb[cols].double()).sum(0)
        scale = float(res.z.data.double().abs().max())
        assert float((res.z.data[r].double() - exact).abs().max()) / scale <= BF16_TOL


@pytest.mark.parametrize("precision", ["bf16", "tf32"])
@pytest.mark.parametrize("dim", [8, 32, 40, 64, 128, 200])
def test_tile_path_dims(cuda_ok, precision, dim):
    """The tile path (every window on the tensor cores) against the exact product."""
    a = plaw8k_csr()
    x = orc.random_dense(a.num_cols, dim, seed=dim)
    ws = hc.partition(to_hc(a))
    res = hc.spmm_tile(ws, hc.DenseMatrix(x), precision=precision)
    assert orc.max_rel_err(res.z.data, orc.spmm_exact(a, x)) <= (BF16_TOL if precision == "bf16" else 1e-3)


@pytest.mark.parametrize("vectors", [4, 8])
@pytest.mark.parametrize("dim", [8, 32, 41, 64, 96, 128, 200])
def test_warp_kernel_slice_widths(cuda_ok, vectors, dim):
    """Engine 2 with 32- and 64-feature row slices; deterministic across repeats."""
    from paper_2412_08902_b200 import _lib

    a = plaw8k_csr()
    x = orc.random_dense(a.num_cols, dim, seed=dim + 1)
    ws = hc.partition(to_hc(a))
    try:
        _lib.call("hcs_set_tile_slice", vectors)
        r1 = hc.spmm_tile(ws, hc.DenseMatrix(x))
        r2 = hc.spmm_tile(ws, hc.DenseMatrix(x))
    finally:
        _lib.call("hcs_set_tile_slice", 0)
    assert orc.max_rel_err(r1.z.data, orc.spmm_exact(a, x)) <= BF16_TOL
    assert np.array_equal(r1.z.data, r2.z.data)


TF32_TOL = 1e-3


@pytest.mark.parametrize("name", ["windows_cora", "windows_corpus_block125", "windows_corpus_clique64", "windows_rand6",
                                  "windows_rand9", "windows_corpus_star256"])
def test_tf32_matches_reference(cuda_ok, name):
    """precision='tf32' (RNA-rounded tf32 tensor-core inputs, fp32 accumulate): <= 1e-3 vs the
    reference's f32 / exact results (BASELINE north_star)."""
    g = load_golden(name)
    csr = golden_csr(g)
    x = orc.random_dense(csr.num_cols, int(g["dim"]), int(g["xseed"]))
    ws = hc.partition(to_hc(csr))
    asg = hc.classify_windows(hc.default_model(), ws)
    res = hc.spmm_hybrid(ws, asg, hc.DenseMatrix(x), precision="tf32")
    assert orc.max_rel_err(res.z.data, g["z_f64"]) <= TF32_TOL
    assert orc.max_rel_err(res.z.data, g["z_f32"]) <= TF32_TOL
    t = hc.spmm_tile(ws, hc.DenseMatrix(x), precision="tf32")
    assert orc.max_rel_err(t.z.data, g["z_f64"]) <= TF32_TOL


@pytest.mark.parametrize("dim", [1, 5, 32, 41, 64, 128, 200])
def test_tf32_tile_dims_plaw(cuda_ok, dim):
    a = plaw8k_csr()
    x = orc.random_dense(a.num_cols, dim, seed=dim + 3)
    ws = hc.partition(to_hc(a))
    r1 = hc.spmm_tile(ws, hc.DenseMatrix(x), precision="tf32")
    r2 = hc.spmm_tile(ws, hc.DenseMatrix(x), precision="tf32")
    assert orc.max_rel_err(r1.z.data, orc.spmm_exact(a, x)) <= TF32_TOL
    assert np.array_equal(r1.z.data, r2.z.data)


def test_host_pipelined_path(cuda_ok):
    """Host inputs with >= 4096 windows: partial launches with D2H overlapped; same result
    (to fp32 summation order) as the device-resident path and the exact product."""
    import gen_graphs as gg
    from paper_2412_08902_b200 import executors as ex

    n, rr, cc = gg.power_law(70000, 24.0, seed=5)
    adj = orc.from_coo(n, n, rr, cc, np.ones(len(rr)))
    a = orc.normalize_adj(adj, "gcn")
    ws = hc.partition(to_hc(a))
    assert len(ws) >= ex.HOST_PIPELINE_MIN_WINDOWS
    asg = hc.classify_windows(hc.default_model(), ws)
    x = orc.random_dense(n, 64, seed=2)
    host = hc.spmm_hybrid(ws, asg, hc.DenseMatrix(x))            # numpy in -> numpy out (pipelined)
    xt = torch.from_numpy(x).to(torch.bfloat16).cuda()
    dev = hc.spmm_hybrid(ws, asg, xt)                            # device in -> device out
    assert isinstance(host.z.data, np.ndarray)
    d = dev.z.data.cpu().numpy()
    assert np.abs(host.z.data - d).max() <= 1e-5 * np.abs(d).max()
    assert orc.max_rel_err(host.z.data, orc.spmm_exact(a, x)) <= BF16_TOL
    assert host.stats == dev.stats
    # the float64 operand (4.5 M elements) took the pipelined host staging path (host threads
    # convert blocks into pinned bf16 while the previous block uploads): the staged operand is
    # torch's own cast bit for bit, for bf16 and for the tf32 path's fp32 + RNA rounding
    assert x.size >= ex.HOST_STAGE_MIN_ELEMS
    for prec, want in (("bf16", torch.bfloat16), ("tf32", torch.float32)):
        op, was_host = ex.stage_operand(hc.DenseMatrix(x), prec, xt.device, tf32_round=prec == "tf32")
        assert was_host
        ref = torch.from_numpy(x).to(want).cuda()
        if prec == "tf32":
            rnd = torch.empty_like(ref)
            from paper_2412_08902_b200 import _lib

            _lib.call("hcs_convert", ref.data_ptr(), rnd.data_ptr(), ref.numel(), 0, _lib.stream())
            ref = rnd
        assert torch.equal(op.t[:, : x.shape[1]], ref)
        assert not op.t[:, x.shape[1]:].any()


@pytest.mark.parametrize("big", [False, True])
def test_async_requests_match_sync(cuda_ok, big):
    """spmm_hybrid_async with three requests in flight (different X each, pinned torch and
    numpy inputs) returns what spmm_hybrid returns for each of them: bit for bit when the
    product runs as one launch, to fp32 summation order when it runs in row ranges (the async
    path uses fewer, larger ranges than the synchronous one, so warp-range cuts differ)."""
    import gen_graphs as gg

    n, rr, cc = gg.power_law(70000 if big else 3000, 24.0, seed=5)
    adj = orc.from_coo(n, n, rr, cc, np.ones(len(rr)))
    a = orc.normalize_adj(adj, "gcn")
    ws = hc.partition(to_hc(a))
    asg = hc.classify_windows(hc.default_model(), ws)
    xs = [orc.random_dense(n, d, seed=10 + i) for i, d in enumerate((64, 128, 40))]
    ins = [hc.DenseMatrix(xs[0]), torch.from_numpy(xs[1]).to(torch.bfloat16).pin_memory(),
           torch.from_numpy(xs[2]).float()]
    reqs = [hc.spmm_hybrid_async(ws, asg, x) for x in ins]
    got = [r.result() for r in reqs]
    def same(gz, wz):
        if big:
            return np.abs(gz - wz).max() <= 1e-5 * np.abs(wz).max()
        return np.array_equal(gz, wz)

    rows_tile = np.repeat(asg.codes, ws.window_height)[:n] == 1

    def diag(gz, wz):
        bad = np.nonzero(np.abs(gz - wz).max(1))[0]
        rl = np.diff(a.row_ptr)[bad]
        return (f"{bad.size} rows differ ({int(rows_tile[bad].sum())} on tile windows), first {bad[:8].tolist()}, "
                f"row lengths {rl[:8].tolist()}, max diff {float(np.abs(gz - wz).max())}")

    for x, g in zip(ins, got):
        want = hc.spmm_hybrid(ws, asg, x)
        assert type(g.z.data) is type(want.z.data)
        gz = g.z.data if isinstance(g.z.data, np.ndarray) else g.z.data.numpy()
        wz = want.z.data if isinstance(want.z.data, np.ndarray) else want.z.data.numpy()
        assert same(gz, wz), diag(gz, wz)
        assert g.stats == want.stats
    assert orc.max_rel_err(got[0].z.data, orc.spmm_exact(a, xs[0])) <= BF16_TOL
    # caller-owned pinned result buffers (a ring of two, three requests)
    ring = [torch.full((n + 3, 130), float("nan")).pin_memory() for _ in range(2)]
    reqs = [hc.spmm_hybrid_async(ws, asg, ins[1], out=ring[0]), hc.spmm_hybrid_async(ws, asg, ins[2], out=ring[1])]
    z1 = reqs[0].result().z.data.clone()
    reqs.append(hc.spmm_hybrid_async(ws, asg, ins[0], out=ring[0]))
    z2, z0 = reqs[1].result().z.data, reqs[2].result().z.data
    as_np = lambda v: v if isinstance(v, np.ndarray) else v.numpy()  # noqa: E731
    for gz, x in ((z1, ins[1]), (z2, ins[2]), (z0, ins[0])):
        assert same(as_np(gz), as_np(hc.spmm_hybrid(ws, asg, x).z.data))
    with pytest.raises(ValueError, match="out must be"):
        hc.spmm_hybrid_async(ws, asg, ins[1], out=torch.empty(n, 8))
    with pytest.raises(ValueError, match="host operand"):
        hc.spmm_hybrid_async(ws, asg, torch.zeros(n, 8, device="cuda"))


@pytest.mark.parametrize("variant", ["auto", "warp", "rows", "block", "warp16"])
@pytest.mark.parametrize("precision", ["bf16", "tf32"])
def test_scalar_variants(cuda_ok, variant, precision):
    """Every K3 kernel variant == the exact product within the precision's tolerance, on
    windows below and above the shared-memory staging cap (256 entries), short last
    windows, odd window heights and dims that are not multiples of the vector width;
    run-to-run bitwise identical."""
    from paper_2412_08902_b200.executors import set_scalar_variant

    tol = BF16_TOL if precision == "bf16" else 1e-3
    rng = np.random.default_rng(7)
    # rows 0..159: 1-8 nnz; rows 160..239: 40-90 nnz (windows over the cap); 245 rows total;
    # a few hub rows of 250-400 nnz (several 32-entry batches in the rows kernel)
    rows, cols = [], []
    for r in range(245):
        k = int(rng.integers(1, 9)) if r < 160 else int(rng.integers(40, 90))
        if r % 41 == 3:
            k = int(rng.integers(250, 400))
        if r % 37 == 5:
            k = 0  # empty rows
        cs = rng.choice(900, size=k, replace=False)
        rows += [r] * k
        cols += list(cs)
    a = orc.from_coo(245, 900, rows, cols, rng.uniform(-1, 1, len(rows)))
    try:
        set_scalar_variant(variant)
        for wh in (16, 7):
            for dim in (1, 24, 64, 100, 128, 200):
                x = orc.random_dense(900, dim, seed=dim)
                ws = hc.partition(to_hc(a), window_height=wh)
                asg = Assignment.uniform(len(ws), Path.SCALAR)
                r1 = hc.spmm_hybrid(ws, asg, hc.DenseMatrix(x), precision=precision)
                exact = orc.spmm_exact(a, x)
                assert orc.max_rel_err(r1.z.data, exact) <= tol, (wh, dim)
                r2 = hc.spmm_hybrid(ws, asg, hc.DenseMatrix(x), precision=precision)
                assert np.array_equal(r1.z.data, r2.z.data)
    finally:
        set_scalar_variant("auto")


@pytest.mark.parametrize("dim", [72, 128, 256])
def test_tile_slice_pairing(cuda_ok, dim):
    """Paired feature slices (sibling warps walk one (window, chunk) range, a slice each) ==
    the exact product within tolerance, run-to-run bitwise, and == the unpaired schedule up to
    the fp32 rounding of different cut points; windows cut by ranges are exercised (plaw8k has
    ~46 K chunks for 1,184 warps)."""
    from paper_2412_08902_b200 import _lib

    a = plaw8k_csr()
    x = orc.random_dense(a.num_cols, dim, 5)
    ws = hc.partition(to_hc(a))
    exact = orc.spmm_exact(a, x)
    out = {}
    try:
        for mode in (0, 1):
            _lib.call("hcs_set_tile_pairing", mode)
            r1 = hc.spmm_tile(ws, hc.DenseMatrix(x))
            r2 = hc.spmm_tile(ws, hc.DenseMatrix(x))
            assert np.array_equal(r1.z.data, r2.z.data)
            assert orc.max_rel_err(r1.z.data, exact) <= BF16_TOL
            out[mode] = r1.z.data
    finally:
        _lib.call("hcs_set_tile_pairing", 1)
    assert orc.max_rel_err(out[1], out[0]) <= 1e-4


@pytest.mark.parametrize("precision", ["bf16", "tf32"])
def test_plan_builders_identical(cuda_ok, precision):
    """K2: the per-window bucketing builder (default) and the global radix-sort builder give
    identical plans (gidx, ent_ptr, packed entries), incl. a window with > 3,072 chunks
    (several bucketing passes) and a short last window."""
    from paper_2412_08902_b200 import _lib
    from paper_2412_08902_b200.executors import HybridPlan

    rng = np.random.default_rng(11)
    rows, cols = [], []
    for r in range(16):  # one very wide window: ~222 K condensed columns
        cs = rng.choice(250_000, size=32_000, replace=False)
        rows += [r] * len(cs)
        cols += list(cs)
    for r in range(16, 16 + 37):  # narrower windows, the last one short
        cs = rng.choice(250_000, size=int(rng.integers(1, 3000)), replace=False)
        rows += [r] * len(cs)
        cols += list(cs)
    a = orc.from_coo(53, 250_000, rows, cols, rng.uniform(-1, 1, len(rows)))
    ws = hc.partition(to_hc(a))
    codes = torch.ones(len(ws), dtype=torch.uint8, device="cuda")
    plans = []
    try:
        for builder in (0, 1):
            _lib.call("hcs_set_tile_plan_builder", builder)
            plans.append(HybridPlan(ws, codes, precision))
    finally:
        _lib.call("hcs_set_tile_plan_builder", 0)
    p0, p1 = plans
    assert int(p0.chunk_ptr[1] - p0.chunk_ptr[0]) > 3072
    assert torch.equal(p0.gidx, p1.gidx)
    assert torch.equal(p0.ent_ptr, p1.ent_ptr)
    assert torch.equal(p0.ent, p1.ent)


@pytest.mark.parametrize("shape", ["no_rows", "no_entries", "one_row", "ragged_17", "one_col"])
def test_degenerate_shapes(cuda_ok, shape):
    """Empty and ragged inputs on every path (reference executors.py:216-272 semantics: Z has
    total_rows(windows) rows, untouched rows are zero, stats count only non-empty windows)."""
    n, m = {"no_rows": (0, 5), "no_entries": (40, 7), "one_row": (1, 9), "ragged_17": (17, 30),
            "one_col": (33, 1)}[shape]
    rng = np.random.default_rng(3)
    if shape in ("no_rows", "no_entries"):
        rows, cols = [], []
    else:
        rows = list(rng.integers(0, n, size=3 * n))
        cols = list(rng.integers(0, m, size=3 * n))
    a = orc.from_coo(n, m, rows, cols, rng.uniform(-1, 1, len(rows)))
    x = orc.random_dense(m, 6, 4)
    exact = orc.spmm_exact(a, x)
    ws = hc.partition(to_hc(a))
    assert len(ws) == -(-n // 16)
    asg = hc.classify_windows(hc.default_model(), ws)
    for res in (hc.spmm_hybrid(ws, asg, hc.DenseMatrix(x)), hc.spmm_tile(ws, hc.DenseMatrix(x)),
                hc.spmm_scalar(to_hc(a), hc.DenseMatrix(x)),
                hc.spmm_hybrid(ws, asg, hc.DenseMatrix(x), precision="tf32")):
        z = np.asarray(res.z.data)
        assert z.shape == (n, 6)
        if n:
            assert orc.max_rel_err(z, exact) <= BF16_TOL if np.abs(exact).max() > 0 else not z.any()
        live = int((ws.nnz_per_window() > 0).sum()) if n else 0
        s = res.stats
        assert s.windows_scalar + s.windows_tile == live
        assert s.entries_scalar + s.entries_tile == a.nnz


@pytest.mark.parametrize("precision", ["bf16", "tf32"])
def test_spmm_graph_replay(cuda_ok, precision):
    """SpmmGraph (one CUDA-graph launch per product) == spmm_hybrid bit for bit, and replays
    pick up in-place updates of X."""
    a = plaw8k_csr()
    ws = hc.partition(to_hc(a))
    asg = hc.classify_windows(hc.default_model(), ws)
    dt = torch.bfloat16 if precision == "bf16" else torch.float32
    x = torch.from_numpy(orc.random_dense(a.num_cols, 64, 2)).to("cuda", dt)
    g = hc.SpmmGraph(ws, asg, x, precision=precision)
    z1 = g.replay().clone()
    ref = hc.spmm_hybrid(ws, asg, x, precision=precision).z.data
    assert torch.equal(z1, ref)
    if precision == "bf16":  # operand used in place: replay sees the new X
        x.mul_(2)
        z2 = g.replay()
        bad = torch.nonzero((z2 - 2 * z1).abs().amax(1)).flatten().cpu().numpy()
        rows_tile = np.repeat(asg.codes, ws.window_height)[:a.num_rows] == 1
        assert torch.equal(z2, 2 * z1), (f"{bad.size} rows differ ({int(rows_tile[bad].sum())} tile), first "
                                         f"{bad[:8].tolist()}, row lengths {np.diff(a.row_ptr)[bad[:8]].tolist()}")
    with pytest.raises(ValueError, match="CUDA tensor"):
        hc.SpmmGraph(ws, asg, x.cpu())





@pytest.mark.parametrize("precision,dim", [("bf16", 520), ("bf16", 1000), ("tf32", 300), ("tf32", 7)])
def test_scalar_pieces_wide_rows_and_hubs(cuda_ok, precision, dim):
    """The small-plan K3 piece kernel with feature rows wider than one warp covers (several
    32-vector chunks per piece: bf16 N > 512, fp32 N > 256) and hub rows split into many pieces:
    == the exact product within tolerance, bitwise run-to-run, and == spmm_scalar."""
    rng = np.random.default_rng(11)
    n, m = 100, 2000
    rows, cols = [], []
    for r in range(n):
        k = 700 if r in (3, 50) else int(rng.integers(0, 40))
        rows += [r] * k
        cols += list(rng.choice(m, size=k, replace=False))
    a = orc.from_coo(n, m, rows, cols, rng.uniform(-1, 1, len(rows)))
    x = orc.random_dense(m, dim, seed=5)
    ws = hc.partition(to_hc(a))
    asg = Assignment.uniform(len(ws), Path.SCALAR)
    r1 = hc.spmm_hybrid(ws, asg, hc.DenseMatrix(x), precision=precision).z.data
    r2 = hc.spmm_hybrid(ws, asg, hc.DenseMatrix(x), precision=precision).z.data
    assert np.array_equal(r1, r2)
    tol = BF16_TOL if precision == "bf16" else 1e-3
    assert orc.max_rel_err(r1, orc.spmm_exact(a, x)) <= tol
    s = hc.spmm_scalar(to_hc(a), hc.DenseMatrix(x), precision=precision).z.data
    assert np.array_equal(r1, s)


def test_tile_balanced_ranges_on_skewed_plan(cuda_ok):
    """A skewed plan (hub windows whose 64-column chunks hold up to 1,024 entries, plus enough
    ordinary windows for the weighted split to apply): HybridPlan picks cost-weighted warp
    ranges (hcs_spmm_tile_balanced, k_tile_bounds); the product == the exact one within the bf16
    tolerance, bitwise run to run, and == the uniform-range product to fp32 summation order."""
    rng = np.random.default_rng(21)
    n, m, dim = 16 * 6000, 30000, 128
    hub_cols = rng.choice(m, size=300, replace=False)
    rows, cols = [], []
    for w in range(n // 16):
        for r in range(16 * w, 16 * w + 16):
            if w % 40 == 0:  # hub window: every row on the same 300 columns
                c = hub_cols
            else:
                c = rng.choice(m, size=int(rng.integers(8, 24)), replace=False)
            rows += [r] * len(c)
            cols += list(c)
    a = orc.from_coo(n, m, rows, cols, rng.uniform(-1, 1, len(rows)))
    ws = hc.partition(to_hc(a))
    asg = Assignment.uniform(len(ws), Path.TILE)
    from paper_2412_08902_b200.executors import get_plan

    plan = get_plan(ws, asg, "bf16")
    assert plan.tile_alpha > 0  # chunks above 128 entries were detected
    x = orc.random_dense(m, dim, seed=8)
    xt = torch.from_numpy(x).to(torch.bfloat16).cuda()
    r1 = hc.spmm_hybrid(ws, asg, xt).z.data.clone()
    r2 = hc.spmm_hybrid(ws, asg, xt).z.data.clone()
    assert torch.equal(r1, r2)
    exact = orc.spmm_exact(a, xt.float().cpu().numpy().astype(np.float64))
    assert orc.max_rel_err(r1.cpu().numpy(), exact) <= BF16_TOL
    alpha, plan.tile_alpha = plan.tile_alpha, 0
    try:
        r0 = hc.spmm_hybrid(ws, asg, xt).z.data.clone()
    finally:
        plan.tile_alpha = alpha
    assert orc.max_rel_err(r1.cpu().numpy(), r0.cpu().numpy().astype(np.float64)) <= 1e-5
    # small grids: few warp groups, many windows cut by weighted bounds (split owners found by
    # binary search over the bounds), every paired / single-slice width
    from paper_2412_08902_b200 import _lib

    for ctas in (1, 4, 37):
        _lib.call("hcs_set_tile_grid", ctas)
        try:
            for d in (128, 64, 41):
                xd = torch.from_numpy(x[:, :d].copy()).to(torch.bfloat16).cuda()
                ex = orc.spmm_exact(a, xd.float().cpu().numpy().astype(np.float64))
                za = hc.spmm_hybrid(ws, asg, xd).z.data.clone()
                zb = hc.spmm_hybrid(ws, asg, xd).z.data
                assert torch.equal(za, zb), (ctas, d)
                assert orc.max_rel_err(za.cpu().numpy(), ex) <= BF16_TOL, (ctas, d)
        finally:
            _lib.call("hcs_set_tile_grid", 0)


def test_plain_tile_entry_point_matches_plan(cuda_ok):
    """hcs_spmm_tile (the C-ABI entry INTEGRATION.md binds; HybridPlan launches its
    hcs_spmm_tile_balanced superset) on a plan's arrays == the plan's own tile launch, bitwise,
    when neither weighting nor grid sizing changes the warp ranges."""
    from paper_2412_08902_b200 import _lib
    from paper_2412_08902_b200.executors import get_plan, stage_operand, _alloc_z

    a = plaw8k_csr()
    ws = hc.partition(to_hc(a))
    asg = Assignment.uniform(len(ws), Path.TILE)
    plan = get_plan(ws, asg, "bf16")
    assert plan.tile_alpha == 0
    groups = torch.cuda.get_device_properties(0).multi_processor_count * 4  # 8 warps, paired slices
    assert plan.nchunks >= groups  # the plan's launch keeps the full grid
    x = orc.random_dense(a.num_cols, 128, seed=6)
    xop, _ = stage_operand(x, "bf16", torch.device("cuda"))
    z1, ldz = _alloc_z(a.num_rows, 128, torch.device("cuda"))
    z2, _ = _alloc_z(a.num_rows, 128, torch.device("cuda"))
    plan.run(xop, z1, ldz)
    scr = plan.new_scratch()
    _lib.call("hcs_spmm_tile", plan.tile_list.data_ptr(), plan.n_tile, plan.chunk_ptr.data_ptr(), plan.gidx.data_ptr(),
              plan.ent_ptr.data_ptr(), plan.ent.data_ptr(), plan.ent_dtype, a.num_rows, ws.window_height,
              xop.t.data_ptr(), xop.dtype_code, xop.rows, xop.dim, xop.ld, z2.data_ptr(), ldz, scr.data_ptr(),
              scr.numel() * 4, _lib.stream())
    torch.cuda.synchronize()
    assert torch.equal(z1[:, :128], z2[:, :128])


def test_tile_grid_setter(cuda_ok):
    """hcs_set_tile_grid (SMs left to the NCCL kernels of the multi-GPU exchange): any CTA count gives
    the product to fp32 summation order (different warp ranges), deterministic per grid; the
    fused GCN epilogue too; 0 restores one CTA per SM."""
    from paper_2412_08902_b200 import _lib, gnn

    a = plaw8k_csr()
    ws = hc.partition(to_hc(a))
    asg = hc.classify_windows(hc.default_model(), ws)
    x = torch.from_numpy(orc.random_dense(a.num_cols, 128, 3)).to(torch.bfloat16).cuda()
    z0 = hc.spmm_hybrid(ws, asg, x).z.data.clone()
    layer = gnn.GnnLayer.random(128, 64, seed=1)
    f0, _, _ = gnn.forward(layer, ws, x.float(), mode="fused", assignment=asg, windows=ws)
    try:
        for ctas in (1, 37, 132):
            _lib.call("hcs_set_tile_grid", ctas)
            z1 = hc.spmm_hybrid(ws, asg, x).z.data
            z2 = hc.spmm_hybrid(ws, asg, x).z.data
            assert torch.equal(z1, z2)
            assert float((z1 - z0).abs().max() / z0.abs().max()) <= 1e-5
            f1, _, _ = gnn.forward(layer, ws, x.float(), mode="fused", assignment=asg, windows=ws)
            assert float((f1.data - f0.data).abs().max() / f0.data.abs().max()) <= 1e-2
    finally:
        _lib.call("hcs_set_tile_grid", 0)
    assert torch.equal(hc.spmm_hybrid(ws, asg, x).z.data, z0)
