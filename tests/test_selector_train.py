"""CPU: the selector-training restatement (selector_train.py) against the reference's own
generate_synthetic / default_grid / holdout_split / train outputs (tests/golden/selector_train.npz,
made by tests/golden/make_selector_golden.py from /root/reference selector.py:67-242).
GPU: the B200 timing provider and the train-selector CLI."""

import json
import os

import numpy as np
import pytest

from paper_2412_08902_b200 import selector_train as T

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "selector_train.npz"))


def golden_samples():
    return [T.TrainingSample.from_timings(int(a), float(b), float(c), float(d))
            for a, b, c, d in zip(G["s_ncols"], G["s_density"], G["s_ts"], G["s_tt"])]


def test_grid_matches_reference():
    assert np.array_equal(np.array(T.default_grid(), dtype=np.int64), G["grid"])
    assert len(T.dense_grid()) == 130 * 8 * 5
    assert all(nc <= nnz <= 15 * nc for nc, nnz, _ in T.b200_grid())


def test_generate_synthetic_matches_reference():
    keys = [k for k in G.files if k.startswith("syn_") and k.endswith("_ptr")]
    assert len(keys) > 5
    for k in keys:
        nc, nnz, sd = map(int, k.split("_")[1:4])
        w = T.generate_synthetic(nc, nnz, sd)
        assert np.array_equal(w.local_ptr, G[k]), k
        assert np.array_equal(w.cond_cols, G[k.replace("_ptr", "_cols")]), k
        assert w.nnz == nnz and len(np.unique(w.cond_cols)) == nc


def test_generate_synthetic_errors():
    with pytest.raises(ValueError, match="ncols"):
        T.generate_synthetic(131, 200, 0)
    with pytest.raises(ValueError, match="nnz"):
        T.generate_synthetic(4, 61, 0)
    w = T.generate_synthetic(4096, 5000, 3, max_ncols=8192)
    assert w.ncols == 4096 and w.nnz == 5000


def test_train_bit_exact_with_reference():
    s = golden_samples()
    assert [x.label for x in s] == list(G["s_label"])
    tr, ho = T.holdout_split(s, frac=0.25, seed=0)
    assert [s.index(x) for x in tr] == list(G["train_idx"])
    m = T.train(tr, seed=0)
    got = np.array([m.w_ncols, m.w_density, m.bias, *m.feature_means, *m.feature_scales])
    assert np.array_equal(got, G["model"])  # same float operations -> same bits
    assert [T.accuracy(m, tr), T.accuracy(m, ho)] == list(G["acc"])


def test_train_errors():
    with pytest.raises(ValueError, match="no training samples"):
        T.train([])
    with pytest.raises(ValueError, match="single class"):
        T.train([T.TrainingSample.from_timings(4, 0.5, 1.0, 2.0)] * 3)
    with pytest.raises(ValueError, match="frac"):
        T.holdout_split(golden_samples(), frac=1.0)


@pytest.mark.gpu
def test_b200_provider_and_cli(cuda_ok, tmp_path):
    from paper_2412_08902_b200 import cli
    from paper_2412_08902_b200.selector import load_model

    prov = T.B200Provider(min_nnz=200_000, reps=3)
    w = T.generate_synthetic(64, 300, 1)
    ts, tt = prov(w, 32)
    assert ts > 0 and tt > 0
    # the batch matrix holds `batch` copies of the pattern with distinct columns per row
    csr = prov.batch_matrix(w, 8)
    assert csr.nnz == 8 * 300 and csr.num_rows == 128
    rp = csr.row_ptr.cpu().numpy()
    assert np.array_equal(np.diff(rp[:17]), np.diff(w.local_ptr))
    out = tmp_path / "m.json"
    rc = cli.main(["--report-file", str(tmp_path / "r.json"), "train-selector", "--grid", "b200", "--dim", "32",
                   "--repeats", "2", "--out", str(out)])
    if rc == 2:  # every grid window faster on one path -> the reference's single-class error
        pytest.skip("B200 timings gave a single class on this grid")
    assert rc == 0
    rep = json.loads((tmp_path / "r.json").read_text())
    assert rep["metrics"]["n_samples"] == len(T.b200_grid())
    m = load_model(str(out))
    assert np.isfinite([m.w_ncols, m.w_density, m.bias]).all()


def test_b200_model_is_opt_in():
    import paper_2412_08902_b200 as hc

    m, d = hc.b200_model(), hc.default_model()
    assert m != d
    # the shipped reference model is still the default; the B200 model prefers TILE for wide windows
    assert m.decide(512, 0.07).value == "tile"
    assert m.decide(0, 0.0).value == "scalar"
