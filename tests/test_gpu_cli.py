"""The reference CLI's hot-path commands (rowwin.cli: spmm, partition-report, classify, loa,
gnn-bench, pipeline) run through paper_2412_08902_b200.cli on the GPU with the same
command lines as the golden reports of tests/golden/make_cli_golden.py: integer metrics and
the features-derived means are exact; checksums agree within the bf16 tolerance."""

import json
import os

import pytest

from conftest import GOLDEN

from paper_2412_08902_b200 import cli

pytestmark = pytest.mark.gpu
CLI_DIR = os.path.join(GOLDEN, "cli")
with open(os.path.join(CLI_DIR, "index.json")) as fh:
    CASES = json.load(fh)

EXACT_FLOAT = {"mean_density", "mean_ci", "mean_ci_before", "mean_ci_after"}


def _argv(name):
    return [os.path.join(CLI_DIR, a) if a.endswith((".edges", ".mtx")) else a for a in CASES[name]]


@pytest.mark.parametrize("name", sorted(CASES))
def test_cli_matches_reference_report(cuda_ok, name, tmp_path):
    with open(os.path.join(CLI_DIR, name + ".json")) as fh:
        ref = json.load(fh)
    out = tmp_path / "report.json"
    assert cli.main(["--report-file", str(out)] + _argv(name)) == 0
    got = json.loads(out.read_text())
    assert got["command"] == ref["command"]
    assert set(got["metrics"]) == set(ref["metrics"])
    for k, v in ref["metrics"].items():
        g = got["metrics"][k]
        if k == "checksum":
            n_el = ref["metrics"].get("rows", ref["metrics"].get("num_vertices", 1)) * ref["metrics"].get("dim", 32)
            assert abs(g - v) <= 1e-3 * n_el, (k, g, v)
        elif k == "max_rel_diff":
            assert g <= 1e-2
        elif k in EXACT_FLOAT:
            assert g == pytest.approx(v, rel=1e-12, abs=0), k
        else:
            assert g == v, k
