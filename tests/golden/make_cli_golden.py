"""Golden run reports of the REFERENCE CLI (rowwin.cli.main) for the hot-path commands.

Usage (dev container only): PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_cli_golden.py
Writes tests/golden/cli/: the input files (Cora-shaped and block-community edge lists, a
Matrix Market file) and one JSON report per command, so tests/test_gpu_cli.py can run
the same command lines through paper_2412_08902_b200.cli on the GPU and compare metrics.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "cli")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, HERE)

from rowwin import cli as rcli  # noqa: E402

import gen_graphs as gg  # noqa: E402


def write_edges(path, n, rr, cc):
    keep = rr < cc  # one line per undirected edge
    with open(path, "w") as fh:
        fh.write("# synthetic graph\n")
        for u, v in zip(rr[keep].tolist(), cc[keep].tolist()):
            fh.write(f"{u} {v}\n")
        if n - 1 not in set(rr.tolist()) | set(cc.tolist()):
            pass


def run(argv, name):
    rep = os.path.join(OUT, name + ".json")
    code = rcli.main(argv + [] if argv[0].startswith("--") else argv)
    assert code == 0, (argv, code)
    return rep


def main():
    os.makedirs(OUT, exist_ok=True)
    n, rr, cc = gg.cora_shaped(seed=0)
    cora = os.path.join(OUT, "cora.edges")
    write_edges(cora, n, rr, cc)
    n2, r2, c2 = gg.block_pairs(64, 16, 0.6, 0.02, seed=9, scramble_seed=10)
    block = os.path.join(OUT, "block.edges")
    write_edges(block, n2, r2, c2)
    rel = lambda p: os.path.relpath(p, OUT)  # noqa: E731
    cases = {
        "partition_cora": ["partition-report", "--matrix", cora],
        "classify_cora": ["classify", "--matrix", cora],
        "spmm_hybrid_cora": ["spmm", "--matrix", cora, "--dense", "random:dim=32,seed=1"],
        "spmm_tile_cora": ["spmm", "--matrix", cora, "--dense", "random:dim=16,seed=2", "--mode", "tile"],
        "spmm_scalar_cora": ["spmm", "--matrix", cora, "--dense", "random:dim=8,seed=3", "--mode", "scalar"],
        "loa_block": ["loa", "--graph", block],
        "pipeline_block_loa": ["pipeline", "--graph", block, "--dim", "16", "--loa"],
        "pipeline_cora": ["pipeline", "--graph", cora, "--dim", "32"],
        "gnn_cora": ["gnn-bench", "--graph", cora, "--din", "32", "--dout", "16", "--repeats", "1"],
    }
    index = {}
    for name, argv in cases.items():
        rep = os.path.join(OUT, name + ".json")
        code = rcli.main(["--report-file", rep] + argv)
        assert code == 0, (name, code)
        index[name] = [a if not os.path.isabs(a) else rel(a) for a in argv]
        print(name, "ok")
    with open(os.path.join(OUT, "index.json"), "w") as fh:
        json.dump(index, fh, indent=2, sort_keys=True)


if __name__ == "__main__":
    main()
