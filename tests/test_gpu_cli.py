"""The command line (python -m paper_1501_03105_b200) on a BASELINE config
and on a graph file: runs, writes the trace CSV and the side, and its cut
values equal the oracle's."""
import csv
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from synthetic import generators as gen

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ready():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def run(*args):
    out = subprocess.run([sys.executable, "-m", "paper_1501_03105_b200", *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout)


def test_cli_config1(ready, tmp_path):
    trace = tmp_path / "trace.csv"
    r = run("--config", "1", "--T", "4", "--rounding", "both", "--exact", "--lambda2", "--trace", str(trace))
    S = oracle.Solver(oracle.Graph(gen.config1()), T=4, cg_rtol=1e-10, cg_max_iter=100000, cg_norm=1)
    _, reps = S.run(record=False)
    assert r["cg_iters"] == sum(x["cg_iters"] for x in reps)
    assert r["sweep"]["cut"] == S.sweep().cut_value
    assert r["two_level"]["cut"] == S.two_level().cut_value
    rows = list(csv.DictReader(open(trace)))
    assert len(rows) == 5 and [int(x["cg_iters"]) for x in rows] == [x["cg_iters"] for x in reps]
    assert float(rows[-1]["S_eps"]) == reps[-1]["S_eps"]
    assert r["mu_star"] <= r["two_level"]["cut"] <= r["sweep"]["cut"]


def test_cli_graph_file(ready, tmp_path):
    spec = gen.random_small_graph(300, 400, seed=5)
    path = tmp_path / "g.npz"
    np.savez(path, **spec)
    side_path = tmp_path / "side.npy"
    r = run("--graph", str(path), "--T", "6", "--rounding", "two_level", "--side", str(side_path))
    S = oracle.Solver(oracle.Graph(spec), T=6)
    S.run(record=False)
    tl = S.two_level()
    assert r["two_level"]["cut"] == tl.cut_value
    assert np.array_equal(np.load(side_path), tl.side)


def test_cli_virtual_ranks(tmp_path):
    """--virtual-ranks W runs the W-rank data path on one GPU: the same cut as
    the single-rank run."""
    import json
    import subprocess
    import sys
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    single = json.loads(subprocess.run([sys.executable, "-m", "paper_1501_03105_b200", "--config", "2", "--T", "10"],
                                       check=True, capture_output=True, text=True, cwd=root).stdout)
    multi = json.loads(subprocess.run([sys.executable, "-m", "paper_1501_03105_b200", "--config", "2", "--T", "10",
                                       "--virtual-ranks", "4", "--p2p"],
                                      check=True, capture_output=True, text=True, cwd=root).stdout)
    assert multi["cg_iters"] == single["cg_iters"]
    assert multi["sweep"]["cut"] == single["sweep"]["cut"] and multi["sweep"]["k"] == single["sweep"]["k"]
