"""CLI end to end on the device (spmv / solve / bench on a generated
container) and the device container loader against the host path."""

import csv
import os

import numpy as np
import pytest
import torch

import paper_1905_06234_b200 as L
from paper_1905_06234_b200 import cli, io

from conftest import GOLDEN, rel_l2

pytestmark = pytest.mark.gpu


def _container(tmp_path):
    d = L.Dims(n_atoms=40, n_voxels=300, n_fibers=200, n_dirs=96, n_coeffs=20000)
    p = L.generate(L.GenConfig(dims=d, mean_run_length=60.0, weight_density=0.5,
                               noise_sigma=0.1, seed=0))
    path = str(tmp_path / "p.life")
    io.save(p, path)
    return path, io.load(path)


def test_spmv_solve_bench(tmp_path, capsys):
    life, p = _container(tmp_path)
    rep = str(tmp_path / "spmv.csv")
    assert cli.main(["spmv", "--in", life, "--op", "dsc", "--restructure", "voxel", "--partition",
                     "coeff", "--sync-free", "--threads", "4", "--repeat", "3", "--report", rep]) == 0
    rows = io.read_report(rep)
    assert [r.iteration for r in rows] == [1, 2, 3] and all(r.partition == "coeff+syncfree" for r in rows)
    assert all(r.elapsed_s > 0 and r.threads == 4 for r in rows)
    assert cli.main(["spmv", "--in", life, "--op", "wc", "--restructure", "auto", "--repeat", "1"]) == 0
    assert "autotune picked" in capsys.readouterr().out
    tr, wout = str(tmp_path / "trace.csv"), str(tmp_path / "w.txt")
    assert cli.main(["solve", "--in", life, "--iters", "6", "--grad-tol", "0", "--trace", tr,
                     "--out-weights", wout]) == 0
    with open(tr) as f:
        rows = list(csv.reader(f))
    assert tuple(rows[0]) == cli.TRACE_COLUMNS and len(rows) == 7
    w = np.loadtxt(wout)
    w_ref, _ = L.solve(p, config=L.SolverConfig(max_iters=6, grad_tol=0.0))
    assert rel_l2(w, w_ref) <= 1e-12
    assert cli.main(["solve", "--in", life, "--iters", "3", "--precision", "fp64",
                     "--out-weights", wout]) == 0
    assert L.default_precision() == "fp32"  # --precision is scoped to the call
    bench = str(tmp_path / "bench.csv")
    assert cli.main(["bench", "--in", life, "--threads-list", "1,2", "--iters", "3",
                     "--report", bench]) == 0
    with open(bench) as f:
        rows = list(csv.reader(f))
    assert tuple(rows[0]) == cli.BENCH_COLUMNS and [r[0] for r in rows[1:]] == ["1", "2"]


def test_load_device_matches_host_path():
    path = os.path.join(GOLDEN, "ref_small.life")
    p = io.load(path)
    op, dims, y, w_true = io.load_device(path, exact=True)
    assert dims == p.dims and np.array_equal(y, p.y) and np.array_equal(w_true, p.w_true)
    yd = torch.zeros(dims.signal_len, dtype=torch.float64, device="cuda")
    op.dsc_f64(torch.from_numpy(w_true).cuda(), yd)
    yh = L.zeros_signal(dims)
    L.dsc_sequential(p.tensor, p.dictionary, w_true, yh, precision="fp64")
    assert np.array_equal(yd.cpu().numpy(), yh)
