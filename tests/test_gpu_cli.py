"""CLI end to end on the device (gen -> spmv / solve / tune / bench, verify)
and the device container loader against the host path."""

import csv
import os

import numpy as np
import pytest
import torch

import paper_1905_06234_b200 as L
from paper_1905_06234_b200 import cli, io

from conftest import GOLDEN, rel_l2

pytestmark = pytest.mark.gpu


def test_gen_spmv_solve_tune_bench(tmp_path, capsys):
    life = str(tmp_path / "p.life")
    assert cli.main(["gen", "--voxels", "300", "--fibers", "200", "--atoms", "40", "--coeffs", "20000",
                     "--run-len", "60", "--noise", "0.1", "--out", life]) == 0
    p = io.load(life)
    assert p.dims.n_coeffs == 20000 and p.y is not None
    rep = str(tmp_path / "spmv.csv")
    assert cli.main(["spmv", "--in", life, "--op", "dsc", "--restructure", "voxel", "--partition",
                     "coeff", "--sync-free", "--threads", "4", "--repeat", "3", "--report", rep]) == 0
    rows = io.read_report(rep)
    assert [r.iteration for r in rows] == [1, 2, 3] and all(r.partition == "coeff+syncfree" for r in rows)
    assert all(r.elapsed_s > 0 for r in rows)
    assert cli.main(["spmv", "--in", life, "--op", "wc", "--restructure", "auto", "--repeat", "1"]) == 0
    tr, wout = str(tmp_path / "trace.csv"), str(tmp_path / "w.txt")
    assert cli.main(["solve", "--in", life, "--iters", "6", "--grad-tol", "0", "--trace", tr,
                     "--out-weights", wout]) == 0
    with open(tr) as f:
        rows = list(csv.reader(f))
    assert rows[0] == ["iteration", "objective", "alpha", "grad_norm", "zeros", "dsc_s", "wc_s"]
    assert len(rows) == 7
    w = np.loadtxt(wout)
    w_ref, _ = L.solve(p, config=L.SolverConfig(max_iters=6, grad_tol=0.0))
    assert rel_l2(w, w_ref) <= 1e-12
    assert cli.main(["tune", "--in", life, "--op", "dsc", "--trials", "1", "--layouts"]) == 0
    out = capsys.readouterr().out
    assert "selected: " in out and "selected layout: " in out
    bench = str(tmp_path / "bench.csv")
    assert cli.main(["bench", "--in", life, "--threads-list", "1,2", "--iters", "3", "--report", bench]) == 0
    with open(bench) as f:
        assert next(csv.reader(f)) == ["threads", "iters", "elapsed_s", "speedup_vs_1thread"]


def test_verify_suite():
    assert cli.main(["verify", "--seeds", "4"]) == cli.EXIT_OK


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
