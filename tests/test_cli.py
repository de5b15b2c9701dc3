"""CLI surface: the reference's flags for spmv / solve /
bench, its CSV schemas and the exit codes of the host-side error paths (no
GPU needed for these)."""

import os

from paper_1905_06234_b200 import cli

from conftest import GOLDEN

REF = os.path.join(GOLDEN, "ref_small.life")


def test_parser_mirrors_reference_flags():
    p = cli.build_parser()
    a = p.parse_args(["spmv", "--in", "x", "--op", "wc", "--restructure", "auto", "--partition",
                      "voxel", "--sync-free", "--threads", "4", "--repeat", "3", "--report", "r.csv"])
    assert (a.op, a.restructure, a.partition, a.sync_free, a.threads, a.repeat) == \
        ("wc", "auto", "voxel", True, 4, 3)
    a = p.parse_args(["solve", "--in", "x"])
    assert a.iters == 500 and a.grad_tol == 1e-12 and a.precision is None
    a = p.parse_args(["bench", "--in", "x", "--report", "r"])
    assert a.threads_list == "1,2,4,8" and a.iters == 10
    assert cli.TRACE_COLUMNS == ("iteration", "objective", "alpha", "grad_norm", "zeros",
                                 "dsc_s", "wc_s")
    assert cli.BENCH_COLUMNS == ("threads", "iters", "elapsed_s", "speedup_vs_1thread")


def test_threads_default_from_env(monkeypatch):
    monkeypatch.setenv("LIFE_THREADS", "6")
    assert cli.host_threads(None) == 6 and cli.host_threads(2) == 2
    monkeypatch.setenv("LIFE_THREADS", "x")
    assert cli.host_threads(None) == 1


def test_exit_codes(tmp_path, capsys):
    assert cli.main(["spmv", "--in", str(tmp_path / "missing.life"), "--op", "dsc"]) == cli.EXIT_BAD_INPUT
    bad = tmp_path / "bad.life"
    bad.write_bytes(b"NOPE" + open(REF, "rb").read()[4:])
    assert cli.main(["solve", "--in", str(bad)]) == cli.EXIT_BAD_INPUT
    # voxel partitioning needs a voxel-sorted tensor: strategy error, exit 3
    assert cli.main(["spmv", "--in", REF, "--op", "dsc", "--partition", "voxel"]) == cli.EXIT_BAD_STRATEGY
    assert cli.main(["bench", "--in", REF, "--report", str(tmp_path / "b.csv"),
                     "--threads-list", "0"]) == cli.EXIT_BAD_INPUT
    err = capsys.readouterr().err
    assert err.count("error:") == 4
