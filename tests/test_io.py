"""LIFE container and CSV report (io.py:1-172 of the reference): byte-level
compatibility with containers the reference wrote (tests/golden/*.life,
made by tests/golden/make_container.py), round trips and the error family."""

import os
import struct

import numpy as np
import pytest

from paper_1905_06234_b200 import io
from paper_1905_06234_b200.errors import CorruptContainer, IoFailure, UnsupportedVersion

from conftest import GOLDEN

REF = [os.path.join(GOLDEN, n) for n in ("ref_small.life", "ref_sorted.life")]


@pytest.mark.parametrize("path", REF)
def test_reference_container_round_trip_bitwise(path, tmp_path):
    p = io.load(path)
    out = tmp_path / "x.life"
    io.save(p, out)
    assert out.read_bytes() == open(path, "rb").read()


def test_reference_container_fields():
    p = io.load(REF[0])
    d = p.dims
    assert (d.n_atoms, d.n_voxels, d.n_fibers, d.n_dirs, d.n_coeffs) == (12, 30, 20, 8, 400)
    assert p.tensor.ordering == "unsorted" and p.y is not None and p.w_true is not None
    q = io.load(REF[1])
    assert q.tensor.ordering == "by_voxel" and q.w_true is None
    assert np.all(np.diff(q.tensor.voxels.astype(np.int64)) >= 0)


def _corrupt(tmp_path, mutate):
    raw = bytearray(open(REF[0], "rb").read())
    raw = mutate(raw)
    path = tmp_path / "bad.life"
    path.write_bytes(bytes(raw))
    return path


def test_errors(tmp_path):
    with pytest.raises(CorruptContainer):
        io.load(_corrupt(tmp_path, lambda r: b"LIFX" + r[4:]))
    with pytest.raises(UnsupportedVersion):
        io.load(_corrupt(tmp_path, lambda r: r[:4] + struct.pack("<I", 2) + r[8:]))
    with pytest.raises(CorruptContainer):
        io.load(_corrupt(tmp_path, lambda r: r[:8] + struct.pack("<I", 8) + r[12:]))
    with pytest.raises(CorruptContainer):
        io.load(_corrupt(tmp_path, lambda r: r[:-3]))
    with pytest.raises(CorruptContainer):
        io.load(_corrupt(tmp_path, lambda r: r + b"\0"))
    with pytest.raises(CorruptContainer):  # atom index out of range fails validation
        io.load(_corrupt(tmp_path, lambda r: r[:52] + struct.pack("<I", 999) + r[56:]))
    with pytest.raises(IoFailure):
        io.load(tmp_path / "missing.life")


def test_report_round_trip(tmp_path):
    rows = [io.ReportRow(1, "dsc", "voxel", "coeff+syncfree", 1, 1.25e-4, 3),
            io.ReportRow(2, "wc", "atom", "coeff", 8, 0.1 + 0.2, 0)]
    path = tmp_path / "r.csv"
    io.export_report(rows, path)
    assert open(path).readline().strip() == ",".join(io.REPORT_COLUMNS)
    assert io.read_report(path) == rows
