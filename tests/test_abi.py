"""The C-ABI library loads and exports exactly what include/life_b200.h
declares (no GPU needed: no compute calls here)."""

import os
import re

import pytest

from paper_1905_06234_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "life_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"LIFE_API[^;(]*?\b(life_\w+)\s*\(", text)))


def test_header_declares_api():
    names = declared_symbols()
    assert "life_dsc_f32" in names and "life_solve" in names and len(names) >= 15


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) == set(_native.SIGNATURES), \
        "ctypes signature table out of sync with the header"


def test_abi_version_and_status_strings():
    lib = _native.lib()
    assert lib.life_abi_version() == 1
    assert lib.life_status_string(2) == b"DimensionMismatch"
    assert lib.life_status_string(5) == b"DegenerateStep"
    assert isinstance(_native.launch_count(), int)


def test_null_arguments_rejected_without_device():
    lib = _native.lib()
    rc = lib.life_dsc_f32(None, None, None, None, 0, None, None)
    assert rc == 22  # LIFE_ERR_INVALID_ARGUMENT, before any CUDA call
    assert b"null" in lib.life_last_error()
    assert lib.life_phi_destroy(None) == 0


def test_status_mapping():
    from paper_1905_06234_b200 import errors as E
    for status, cls in ((1, E.ConfigInvalid), (2, E.DimensionMismatch),
                        (3, E.PlanTensorMismatch), (5, E.DegenerateStep),
                        (8, E.NotSorted), (6, E.IndexOutOfRange), (20, E.DeviceError)):
        with pytest.raises(cls):
            E.raise_for_status(status, "atom index out of range", 3)


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np

    import paper_1905_06234_b200 as L
    d = L.Dims(1, 1, 1, 2, 1)
    t = L.PhiTensor(atoms=[0], voxels=[0], fibers=[0], values=[2.0], dims=d)
    with pytest.raises(_native.NativeUnavailable):
        L.dsc_sequential(t, L.Dictionary(data=[1.0, 0.5], dims=d), np.array([3.0]),
                         np.zeros(2))
