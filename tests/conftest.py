import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: larger CPU cases")


@pytest.fixture(scope="session")
def golden():
    with np.load(os.path.join(GOLDEN, "golden_small.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden_hashes():
    import json
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.lib()
    return O


def golden_problem(g, seed):
    pre = f"s{seed}_"
    return dict(atoms=g[pre + "atoms"], voxels=g[pre + "voxels"],
                fibers=g[pre + "fibers"], values=g[pre + "values"],
                dict=g[pre + "dict"], y=g[pre + "y"], w_true=g[pre + "w_true"],
                dims=tuple(int(x) for x in g[pre + "dims"]), ordering="unsorted")


def assert_rel(actual, desired, tol):
    """Relative check with a scale-aware floor (mirrors the reference's
    tests/conftest.py:7-17 helper)."""
    desired = np.asarray(desired, dtype=np.float64)
    scale = float(np.max(np.abs(desired))) if desired.size else 0.0
    np.testing.assert_allclose(np.asarray(actual, dtype=np.float64), desired,
                               rtol=tol, atol=tol * max(scale, 1e-300))


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = float(np.linalg.norm(b))
    return float(np.linalg.norm(a - b)) / (nb if nb > 0 else 1.0)
