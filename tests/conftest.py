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


def solver_case(g, name):
    """Golden solver case `name` as an oracle problem dict."""
    pre = f"solp_{name}_"
    return dict(atoms=g[pre + "atoms"], voxels=g[pre + "voxels"],
                fibers=g[pre + "fibers"], values=g[pre + "values"],
                dict=g[pre + "dict"], y=g[pre + "y"], ordering="unsorted",
                dims=tuple(int(x) for x in g[pre + "dims"]))


def fp32_product_floor(g, name, iters=30, eps=0.0, seeds=1):
    """How far the reference's `iters`-iteration trajectory moves when the
    inputs are rounded to fp32 and every DSC/WC product carries a relative
    L2 error `eps` (random, per product) before being rounded to fp32
    (eps=0: correctly rounded fp32 products, the least any fp32 solver can
    inherit).  Returns the max over `seeds` of (rel L2 of w, relative error
    of the final objective, rel L2 of the objective trajectory).

    Ill-conditioned cases amplify one-ulp product errors far beyond the
    north_star 1e-4 bound (small11: 6.8e-4 with exact rounding, ~4e-2 at
    eps = 3e-7); well-conditioned ones stay ~1e-8."""
    from oracle import oracle as O

    def f32(a):
        return np.asarray(a).astype(np.float32).astype(np.float64)

    dsc0, wc0 = O.dsc_chunks, O.wc_chunks
    fo = float(g[f"sol_{name}_t1_final_objective"])
    worst = np.zeros(3)
    for seed in range(seeds):
        rng = np.random.default_rng(seed)
        p = solver_case(g, name)
        for k in ("values", "dict", "y"):
            p[k] = f32(p[k])

        def noisy(t):
            if eps > 0.0 and t.size:
                t = t + eps * np.linalg.norm(t) / np.sqrt(t.size) * rng.standard_normal(t.size)
            return f32(t)

        def dsc(q, w, y, chunks, aligned, skip_zero=True):
            t = np.zeros_like(y)
            r = dsc0(q, w, t, chunks, aligned, skip_zero)
            y += noisy(t)
            return r

        def wc(q, y, w, chunks, kind="coefficient"):
            t = np.zeros_like(w)
            wc0(q, f32(y), t, chunks, kind)
            w += noisy(t)

        O.dsc_chunks, O.wc_chunks = dsc, wc
        try:
            w, tr = O.solve(p, max_iters=iters, grad_tol=0.0)
        finally:
            O.dsc_chunks, O.wc_chunks = dsc0, wc0
        objs = [r["objective"] for r in tr["records"]]
        worst = np.maximum(worst, [rel_l2(w, g[f"sol_{name}_t1_w"]),
                                   abs(tr["final_objective"] - fo) / abs(fo),
                                   rel_l2(objs, g[f"sol_{name}_t1_objective"])])
    return worst
