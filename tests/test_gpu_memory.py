"""Device block cache of the library (life_release_cached_memory /
life_cached_memory_bytes): an operator rebuilt from cached blocks gives the
same bits as a fresh one, solver sessions reuse blocks, release empties it."""

import numpy as np
import pytest
import torch

import paper_1905_06234_b200 as L
from paper_1905_06234_b200 import _native as N, device

pytestmark = pytest.mark.gpu


def _problem():
    dims = L.Dims(1057, 2_000, 4_000, 96, 1_000_000)
    return L.generate(L.GenConfig(dims=dims, mean_run_length=520.0, weight_density=0.5,
                                  noise_sigma=0.1, seed=3))


def _products(p):
    op = device.DeviceOperator(p.tensor, p.dictionary)
    d = p.tensor.dims
    w = torch.from_numpy(p.w_true).to("cuda", torch.float32)
    y = torch.zeros(d.signal_len, dtype=torch.float32, device="cuda")
    g = torch.zeros(d.n_fibers, dtype=torch.float32, device="cuda")
    op.dsc_f32(w, y, flags=N.SKIP_ZERO)
    op.wc_f32(y, g)
    torch.cuda.synchronize()
    out = (y.cpu().numpy(), g.cpu().numpy())
    op.close()
    return out


def test_rebuild_from_cached_blocks_is_bitwise_equal():
    p = _problem()
    N.release_cached_memory()
    assert N.cached_memory_bytes() == 0
    y0, g0 = _products(p)
    cached = N.cached_memory_bytes()
    assert cached > 0  # the destroyed operator's blocks (and construction temporaries)
    y1, g1 = _products(p)  # served from the cache
    assert np.array_equal(y0, y1) and np.array_equal(g0, g1)
    assert N.cached_memory_bytes() == cached  # same blocks back, nothing new mapped
    N.release_cached_memory()
    assert N.cached_memory_bytes() == 0


def test_solves_reuse_session_blocks():
    p = _problem()
    cfg = L.SolverConfig(max_iters=6, grad_tol=0.0)
    w0, t0 = L.solve(p, config=cfg)
    before = N.cached_memory_bytes()
    w1, t1 = L.solve(p, config=cfg)
    assert np.array_equal(w0, w1)
    assert t0.final_objective == t1.final_objective
    assert N.cached_memory_bytes() == before
