"""Skewed operators on the default binned tcgen05 products (SURVEY.md 8 rows
a7 and f4).

* a7, long voxel segments: one voxel holds 5% of a 16M-coefficient problem.
  The reference splits such a segment across threads and merges the partial
  rows in a fixed order (engine.py:292-346 over _kernels.py:36-54); here the
  voxel is split over many tile rows (virtual rows) whose partial y rows are
  folded by the two-step fixup (life_bin.cu k_tile_dsc_fix / _fold) in a
  fixed order.  Parity against the device fp64 products (themselves pinned
  bit for bit to the reference in test_gpu_parity / test_gpu_scale), bitwise
  repeatability, and DSC time within 1.25x of the same problem unskewed.
* f4, skewed fascicle lengths: Zipf(1.3) fascicles (the hottest holds ~25% of
  the coefficients), split into virtual fascicle slots and folded per
  fascicle; same parity, WC within 1.3x of uniform.
* the host-input path of life_phi_create (LIFE_PHI_HOST_INPUT with fibers
  staged on a side stream) still reports the first out-of-range fiber.
"""

import numpy as np
import pytest
import torch

import paper_1905_06234_b200 as L
from paper_1905_06234_b200 import _native as N, device
from paper_1905_06234_b200.errors import IndexOutOfRange

pytestmark = pytest.mark.gpu
TOL32 = 1e-5


def _custom(nc, seed, zipf=None, hot_voxel=None, na=1057, nv=40_000, nf=100_000, nt=96):
    rng = np.random.default_rng(seed)
    a = rng.integers(0, na, nc, dtype=np.uint32)
    v = rng.integers(0, nv, nc, dtype=np.uint32)
    if zipf:
        f = ((rng.zipf(zipf, nc) - 1) % nf).astype(np.uint32)
    else:
        f = rng.integers(0, nf, nc, dtype=np.uint32)
    if hot_voxel:
        v[: int(hot_voxel * nc)] = 7
    val = 1.0 - rng.random(nc)
    d = L.Dims(n_atoms=na, n_voxels=nv, n_fibers=nf, n_dirs=nt, n_coeffs=nc)
    rows = rng.standard_normal((na, nt))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    t = L.PhiTensor(atoms=a, voxels=v, fibers=f, values=val, dims=d)
    return t, L.Dictionary(data=rows.ravel(), dims=d)


def _run(t, dic, reps=20):
    """fp32 products vs the fp64 exact ones; repeatability; mean call times."""
    d = t.dims
    op = device.DeviceOperator(t, dic, exact=True)
    assert op.kind == "bin" and op.tensor_ops == ("dsc", "wc")
    rng = np.random.default_rng(1)
    w64 = rng.random(d.n_fibers)
    w64[rng.random(d.n_fibers) < 0.3] = 0.0
    y64 = rng.standard_normal(d.signal_len)
    cu = (lambda x, dt: torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dt))
    yr = torch.zeros(d.signal_len, dtype=torch.float64, device="cuda")
    skr = torch.zeros(1, dtype=torch.int64, device="cuda")
    op.dsc_f64(cu(w64, torch.float64), yr, N.SKIP_ZERO, skr)
    wr = torch.zeros(d.n_fibers, dtype=torch.float64, device="cuda")
    op.wc_f64(cu(y64, torch.float64), wr)
    w32, yin = cu(w64, torch.float32), cu(y64, torch.float32)
    y = torch.empty(d.signal_len, dtype=torch.float32, device="cuda")
    g = torch.empty(d.n_fibers, dtype=torch.float32, device="cuda")
    sk = torch.zeros(1, dtype=torch.int64, device="cuda")
    op.dsc_f32(w32, y, None, N.SKIP_ZERO, sk)
    op.wc_f32(yin, g)
    y2, g2 = torch.empty_like(y), torch.empty_like(g)
    op.dsc_f32(w32, y2, None, N.SKIP_ZERO)
    op.wc_f32(yin, g2)
    torch.cuda.synchronize()
    out = {
        "dsc_err": (torch.linalg.norm(y.double() - yr) / torch.linalg.norm(yr)).item(),
        "wc_err": (torch.linalg.norm(g.double() - wr) / torch.linalg.norm(wr)).item(),
        "skips": (int(sk.item()), int(skr.item())),
        "repeat": bool(torch.equal(y, y2)) and bool(torch.equal(g, g2)),
    }
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for _ in range(3):
        op.dsc_f32(w32, y, None, N.SKIP_ZERO)
        op.wc_f32(yin, g)
    ev[0].record()
    for _ in range(reps):
        op.dsc_f32(w32, y, None, N.SKIP_ZERO)
    ev[1].record()
    for _ in range(reps):
        op.wc_f32(yin, g)
    ev[2].record()
    torch.cuda.synchronize()
    out["dsc_ms"] = ev[0].elapsed_time(ev[1]) / reps
    out["wc_ms"] = ev[1].elapsed_time(ev[2]) / reps
    op.close()
    return out


@pytest.fixture(scope="module")
def uniform16m():
    return _run(*_custom(16_000_000, 11))


def _check(r):
    assert r["dsc_err"] <= TOL32, r
    assert r["wc_err"] <= TOL32, r
    assert r["skips"][0] == r["skips"][1], r
    assert r["repeat"], r


def test_uniform_16m(uniform16m):
    _check(uniform16m)


def test_hot_voxel_5pct_of_16m(uniform16m):
    r = _run(*_custom(16_000_000, 11, hot_voxel=0.05))
    _check(r)
    ratio = r["dsc_ms"] / uniform16m["dsc_ms"]
    print(f"hot voxel DSC {r['dsc_ms']:.3f} ms vs uniform {uniform16m['dsc_ms']:.3f} ms: {ratio:.2f}x")
    assert ratio <= 1.25, (r, uniform16m)


def test_zipf_fascicles_16m(uniform16m):
    r = _run(*_custom(16_000_000, 11, zipf=1.3))
    _check(r)
    ratio = r["wc_ms"] / uniform16m["wc_ms"]
    print(f"Zipf WC {r['wc_ms']:.3f} ms vs uniform {uniform16m['wc_ms']:.3f} ms: {ratio:.2f}x")
    assert ratio <= 1.3, (r, uniform16m)
    assert r["dsc_ms"] / uniform16m["dsc_ms"] <= 1.3, (r, uniform16m)


def test_host_input_reports_first_bad_fiber():
    t, dic = _custom(200_000, 3, nv=2000, nf=3000)
    f = t.fibers.copy()
    f[123_457] = t.dims.n_fibers + 5
    f[150_000] = t.dims.n_fibers
    bad = L.PhiTensor(atoms=t.atoms, voxels=t.voxels, fibers=f, values=t.values, dims=t.dims)
    with pytest.raises(IndexOutOfRange) as ei:
        device.DeviceOperator(bad, dic)
    assert ei.value.dimension == "fiber" and ei.value.position == 123_457, str(ei.value)


@pytest.mark.parametrize("dim,big", [("atom", 1_000_000), ("atom", 2**31 + 7), ("atom", None),
                                     ("voxel", 2**20), ("voxel", 2**32 - 1), ("voxel", None)])
def test_host_input_reports_first_bad_atom_voxel(dim, big):
    """Atoms and voxels cross PCIe packed into one word (saturated fields):
    an index just past the dimension, or far beyond the packed field, still
    fails with its dimension and the first bad position."""
    t, dic = _custom(200_000, 4, nv=2000, nf=3000)
    arrs = {"atom": t.atoms.copy(), "voxel": t.voxels.copy()}
    n_dim = t.dims.n_atoms if dim == "atom" else t.dims.n_voxels
    arrs[dim][98_765] = n_dim if big is None else big
    arrs[dim][150_000] = n_dim + 1
    bad = L.PhiTensor(atoms=arrs["atom"], voxels=arrs["voxel"], fibers=t.fibers, values=t.values,
                      dims=t.dims)
    with pytest.raises(IndexOutOfRange) as ei:
        device.DeviceOperator(bad, dic)
    assert ei.value.dimension == dim and ei.value.position == 98_765, str(ei.value)


@pytest.mark.parametrize("skew", ["lognormal", "zipf"])
def test_device_generator_c5(skew):
    """The C5 device generator (datagen.draw_skewed_device): deterministic per
    seed, skewed as asked, and the default products within tolerance of the
    fp64 ones on what it draws (tools/sweep_c5.py checks up to 16M)."""
    from paper_1905_06234_b200 import datagen
    d1 = datagen.draw_skewed_device(2_000_000, skew, seed=5)
    d2 = datagen.draw_skewed_device(2_000_000, skew, seed=5)
    for x, y in zip(d1[1:6], d2[1:6]):
        assert torch.equal(x, y)
    dims, a, v, f, val, dic, fmax = d1
    assert dims.n_coeffs == 2_000_000 and int(torch.bincount(f).max()) == fmax
    assert fmax > 20 * dims.n_coeffs // dims.n_fibers  # long fascicles present
    op = device.DeviceOperator.from_device(dims, a, v, f, val, dic, exact=True)
    assert op.kind == "bin"
    w = torch.rand(dims.n_fibers, device="cuda")
    y = torch.empty(dims.signal_len, device="cuda")
    g = torch.empty(dims.n_fibers, device="cuda")
    op.dsc_f32(w, y)
    op.wc_f32(y, g)
    y64 = torch.zeros(dims.signal_len, dtype=torch.float64, device="cuda")
    op.dsc_f64(w.double(), y64)
    g64 = torch.zeros(dims.n_fibers, dtype=torch.float64, device="cuda")
    op.wc_f64(y.double(), g64)
    assert float((y.double() - y64).norm() / y64.norm()) <= TOL32
    assert float((g.double() - g64).norm() / g64.norm()) <= TOL32
    op.close()
