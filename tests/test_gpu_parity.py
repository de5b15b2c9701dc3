"""Parity of the B200 path with the reference (golden vectors) and the oracle.

Tolerances (north_star): fp32 DSC/WC within 1e-5 relative L2; the fp64
path is bit-exact; SBBNNLS weights/objective within 1e-4 relative after a
fixed iteration count (fp32) and 1e-9 (fp64); restructuring permutations
and zero-skip counts are exact.
"""

import hashlib

import numpy as np
import pytest

import paper_1905_06234_b200 as L
from paper_1905_06234_b200 import datagen

from conftest import fp32_product_floor, golden_problem, rel_l2

pytestmark = pytest.mark.gpu
SEEDS = range(30)
TOL32 = 1e-5


# set_layout name -> DeviceOperator.kind it yields (at n_dirs <= 128)
KIND = {"sparse": "sparse", "dense": "bin", "bin": "bin"}
TENSOR_OPS = {"sparse": (), "dense": ("dsc", "wc"), "bin": ("dsc", "wc")}


@pytest.fixture(params=["sparse", "bin"])
def layout(request):
    """Run a test against every fp32 kernel family: voxel-segment (sparse)
    and the binned two-phase products on tcgen05 (bin, the default)."""
    from paper_1905_06234_b200 import device
    device.set_layout(request.param)
    yield request.param
    device.set_layout("auto")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).tobytes()).hexdigest()


def tensor_of(g, ordering="unsorted", perm=None):
    d = L.Dims(*g["dims"])
    idx = slice(None) if perm is None else perm
    t = L.PhiTensor(atoms=g["atoms"][idx], voxels=g["voxels"][idx], fibers=g["fibers"][idx],
                    values=g["values"][idx], dims=d, ordering=ordering)
    return t, L.Dictionary(data=g["dict"], dims=d), d


def dsc(t, dic, d, w, precision, skip=True):
    y = L.zeros_signal(d)
    st = L.dsc_sequential(t, dic, w, y, skip_zero=skip, precision=precision)
    return y, st.skipped_coefficients


def wc(t, dic, d, y, precision):
    w = L.zeros_weights(d)
    L.wc_sequential(t, dic, y, w, precision=precision)
    return w


# ---- known answers ---------------------------------------------------------


@pytest.mark.parametrize("precision", ["fp32", "fp64"])
def test_kat_single_coefficient(precision):
    d = L.Dims(1, 1, 1, 2, 1)
    t = L.PhiTensor(atoms=[0], voxels=[0], fibers=[0], values=[2.0], dims=d)
    dic = L.Dictionary(data=[1.0, 0.5], dims=d)
    y, _ = dsc(t, dic, d, np.array([3.0]), precision)
    assert y.tolist() == [6.0, 3.0]                     # test_engine.py:21-25
    w = wc(t, dic, d, np.array([6.0, 3.0]), precision)
    assert w.tolist() == [15.0]                         # test_engine.py:37-41


def test_kat_sort_runs():
    d = L.Dims(3, 3, 3, 2, 3)
    t = L.PhiTensor(atoms=[0, 1, 2], voxels=[2, 0, 1], fibers=[1, 2, 0],
                    values=[1.0, 2.0, 3.0], dims=d)
    s, perm = L.sort_by(t, "voxel")
    assert perm.tolist() == [1, 2, 0] and s.values.tolist() == [2.0, 3.0, 1.0]
    d = L.Dims(1, 2, 4, 1, 4)
    t = L.PhiTensor(atoms=[0, 0, 0, 0], voxels=[1, 0, 1, 0], fibers=[0, 1, 2, 3],
                    values=[10.0, 11.0, 12.0, 13.0], dims=d)
    s, _ = L.sort_by(t, "voxel")
    assert s.values.tolist() == [11.0, 13.0, 10.0, 12.0]
    d = L.Dims(1, 3, 6, 1, 6)
    t = L.PhiTensor(atoms=[0] * 6, voxels=[0, 0, 1, 1, 1, 2], fibers=range(6),
                    values=np.ones(6), dims=d, ordering="by_voxel")
    runs = L.detect_runs(t)
    assert runs.boundaries.tolist() == [0, 2, 5, 6] and runs.key_values.tolist() == [0, 1, 2]


# ---- golden vectors (reference outputs) -------------------------------------


@pytest.mark.parametrize("seed", SEEDS)
def test_fp64_bitwise(golden, seed):
    g = golden_problem(golden, seed)
    pre = f"s{seed}_"
    t, dic, d = tensor_of(g)
    for wkey in ("w_in", "w_sparse"):
        y, sk = dsc(t, dic, d, golden[pre + wkey], "fp64")
        assert np.array_equal(y, golden[pre + "dsc_" + wkey])
        assert sk == int(golden[pre + "dsc_" + wkey + "_skipped"])
    assert np.array_equal(wc(t, dic, d, golden[pre + "y_in"], "fp64"), golden[pre + "wc_y_in"])
    for key in ("atom", "voxel", "fiber"):
        s, _, _ = tensor_of(g, "by_" + key, golden[pre + "perm_" + key])
        y, _ = dsc(s, dic, d, golden[pre + "w_in"], "fp64")
        assert np.array_equal(y, golden[pre + "dsc_sorted_" + key])
        assert np.array_equal(wc(s, dic, d, golden[pre + "y_in"], "fp64"),
                              golden[pre + "wc_sorted_" + key])


@pytest.mark.parametrize("seed", SEEDS)
def test_fp32_within_tolerance(golden, seed, layout):
    g = golden_problem(golden, seed)
    pre = f"s{seed}_"
    t, dic, d = tensor_of(g)
    for wkey in ("w_in", "w_sparse"):
        y, sk = dsc(t, dic, d, golden[pre + wkey], "fp32")
        assert rel_l2(y, golden[pre + "dsc_" + wkey]) <= TOL32
        assert sk == int(golden[pre + "dsc_" + wkey + "_skipped"])
    assert rel_l2(wc(t, dic, d, golden[pre + "y_in"], "fp32"), golden[pre + "wc_y_in"]) <= TOL32


@pytest.mark.parametrize("seed", SEEDS)
def test_restructuring_bitwise(golden, seed):
    g = golden_problem(golden, seed)
    pre = f"s{seed}_"
    t, _, _ = tensor_of(g)
    for key in ("atom", "voxel", "fiber"):
        s, perm = L.sort_by(t, key)
        assert perm.dtype == np.int64
        assert np.array_equal(perm, golden[pre + "perm_" + key])
        for name in ("atoms", "voxels", "fibers", "values"):
            assert np.array_equal(getattr(s, name), getattr(t, name)[perm])
        runs = L.detect_runs(s)
        assert np.array_equal(runs.boundaries, golden[pre + "runs_" + key])
        assert np.array_equal(runs.key_values, golden[pre + "runkeys_" + key])


def test_parallel_entry_points_and_plans(golden):
    g = golden_problem(golden, 14)
    pre = "s14_"
    s, dic, d = tensor_of(g, "by_voxel", golden[pre + "perm_voxel"])
    off = L.precompute_offsets(s)
    w = golden[pre + "w_in"]
    for T in (2, 4, 8):
        plan = L.build_plan(off, L.PartitionStrategy("coefficient", sync_free=True), T)
        y = L.zeros_signal(d)
        L.dsc_parallel(off, dic, w, y, plan, precision="fp64")
        assert np.array_equal(y, golden[pre + "dsc_sorted_voxel"])
    runs = L.detect_runs(s)
    lens = runs.lengths()
    if lens.max() >= 2:
        inside = int(runs.boundaries[int(np.argmax(lens))]) + 1
        bad = L.ExecutionPlan(strategy=L.PartitionStrategy("coefficient", sync_free=True),
                              threads=2, chunks=((0, inside), (inside, d.n_coeffs)))
        with pytest.raises(L.errors.PlanTensorMismatch):
            L.dsc_parallel(off, dic, w, L.zeros_signal(d), bad)


# ---- solver -------------------------------------------------------------------


def _solver_problem(golden, name):
    pre = f"solp_{name}_"
    d = L.Dims(*[int(x) for x in golden[pre + "dims"]])
    t = L.PhiTensor(atoms=golden[pre + "atoms"], voxels=golden[pre + "voxels"],
                    fibers=golden[pre + "fibers"], values=golden[pre + "values"], dims=d)
    return L.Problem(tensor=t, dictionary=L.Dictionary(data=golden[pre + "dict"], dims=d),
                     y=golden[pre + "y"])


# fp32 tolerance per case.  Well-conditioned cases: the north_star 1e-4 on
# weights, final objective and objective trajectory.  small3 / small11 are
# ill-conditioned: even correctly rounded fp32 products move the reference's
# own 30-iteration weights by 8.4e-5 / 6.8e-4 (> 1e-4 for small11), and the
# drift grows with the product error (tests/test_oracle.py::
# test_fp32_product_rounding_floor_of_solver_cases).  For those the device
# solve is held to 3x the worst drift of the reference trajectory over 8
# random perturbations of every product at the device's OWN measured product
# error on that operator: as close as fp32 products of that accuracy allow.
# The fp64 path is held to 1e-9 on every case.
ILL_CONDITIONED = ("small3", "small11")


def _device_product_error(p):
    rng = np.random.default_rng(0)
    d = p.tensor.dims
    w = np.abs(rng.standard_normal(d.n_fibers))
    ys = [L.zeros_signal(d) for _ in range(2)]
    for y, prec in zip(ys, ("fp32", "fp64")):
        L.dsc_sequential(p.tensor, p.dictionary, w, y, precision=prec)
    ws = [L.zeros_weights(d) for _ in range(2)]
    for wo, prec in zip(ws, ("fp32", "fp64")):
        L.wc_sequential(p.tensor, p.dictionary, p.y, wo, precision=prec)
    return max(rel_l2(ys[0], ys[1]), rel_l2(ws[0], ws[1]))


def _case_tols(golden, name, precision, tol, p):
    if precision == "fp64" or name not in ILL_CONDITIONED:
        return tol, tol, tol
    eps = _device_product_error(p)
    floor = fp32_product_floor(golden, name, eps=eps, seeds=8)
    return tuple(max(tol, 3.0 * f) for f in floor)


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-9), ("fp32", 1e-4)])
def test_solver_matches_reference(golden, precision, tol, layout):
    for name in golden["solver_case_names"]:
        name = str(name)
        p = _solver_problem(golden, name)
        w, tr = L.solve(p, config=L.SolverConfig(max_iters=30, grad_tol=0.0,
                                                 precision=precision))
        pre = f"sol_{name}_t1_"
        ref_w = golden[pre + "w"]
        assert tr.termination == str(golden[pre + "termination"]), name
        assert tr.iterations == len(golden[pre + "objective"]), name
        if name == "noiseless42":
            # objective reaches ~1e-26: compare the fit, not the roundoff
            assert tr.final_objective <= 1e-6 * tr.initial_objective
            continue
        tw, tfo, tobj = _case_tols(golden, name, precision, tol, p)
        assert rel_l2(w, ref_w) <= tw, (name, rel_l2(w, ref_w), tw)
        fo = float(golden[pre + "final_objective"])
        assert abs(tr.final_objective - fo) <= tfo * abs(fo), (name, tfo)
        objs = np.array([r.objective for r in tr.records])
        assert rel_l2(objs, golden[pre + "objective"]) <= tobj, (name, tobj)
        if precision == "fp64":
            assert [r.zeros for r in tr.records] == golden[pre + "zeros"].tolist()


def test_solver_known_answers():
    d = L.Dims(1, 1, 1, 1, 1)
    t = L.PhiTensor(atoms=[0], voxels=[0], fibers=[0], values=[1.0], dims=d)
    p = L.Problem(tensor=t, dictionary=L.Dictionary(data=[1.0], dims=d), y=np.array([3.0]))
    for precision in ("fp32", "fp64"):
        w, tr = L.solve(p, w0=np.array([0.0]),
                        config=L.SolverConfig(max_iters=10, precision=precision))
        assert tr.termination == "grad_tol" and w.tolist() == [3.0]   # test_sbbnnls.py:120-126
        assert tr.iterations == 1 and tr.records[0].alpha == pytest.approx(1.0, rel=1e-7)
    # degenerate denominator: fascicle 1 touches nothing (test_sbbnnls.py:100-107)
    d = L.Dims(1, 1, 2, 1, 1)
    t = L.PhiTensor(atoms=[0], voxels=[0], fibers=[0], values=[1.0], dims=d)
    p = L.Problem(tensor=t, dictionary=L.Dictionary(data=[1.0], dims=d), y=np.array([1.0]))
    with pytest.raises(L.errors.DegenerateStep):
        L.step_size(1, np.array([0.0, 1.0]), p)


def test_solver_call_counts_and_determinism():
    dims = L.Dims(10, 30, 20, 8, 300)
    p = L.generate(L.GenConfig(dims=dims, mean_run_length=4.0, noise_sigma=0.0, seed=9))
    _, tr = L.solve(p, config=L.SolverConfig(max_iters=40, grad_tol=0.0))
    odd = {(r.dsc_calls, r.wc_calls) for r in tr.records if r.iteration % 2 == 1}
    even = {(r.dsc_calls, r.wc_calls) for r in tr.records if r.iteration % 2 == 0}
    assert odd == {(2, 1)} and even == {(2, 2)}                # test_sbbnnls.py:144-154
    cfg = L.SolverConfig(max_iters=30)
    wa, _ = L.solve(p, config=cfg)
    wb, _ = L.solve(p, config=cfg)
    assert np.array_equal(wa, wb)
    # exact solution: immediate grad_tol in the bit-exact mode (test_sbbnnls.py:110-117)
    q = L.generate(L.GenConfig(dims=dims, mean_run_length=4.0, noise_sigma=0.0, seed=42))
    w, tr = L.solve(q, w0=q.w_true, config=L.SolverConfig(max_iters=50, precision="fp64"))
    assert tr.termination == "grad_tol" and tr.iterations == 0 and np.array_equal(w, q.w_true)


# ---- scale: hashed reference outputs (medium, C1) --------------------------


@pytest.mark.parametrize("case", ["medium", "c1"])
def test_hashed_reference_cases(golden_hashes, case, layout):
    rec = golden_hashes[case]
    d = L.Dims(*rec["dims"])
    cfg = L.GenConfig(dims=d, mean_run_length=rec["mean_run_length"],
                      weight_density=rec["weight_density"], noise_sigma=rec["noise_sigma"],
                      seed=rec["seed"])
    p = L.generate(cfg)
    assert sha(p.y) == rec["sha_y"], "generator y (fp64 exact DSC) differs from reference"
    w = wc(p.tensor, p.dictionary, d, p.y, "fp64")
    assert sha(w) == rec["sha_wc_y"]
    y, sk = dsc(p.tensor, p.dictionary, d, w, "fp64")
    assert sha(y) == rec["sha_dsc_wc_y"] and sk == rec["skipped_dsc_wc_y"]
    w32 = wc(p.tensor, p.dictionary, d, p.y, "fp32")
    assert rel_l2(w32, w) <= TOL32
    y32, sk32 = dsc(p.tensor, p.dictionary, d, w, "fp32")
    assert rel_l2(y32, y) <= TOL32
    for key in ("atom", "voxel", "fiber"):
        _, perm = L.sort_by(p.tensor, key)
        assert sha(perm) == rec["sha_perm_" + key], key
    if "solve_iters" in rec:
        w, tr = L.solve(p, config=L.SolverConfig(max_iters=rec["solve_iters"], grad_tol=0.0))
        assert abs(tr.final_objective - rec["solve_final_objective"]) <= \
            1e-4 * rec["solve_final_objective"]
        assert abs(np.linalg.norm(w) - rec["solve_w_norm"]) <= 1e-4 * rec["solve_w_norm"]


# ---- edge cases -------------------------------------------------------------------


def test_empty_tensor():
    d = L.Dims(2, 2, 2, 3, 0)
    t = L.PhiTensor(atoms=np.empty(0, np.uint32), voxels=np.empty(0, np.uint32),
                    fibers=np.empty(0, np.uint32), values=np.empty(0), dims=d,
                    ordering="by_voxel")
    dic = L.Dictionary(data=np.ones(d.dict_len), dims=d)
    y = np.full(d.signal_len, 3.0)
    st = L.dsc_sequential(t, dic, np.ones(2), y)
    assert np.all(y == 3.0) and st.skipped_coefficients == 0
    runs = L.detect_runs(t)
    assert runs.n_runs == 0 and runs.boundaries.tolist() == [0]


@pytest.mark.parametrize("n_dirs", [1, 8, 33, 150, 160, 300])
def test_odd_direction_counts(oracle, n_dirs, layout):
    dims = (7, 60, 40, n_dirs, 3000)
    q = oracle.generate(dims, 20.0, 0.5, 0.1, n_dirs)
    d = L.Dims(*dims)
    t = L.PhiTensor(atoms=q["atoms"], voxels=q["voxels"], fibers=q["fibers"],
                    values=q["values"], dims=d)
    dic = L.Dictionary(data=q["dict"], dims=d)
    w = np.random.default_rng(1).standard_normal(d.n_fibers)
    yo = np.zeros(d.signal_len)
    oracle.dsc(q, w, yo)
    assert rel_l2(dsc(t, dic, d, w, "fp32")[0], yo) <= TOL32
    assert np.array_equal(dsc(t, dic, d, w, "fp64")[0], yo)
    wo = np.zeros(d.n_fibers)
    oracle.wc(q, q["y"], wo)
    assert rel_l2(wc(t, dic, d, q["y"], "fp32"), wo) <= TOL32
    assert np.array_equal(wc(t, dic, d, q["y"], "fp64"), wo)


@pytest.mark.parametrize("n_dirs", [96, 150])
def test_fascicles_beyond_2_20(oracle, n_dirs, layout):
    """Nf > 2^20 (C4: 1M fascicles, C5 at 256M+): the binned products take it
    on the tensor path (round 1's packed 20-bit fascicle field fell back to
    CUDA cores)."""
    from paper_1905_06234_b200 import device
    dims = (1057, 1500, 1_200_000, n_dirs, 450_000)
    q = oracle.generate(dims, 300.0, 0.5, 0.1, 17)
    d = L.Dims(*dims)
    t = L.PhiTensor(atoms=q["atoms"], voxels=q["voxels"], fibers=q["fibers"],
                    values=q["values"], dims=d)
    dic = L.Dictionary(data=q["dict"], dims=d)
    if layout == "bin":
        op = device.operator_for(t, dic)
        assert op.kind == "bin" and op.tensor_ops == ("dsc", "wc")
    w = np.random.default_rng(2).random(d.n_fibers)
    yo = np.zeros(d.signal_len)
    oracle.dsc(q, w, yo)
    assert rel_l2(dsc(t, dic, d, w, "fp32")[0], yo) <= TOL32
    wo = np.zeros(d.n_fibers)
    oracle.wc(q, q["y"], wo)
    assert rel_l2(wc(t, dic, d, q["y"], "fp32"), wo) <= TOL32


def test_single_giant_run_and_long_fascicle(oracle, layout):
    # every coefficient in voxel 0 and fascicle 0 (maximal segments)
    n = 20000
    rng = np.random.default_rng(5)
    d = L.Dims(1057, 3, 8, 96, n)
    q = dict(atoms=rng.integers(0, 1057, n).astype(np.uint32), voxels=np.zeros(n, np.uint32),
             fibers=np.zeros(n, np.uint32), values=rng.random(n) + 0.1,
             dict=rng.standard_normal(1057 * 96), dims=(1057, 3, 8, 96, n), ordering="unsorted")
    t = L.PhiTensor(atoms=q["atoms"], voxels=q["voxels"], fibers=q["fibers"],
                    values=q["values"], dims=d)
    dic = L.Dictionary(data=q["dict"], dims=d)
    w = np.array([0.7, 0.0, 1.0, 2.0, 0.0, 0.0, 0.0, 0.0])
    yo = np.zeros(d.signal_len)
    oracle.dsc(q, w, yo)
    assert rel_l2(dsc(t, dic, d, w, "fp32")[0], yo) <= TOL32
    y_in = rng.standard_normal(d.signal_len)
    wo = np.zeros(8)
    oracle.wc(q, y_in, wo)
    assert rel_l2(wc(t, dic, d, y_in, "fp32"), wo) <= TOL32


def test_zero_skip_exact_count(layout):
    dims = L.Dims(40, 200, 300, 96, 50_000)
    p = L.generate(L.GenConfig(dims=dims, mean_run_length=100.0, seed=22))
    rng = np.random.default_rng(22)
    w = np.abs(rng.standard_normal(dims.n_fibers)) + 0.1
    w[rng.permutation(dims.n_fibers)[:dims.n_fibers // 2]] = 0.0
    brute = int(np.count_nonzero(w[p.tensor.fibers] * p.tensor.values == 0.0))
    for precision in ("fp32", "fp64"):
        y_on, sk = dsc(p.tensor, p.dictionary, dims, w, precision, skip=True)
        y_off, sk_off = dsc(p.tensor, p.dictionary, dims, w, precision, skip=False)
        assert sk == brute
        assert sk_off == 0   # KernelStats counts skips only when skipping (_kernels.py:25-28)
        assert np.array_equal(y_on, y_off)


def test_fp32_repeat_bitwise_and_accumulate(layout):
    import torch
    dims = L.Dims(1057, 2000, 4000, 96, 1_000_000)
    t, dic, w_true, _ = datagen.draw_arrays(L.GenConfig(dims=dims, mean_run_length=520.0,
                                                        seed=4))
    op = L.DeviceOperator(t, dic)
    assert op.kind == KIND[layout]
    assert op.tensor_ops == TENSOR_OPS[layout]
    if layout == "sparse":
        assert op.info.atom_groups == 2  # 1057 x 96 fp32 exceeds one CTA's shared memory
    w = torch.from_numpy(w_true).float().cuda()
    y1 = torch.zeros(dims.signal_len, device="cuda")
    y2 = torch.zeros_like(y1)
    op.dsc_f32(w, y1)
    op.dsc_f32(w, y2)
    assert torch.equal(y1, y2)
    g1 = torch.zeros(dims.n_fibers, device="cuda")
    g2 = torch.zeros_like(g1)
    op.wc_f32(y1, g1)
    op.wc_f32(y1, g2)
    assert torch.equal(g1, g2)
    # accumulate contract: out += M x
    y3 = y1.clone()
    op.dsc_f32(w, y3, flags=L._native.ACCUMULATE)
    scale = float(y1.abs().max())
    assert torch.allclose(y3, 2 * y1, rtol=1e-5, atol=1e-5 * scale)
    # adjointness <M w, y> == <w, M^T y> at scale
    lhs = float(torch.dot(y1.double(), y1.double()))
    rhs = float(torch.dot(w.double(), g1.double()))
    assert abs(lhs - rhs) <= 1e-5 * abs(lhs)


# ---- boundary robustness -------------------------------------------


def test_misaligned_views_and_abi_rejection():
    """Offset views (16-byte misaligned) are copied by the Python layer; the C
    ABI itself rejects a misaligned pointer instead of faulting."""
    import ctypes

    import torch
    dims = L.Dims(40, 200, 300, 96, 50_000)
    p = L.generate(L.GenConfig(dims=dims, mean_run_length=100.0, seed=3))
    w = torch.from_numpy(np.abs(np.random.default_rng(0).standard_normal(dims.n_fibers))).float()
    ref = L.zeros_signal(dims)
    L.dsc_sequential(p.tensor, p.dictionary, w.numpy().astype(np.float64), ref, precision="fp64")
    wbuf = torch.zeros(dims.n_fibers + 1, device="cuda")
    wbuf[1:] = w.cuda()
    ybuf = torch.zeros(dims.signal_len + 1, device="cuda")
    L.dsc_sequential(p.tensor, p.dictionary, wbuf[1:], ybuf[1:])
    assert rel_l2(ybuf[1:].cpu().numpy(), ref) <= TOL32
    gbuf = torch.zeros(dims.n_fibers + 1, device="cuda")
    L.wc_sequential(p.tensor, p.dictionary, ybuf[1:], gbuf[1:])
    assert float(gbuf[0]) == 0.0 and float(gbuf[1:].abs().sum()) > 0
    op = L.DeviceOperator(p.tensor, p.dictionary)
    rc = L._native.lib().life_dsc_f32(op.handle, ctypes.c_void_p(wbuf[1:].data_ptr()),
                                      ctypes.c_void_p(ybuf.data_ptr()), None, 0, None, None)
    assert rc == 22  # LIFE_ERR_INVALID_ARGUMENT
    torch.cuda.synchronize()


def test_solver_nan_propagates():
    """A non-finite signal yields NaN weights/objective like np.maximum would,
    not silently finite weights."""
    dims = L.Dims(10, 30, 20, 8, 300)
    p = L.generate(L.GenConfig(dims=dims, mean_run_length=4.0, noise_sigma=0.1, seed=9))
    y = p.y.copy()
    y[3] = np.nan
    q = L.Problem(tensor=p.tensor, dictionary=p.dictionary, y=y)
    for precision in ("fp32", "fp64"):
        w, tr = L.solve(q, config=L.SolverConfig(max_iters=4, grad_tol=0.0, precision=precision))
        assert not np.all(np.isfinite(w)) and not np.isfinite(tr.final_objective)


def test_operator_cache_follows_layout():
    from paper_1905_06234_b200 import device
    dims = L.Dims(40, 200, 300, 96, 50_000)
    p = L.generate(L.GenConfig(dims=dims, mean_run_length=100.0, seed=3))
    a = device.operator_for(p.tensor, p.dictionary)
    assert device.operator_for(p.tensor, p.dictionary) is a
    try:
        device.set_layout("sparse")
        b = device.operator_for(p.tensor, p.dictionary)
        assert b is not a and b.kind == "sparse"
    finally:
        device.set_layout("auto")
    assert device.operator_for(p.tensor, p.dictionary).kind != "sparse"
