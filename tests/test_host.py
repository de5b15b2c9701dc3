"""Host-side logic of the drop-in package (no GPU needed).

Plans, strategies, validation and the generator's random draws must equal
the reference's (golden vectors made by the reference itself)."""

import hashlib

import numpy as np
import pytest

import paper_1905_06234_b200 as L
from paper_1905_06234_b200 import datagen
from paper_1905_06234_b200.errors import (
    ConfigInvalid,
    IndexOutOfRange,
    LengthMismatch,
    NonFiniteValue,
    PlanTensorMismatch,
    StrategyRequiresSorted,
)

from conftest import golden_problem


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).view(np.uint8).tobytes()).hexdigest()


def _tensor(g, seed, ordering="unsorted", perm=None):
    p = golden_problem(g, seed)
    d = L.Dims(*p["dims"])
    idx = slice(None) if perm is None else perm
    return L.PhiTensor(atoms=p["atoms"][idx], voxels=p["voxels"][idx],
                       fibers=p["fibers"][idx], values=p["values"][idx], dims=d,
                       ordering=ordering)


def test_dims_and_types():
    with pytest.raises(ConfigInvalid):
        L.Dims(0, 1, 1, 1, 0)
    with pytest.raises(ConfigInvalid):
        L.Dims(1, 1, 1, 1, 2)
    d = L.Dims(3, 1, 1, 96, 2)
    t = L.PhiTensor(atoms=[0, 2], voxels=[0, 0], fibers=[0, 0], values=[1.0, 1.0], dims=d)
    assert t.atoms.dtype == np.uint32 and t.values.dtype == np.float64
    assert L.precompute_offsets(t).atom_offsets.tolist() == [0, 192]  # test_tensor.py:99-104
    with pytest.raises(ValueError):
        t.values[0] = 2.0
    with pytest.raises(TypeError):
        L.PhiTensor(atoms=[0.0], voxels=[0], fibers=[0], values=[1.0], dims=L.Dims(1, 1, 1, 1, 1))
    with pytest.raises(ConfigInvalid):
        L.PhiTensor(atoms=[0], voxels=[0], fibers=[0], values=[1.0], dims=L.Dims(1, 1, 1, 1, 1),
                    ordering="by_value")


def test_validate_first_issue_per_category():
    d = L.Dims(2, 2, 2, 1, 3)
    t = L.PhiTensor(atoms=[0, 5, 1], voxels=[0, 0, 0], fibers=[0, 1, 1],
                    values=[1.0, np.nan, 2.0], dims=d)
    rep = L.validate(t, L.Dictionary(data=[1.0, 2.0], dims=d), y=np.zeros(3))
    kinds = [type(i) for i in rep.issues]
    assert kinds == [LengthMismatch, IndexOutOfRange, NonFiniteValue]
    assert rep.issues[1].position == 1 and rep.issues[2].position == 1
    with pytest.raises(LengthMismatch):
        rep.raise_first()


@pytest.mark.parametrize("seed", range(30))
def test_plans_match_reference(golden, oracle, seed):
    g = golden
    pre = f"s{seed}_"
    perm = g[pre + "perm_voxel"]
    s = _tensor(g, seed, "by_voxel", perm)
    for T in (2, 3, 4, 8):
        plan = L.build_plan(s, L.PartitionStrategy("coefficient", sync_free=True), T)
        assert np.array_equal(np.array(plan.chunks).reshape(-1, 2), g[pre + f"plan_sf_{T}"])
        plan = L.build_plan(s, L.PartitionStrategy("voxel"), T)
        assert np.array_equal(np.array(plan.chunks).reshape(-1, 2), g[pre + f"plan_voxel_{T}"])


def test_plan_errors():
    d = L.Dims(1, 8, 2, 1, 10)
    t = L.PhiTensor(atoms=np.zeros(10, int), voxels=[0, 0, 1, 1, 4, 4, 4, 5, 5, 7],
                    fibers=np.zeros(10, int), values=np.ones(10), dims=d, ordering="by_voxel")
    plan = L.build_plan(t, L.PartitionStrategy("coefficient", sync_free=True), 2)
    assert plan.chunks == ((0, 4), (4, 10))  # test_engine.py:121-129
    u = L.PhiTensor(atoms=t.atoms, voxels=t.voxels, fibers=t.fibers, values=t.values, dims=d)
    with pytest.raises(StrategyRequiresSorted):
        L.build_plan(u, L.PartitionStrategy("coefficient", sync_free=True), 2)
    with pytest.raises(StrategyRequiresSorted):
        L.build_plan(t, L.PartitionStrategy("atom"), 2)
    with pytest.raises(ConfigInvalid):
        L.build_plan(t, L.PartitionStrategy("coefficient"), 0)
    with pytest.raises(ConfigInvalid):
        L.PartitionStrategy("warp")
    # giant run swallows every boundary (test_edge_cases.py:119-135)
    g = L.PhiTensor(atoms=np.zeros(12, int), voxels=np.zeros(12, int),
                    fibers=np.zeros(12, int), values=np.ones(12),
                    dims=L.Dims(2, 2, 3, 2, 12), ordering="by_voxel")
    plan = L.build_plan(g, L.PartitionStrategy("coefficient", sync_free=True), 4)
    assert [(s, e) for s, e in plan.chunks if e > s] == [(0, 12)]
    # bad coverage is caught before any device work
    bad = L.ExecutionPlan(strategy=L.PartitionStrategy("coefficient"), threads=1,
                          chunks=((0, 11),))
    with pytest.raises(PlanTensorMismatch):
        L.engine._check_coverage(bad, 10)


def test_solver_config_validation():
    with pytest.raises(ConfigInvalid):
        L.SolverConfig(max_iters=0)
    with pytest.raises(ConfigInvalid):
        L.SolverConfig(grad_tol=-1.0)
    with pytest.raises(ConfigInvalid):
        L.SolverConfig(threads=0)
    with pytest.raises(ConfigInvalid):
        L.SolverConfig(dsc_restructure="bogus")
    with pytest.raises(ConfigInvalid):
        L.SolverConfig(precision="fp16")


def test_projections():
    assert L.project_nonneg(np.array([-1.0, 0.0, 2.0])).tolist() == [0.0, 0.0, 2.0]
    gt = L.project_gradient(np.array([3.0, -1.0, 4.0, -2.0]), np.array([0.0, 0.0, 1.0, 2.0]))
    assert gt.tolist() == [0.0, -1.0, 4.0, -2.0]  # test_sbbnnls.py:68-73


@pytest.mark.parametrize("seed", range(30))
def test_generator_draws_bitwise(golden, oracle, seed):
    """The package generator's random arrays equal the reference's; y (which
    needs a DSC) is completed here with the oracle only to pin the draws."""
    g = golden_problem(golden, seed)
    rng = np.random.default_rng(seed)
    over = dict(n_atoms=int(rng.integers(1, 31)), n_voxels=int(rng.integers(1, 51)),
                n_fibers=int(rng.integers(1, 41)), n_dirs=int(rng.choice([1, 8, 16])),
                n_coeffs=int(rng.integers(1, 501)))
    over["n_coeffs"] = min(over["n_coeffs"],
                           over["n_atoms"] * over["n_voxels"] * over["n_fibers"])
    d = L.Dims(**over)
    mean_run = float(rng.uniform(1.0, min(8.0, d.n_coeffs)))
    cfg = L.GenConfig(dims=d, mean_run_length=mean_run, weight_density=0.5,
                      noise_sigma=0.1, seed=seed)
    t, dic, w_true, noise = datagen.draw_arrays(cfg)
    for name in ("atoms", "voxels", "fibers", "values"):
        assert np.array_equal(getattr(t, name), g[name]), name
    assert np.array_equal(dic.data, g["dict"])
    assert np.array_equal(w_true, g["w_true"])
    q = dict(g)
    y = np.zeros(d.signal_len)
    oracle.dsc(q, w_true, y)
    assert np.array_equal(y + noise, g["y"])


def test_generator_draws_c1_hashes(golden_hashes):
    rec = golden_hashes["medium"]
    d = L.Dims(*rec["dims"])
    cfg = L.GenConfig(dims=d, mean_run_length=rec["mean_run_length"],
                      weight_density=rec["weight_density"], noise_sigma=rec["noise_sigma"],
                      seed=rec["seed"])
    t, dic, w_true, _ = datagen.draw_arrays(cfg)
    for name in ("atoms", "voxels", "fibers", "values"):
        assert sha(getattr(t, name)) == rec["sha_" + name]
    assert sha(dic.data) == rec["sha_dict"] and sha(w_true) == rec["sha_w_true"]


def test_solve_validates_strategy_pairs_like_the_reference():
    """sbbnnls._runners builds a plan per op (sbbnnls.py:119-167); the drop-in
    raises the same errors before touching the device."""
    from paper_1905_06234_b200.errors import StrategyRequiresSorted
    from paper_1905_06234_b200.sbbnnls import check_restructure_pairs
    ok = L.SolverConfig()
    check_restructure_pairs("unsorted", ok)   # voxel/atom defaults pass
    bad = [
        L.SolverConfig(dsc_strategy=L.PartitionStrategy("fiber")),               # by_voxel copy
        L.SolverConfig(wc_strategy=L.PartitionStrategy("coefficient", sync_free=True)),  # by_atom
        L.SolverConfig(dsc_restructure="none"),   # best_partition: coefficient, no sync-free
    ]
    check_restructure_pairs("unsorted", bad[2])
    for cfg in bad[:2]:
        with pytest.raises(StrategyRequiresSorted):
            check_restructure_pairs("unsorted", cfg)
    cfg = L.SolverConfig(dsc_restructure="none",
                         dsc_strategy=L.PartitionStrategy("coefficient", sync_free=True))
    with pytest.raises(StrategyRequiresSorted):
        check_restructure_pairs("unsorted", cfg)
    check_restructure_pairs("by_voxel", cfg)   # the tensor itself is voxel-sorted
    d = L.Dims(1, 1, 1, 1, 1)
    t = L.PhiTensor(atoms=[0], voxels=[0], fibers=[0], values=[1.0], dims=d)
    p = L.Problem(tensor=t, dictionary=L.Dictionary(data=[1.0], dims=d), y=np.array([1.0]))
    with pytest.raises(StrategyRequiresSorted):   # raised before any CUDA work
        L.solve(p, config=bad[0])
