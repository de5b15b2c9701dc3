"""Generate golden vectors from the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python tests/golden/make_golden.py

Writes tests/golden/golden_small.npz (desk-scale inputs + outputs) and
tests/golden/golden.json (SHA-256 digests of larger, regenerable cases).
Nothing at test time reads /root/reference; the committed fixtures are the
reference's outputs.
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import lifespmv as L  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.view(np.uint8).tobytes()).hexdigest()


def small_problem(seed, noise=0.1, **over):
    # verbatim semantics of /root/reference/pkg/tests/conftest.py:20-36
    rng = np.random.default_rng(seed)
    d = dict(n_atoms=int(rng.integers(1, 31)), n_voxels=int(rng.integers(1, 51)),
             n_fibers=int(rng.integers(1, 41)),
             n_dirs=int(rng.choice([1, 8, 16])),
             n_coeffs=int(rng.integers(1, 501)))
    d.update(over)
    d["n_coeffs"] = min(d["n_coeffs"], d["n_atoms"] * d["n_voxels"] * d["n_fibers"])
    dims = L.Dims(**d)
    mean_run = float(rng.uniform(1.0, min(8.0, dims.n_coeffs)))
    return L.generate(L.GenConfig(dims=dims, mean_run_length=mean_run,
                                  weight_density=0.5, noise_sigma=noise, seed=seed))


def dims_tuple(d):
    return [d.n_atoms, d.n_voxels, d.n_fibers, d.n_dirs, d.n_coeffs]


def small_cases(store):
    for seed in range(30):
        p = small_problem(seed)
        t = p.tensor
        pre = f"s{seed}_"
        store[pre + "dims"] = np.array(dims_tuple(p.dims), dtype=np.int64)
        for name in ("atoms", "voxels", "fibers", "values"):
            store[pre + name] = getattr(t, name)
        store[pre + "dict"] = p.dictionary.data
        store[pre + "y"] = p.y
        store[pre + "w_true"] = p.w_true
        rng = np.random.default_rng(seed + 1000)
        w_in = rng.standard_normal(p.dims.n_fibers)
        y_in = rng.standard_normal(p.dims.signal_len)
        w_sparse = np.abs(rng.standard_normal(p.dims.n_fibers))
        w_sparse[rng.random(p.dims.n_fibers) < 0.5] = 0.0
        store[pre + "w_in"], store[pre + "y_in"] = w_in, y_in
        store[pre + "w_sparse"] = w_sparse
        off = L.precompute_offsets(t)
        y = L.zeros_signal(p.dims)
        st = L.dsc_sequential(off, p.dictionary, w_in, y)
        store[pre + "dsc_w_in"] = y
        store[pre + "dsc_w_in_skipped"] = np.int64(st.skipped_coefficients)
        y = L.zeros_signal(p.dims)
        st = L.dsc_sequential(off, p.dictionary, w_sparse, y)
        store[pre + "dsc_w_sparse"] = y
        store[pre + "dsc_w_sparse_skipped"] = np.int64(st.skipped_coefficients)
        w = L.zeros_weights(p.dims)
        L.wc_sequential(off, p.dictionary, y_in, w)
        store[pre + "wc_y_in"] = w
        for key in ("atom", "voxel", "fiber"):
            s, perm = L.sort_by(t, key)
            store[pre + "perm_" + key] = perm
            runs = L.detect_runs(s)
            store[pre + "runs_" + key] = runs.boundaries
            store[pre + "runkeys_" + key] = runs.key_values
            # sorted-copy kernels (restructuring invariance, test_acceptance:73-109)
            soff = L.precompute_offsets(s)
            y = L.zeros_signal(p.dims)
            L.dsc_sequential(soff, p.dictionary, w_in, y)
            store[pre + "dsc_sorted_" + key] = y
            w = L.zeros_weights(p.dims)
            L.wc_sequential(soff, p.dictionary, y_in, w)
            store[pre + "wc_sorted_" + key] = w
            if key == "voxel":
                for T in (2, 3, 4, 8):
                    plan = L.build_plan(s, L.PartitionStrategy("coefficient", True), T)
                    store[pre + f"plan_sf_{T}"] = np.array(plan.chunks, dtype=np.int64)
                    plan = L.build_plan(s, L.PartitionStrategy("voxel"), T)
                    store[pre + f"plan_voxel_{T}"] = np.array(plan.chunks, dtype=np.int64)
                    # edge-private regime on a plain coefficient split
                    plan = L.build_plan(soff, L.PartitionStrategy("coefficient"), T)
                    y = L.zeros_signal(p.dims)
                    L.dsc_parallel(soff, p.dictionary, w_in, y, plan)
                    store[pre + f"dsc_edge_{T}"] = y
            # parallel WC with private buffers (engine.py:401-412)
            plan = L.build_plan(soff, L.PartitionStrategy("coefficient"), 3)
            w = L.zeros_weights(p.dims)
            L.wc_parallel(soff, p.dictionary, y_in, w, plan)
            store[pre + "wc_priv3_" + key] = w
        # full privatization on the unsorted tensor
        plan = L.build_plan(off, L.PartitionStrategy("coefficient"), 4)
        y = L.zeros_signal(p.dims)
        L.dsc_parallel(off, p.dictionary, w_in, y, plan)
        store[pre + "dsc_full4"] = y


def solver_cases(store):
    cases = []
    dims = L.Dims(n_atoms=10, n_voxels=30, n_fibers=20, n_dirs=8, n_coeffs=300)
    cases.append(("noiseless42", L.generate(L.GenConfig(dims=dims, mean_run_length=4.0,
                                                        weight_density=0.5,
                                                        noise_sigma=0.0, seed=42))))
    for seed in (3, 5, 11):
        cases.append((f"small{seed}", small_problem(seed, noise=0.1)))
    dims = L.Dims(n_atoms=40, n_voxels=400, n_fibers=600, n_dirs=16, n_coeffs=20000)
    cases.append(("mid", L.generate(L.GenConfig(dims=dims, mean_run_length=50.0,
                                                weight_density=0.5, noise_sigma=0.1,
                                                seed=5))))
    names = []
    for name, p in cases:
        for threads in (1, 4):
            cfg = L.SolverConfig(max_iters=30, grad_tol=0.0, threads=threads)
            w, tr = L.solve(p, config=cfg)
            pre = f"sol_{name}_t{threads}_"
            store[pre + "w"] = w
            store[pre + "objective"] = np.array([r.objective for r in tr.records])
            store[pre + "alpha"] = np.array([r.alpha for r in tr.records])
            store[pre + "grad_norm"] = np.array([r.grad_norm for r in tr.records])
            store[pre + "zeros"] = np.array([r.zeros for r in tr.records], dtype=np.int64)
            store[pre + "dsc_skipped"] = np.array([r.dsc_skipped for r in tr.records],
                                                  dtype=np.int64)
            store[pre + "final_objective"] = np.float64(tr.final_objective)
            store[pre + "initial_objective"] = np.float64(tr.initial_objective)
            store[pre + "termination"] = np.array(tr.termination)
        pre = f"solp_{name}_"
        store[pre + "dims"] = np.array(dims_tuple(p.dims), dtype=np.int64)
        for k in ("atoms", "voxels", "fibers", "values"):
            store[pre + k] = getattr(p.tensor, k)
        store[pre + "dict"] = p.dictionary.data
        store[pre + "y"] = p.y
        names.append(name)
    store["solver_case_names"] = np.array(names)


def hashed_case(name, dims, mean_run, noise, seed, solve_iters, threads):
    t0 = time.time()
    p = L.generate(L.GenConfig(dims=dims, mean_run_length=mean_run,
                               weight_density=0.5, noise_sigma=noise, seed=seed))
    rec = dict(dims=dims_tuple(dims), mean_run_length=mean_run, noise_sigma=noise,
               seed=seed, weight_density=0.5)
    for k in ("atoms", "voxels", "fibers", "values"):
        rec["sha_" + k] = sha(getattr(p.tensor, k))
    rec["sha_dict"] = sha(p.dictionary.data)
    rec["sha_y"] = sha(p.y)
    rec["sha_w_true"] = sha(p.w_true)
    off = L.precompute_offsets(p.tensor)
    w = L.zeros_weights(p.dims)
    L.wc_sequential(off, p.dictionary, p.y, w)
    rec["sha_wc_y"] = sha(w)
    rec["norm_wc_y"] = float(np.linalg.norm(w))
    y = L.zeros_signal(p.dims)
    st = L.dsc_sequential(off, p.dictionary, w, y)
    rec["sha_dsc_wc_y"] = sha(y)
    rec["norm_dsc_wc_y"] = float(np.linalg.norm(y))
    rec["skipped_dsc_wc_y"] = int(st.skipped_coefficients)
    for key in ("atom", "voxel", "fiber"):
        s, perm = L.sort_by(p.tensor, key)
        rec["sha_perm_" + key] = sha(perm)
        runs = L.detect_runs(s)
        rec["n_runs_" + key] = int(runs.n_runs)
        rec["sha_runs_" + key] = sha(runs.boundaries)
    if solve_iters:
        w, tr = L.solve(p, config=L.SolverConfig(max_iters=solve_iters, grad_tol=0.0,
                                                 threads=threads))
        rec["solve_iters"] = solve_iters
        rec["solve_threads"] = threads
        rec["solve_final_objective"] = float(tr.final_objective)
        rec["solve_initial_objective"] = float(tr.initial_objective)
        rec["solve_objective"] = [float(r.objective) for r in tr.records]
        rec["solve_alpha"] = [float(r.alpha) for r in tr.records]
        rec["solve_zeros"] = [int(r.zeros) for r in tr.records]
        rec["solve_w_norm"] = float(np.linalg.norm(w))
        rec["solve_w_sum"] = float(w.sum())
        rec["sha_solve_w"] = sha(w)
    rec["seconds"] = time.time() - t0
    print(name, f"{rec['seconds']:.1f}s", flush=True)
    return rec


def main():
    store = {}
    small_cases(store)
    solver_cases(store)
    np.savez_compressed(os.path.join(OUT, "golden_small.npz"), **store)
    hashed = {
        "medium": hashed_case("medium", L.Dims(64, 2000, 3000, 96, 200_000),
                              100.0, 0.1, 7, 10, 4),
        "c1": hashed_case("c1", L.Dims(1057, 10_000, 20_000, 96, 5_000_000),
                          520.0, 0.1, 0, 5, 8),
    }
    hashed["_generator"] = {"numpy": np.__version__, "reference": L.__version__}
    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(hashed, f, indent=1)


if __name__ == "__main__":
    main()
