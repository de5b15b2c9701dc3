"""Golden records at the configurations bench.py measures, from the REFERENCE.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python tests/golden/make_golden_scale.py

Writes
  tests/golden/golden_scale.json  per-config digests, norms, per-iteration traces
  tests/golden/golden_scale.npz   C1 50-iteration SBBNNLS weights (full, f64),
                                  C2 5-iteration SBBNNLS weights (full, f32-rounded),
                                  sampled slices of the C2 DSC / WC outputs

Configs (BASELINE.json configs[0] and [1]):
  c1: Dims(1057, 10_000, 20_000, 96, 5_000_000), mean run 520, noise 0.1, seed 0;
      solve(max_iters=50, grad_tol=0) on 8 threads (sbbnnls.py:223-291).
  c2: Dims(1057, 200_000, 500_000, 96, 100_000_000), mean run 520, noise 0.1, seed 0
      (bench.py's workload); dsc_sequential(w_true), wc_sequential(y) (the
      reference kernels _kernels.py:14-68 on the tensor as generated) and
      solve(max_iters=5, grad_tol=0) on 8 threads.

Nothing at test time reads /root/reference: the committed files are the
reference's own outputs.
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
N_SAMPLE = 16384


def sha(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.view(np.uint8).tobytes()).hexdigest()


def sample_idx(n, seed):
    return np.sort(np.random.default_rng(seed).choice(n, size=min(N_SAMPLE, n), replace=False))


def trace_rec(tr):
    return dict(objective=[float(r.objective) for r in tr.records],
                alpha=[float(r.alpha) for r in tr.records],
                grad_norm=[float(r.grad_norm) for r in tr.records],
                zeros=[int(r.zeros) for r in tr.records],
                dsc_skipped=[int(r.dsc_skipped) for r in tr.records],
                initial_objective=float(tr.initial_objective),
                final_objective=float(tr.final_objective),
                termination=str(tr.termination))


def c1(store):
    t0 = time.time()
    dims = L.Dims(1057, 10_000, 20_000, 96, 5_000_000)
    p = L.generate(L.GenConfig(dims=dims, mean_run_length=520.0, weight_density=0.5,
                               noise_sigma=0.1, seed=0))
    w, tr = L.solve(p, config=L.SolverConfig(max_iters=50, grad_tol=0.0, threads=8))
    store["c1_solve50_w"] = w
    rec = dict(dims=[1057, 10_000, 20_000, 96, 5_000_000], mean_run_length=520.0,
               noise_sigma=0.1, seed=0, solve_iters=50, solve_threads=8,
               sha_y=sha(p.y), sha_solve_w=sha(w), solve_w_norm=float(np.linalg.norm(w)),
               **{"solve_" + k: v for k, v in trace_rec(tr).items()})
    rec["seconds"] = time.time() - t0
    print("c1", f"{rec['seconds']:.1f}s", flush=True)
    return rec


def c2(store):
    t0 = time.time()
    dims = L.Dims(1057, 200_000, 500_000, 96, 100_000_000)
    p = L.generate(L.GenConfig(dims=dims, mean_run_length=520.0, weight_density=0.5,
                               noise_sigma=0.1, seed=0))
    rec = dict(dims=[1057, 200_000, 500_000, 96, 100_000_000], mean_run_length=520.0,
               noise_sigma=0.1, seed=0)
    for k in ("atoms", "voxels", "fibers", "values"):
        rec["sha_" + k] = sha(getattr(p.tensor, k))
    rec["sha_dict"] = sha(p.dictionary.data)
    rec["sha_y"] = sha(p.y)
    rec["sha_w_true"] = sha(p.w_true)
    print("c2 generated", f"{time.time() - t0:.1f}s", flush=True)
    off = L.precompute_offsets(p.tensor)
    # DSC of w_true (the generator's own product, without the noise)
    y = L.zeros_signal(p.dims)
    st = L.dsc_sequential(off, p.dictionary, p.w_true, y)
    rec["sha_dsc_w_true"] = sha(y)
    rec["norm_dsc_w_true"] = float(np.linalg.norm(y))
    rec["skipped_dsc_w_true"] = int(st.skipped_coefficients)
    iy = sample_idx(y.size, 1)
    store["c2_dsc_w_true_idx"] = iy.astype(np.int64)
    store["c2_dsc_w_true_val"] = y[iy]
    del y
    print("c2 dsc", f"{time.time() - t0:.1f}s", flush=True)
    # WC of the noisy signal
    w = L.zeros_weights(p.dims)
    L.wc_sequential(off, p.dictionary, p.y, w)
    rec["sha_wc_y"] = sha(w)
    rec["norm_wc_y"] = float(np.linalg.norm(w))
    iw = sample_idx(w.size, 2)
    store["c2_wc_y_idx"] = iw.astype(np.int64)
    store["c2_wc_y_val"] = w[iw]
    del off
    print("c2 wc", f"{time.time() - t0:.1f}s", flush=True)
    w, tr = L.solve(p, config=L.SolverConfig(max_iters=5, grad_tol=0.0, threads=8))
    store["c2_solve5_w_f32"] = w.astype(np.float32)
    rec.update(solve_iters=5, solve_threads=8, sha_solve_w=sha(w),
               solve_w_norm=float(np.linalg.norm(w)),
               **{"solve_" + k: v for k, v in trace_rec(tr).items()})
    rec["seconds"] = time.time() - t0
    print("c2", f"{rec['seconds']:.1f}s", flush=True)
    return rec


def main():
    store = {}
    recs = {"c1": c1(store), "c2": c2(store)}
    recs["_generator"] = {"numpy": np.__version__, "reference": L.__version__,
                          "script": "tests/golden/make_golden_scale.py"}
    np.savez_compressed(os.path.join(OUT, "golden_scale.npz"), **store)
    with open(os.path.join(OUT, "golden_scale.json"), "w") as f:
        json.dump(recs, f, indent=1)


if __name__ == "__main__":
    main()
