"""CPU oracle for the LiFE hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only tests/,
``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product package
(``paper_1905_06234_b200``) must not import, load or call anything here.

It restates the reference package ``lifespmv`` (``/root/reference/pkg``) as
numpy + the C kernels in ``life_oracle.c`` (built by ``oracle/Makefile``):

* ``generate``       <- lifespmv.datagen.generate      datagen.py:65-123
* ``small_problem``  <- tests/conftest.small_problem   tests/conftest.py:20-36
* ``dsc`` / ``wc``   <- engine.dsc_sequential / wc_sequential
                        engine.py:218-244 over _kernels.py:14-68
* ``dsc_chunks`` / ``wc_chunks`` <- engine.dsc_parallel / wc_parallel
                        engine.py:247-413 (three conflict regimes)
* ``stable_argsort`` <- restructure.sort_by            restructure.py:54-73
* ``detect_runs``    <- restructure.detect_runs        restructure.py:76-92
* ``build_plan``     <- engine.build_plan              engine.py:113-184
* ``solve``          <- sbbnnls.solve                  sbbnnls.py:102-291

Parity is PINNED: tests/test_oracle.py checks every routine bit-for-bit
against golden vectors the reference itself produced
(tests/golden/make_golden.py).
"""

import ctypes
import math
import os
import subprocess
import time

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liblife_oracle.so")
_lib = None

_u32p = np.ctypeslib.ndpointer(dtype=np.uint32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i64 = ctypes.c_int64


def build():
    """Compile liblife_oracle.so in place (gcc, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.lo_dsc_range.restype = _i64
        L.lo_dsc_range.argtypes = [_u32p, _u32p, _u32p, _f64p, _f64p, _f64p,
                                   _f64p, _i64, _i64, _i64, ctypes.c_int]
        L.lo_wc_range.restype = None
        L.lo_wc_range.argtypes = [_u32p, _u32p, _u32p, _f64p, _f64p, _f64p,
                                  _f64p, _i64, _i64, _i64]
        L.lo_dsc_chunks_owned.restype = None
        L.lo_dsc_chunks_owned.argtypes = [_u32p, _u32p, _u32p, _f64p, _f64p,
                                          _f64p, _f64p, _i64p, ctypes.c_int,
                                          _i64, ctypes.c_int, _i64p]
        L.lo_dsc_chunks_edge.restype = None
        L.lo_dsc_chunks_edge.argtypes = [_u32p, _u32p, _u32p, _f64p, _f64p,
                                         _f64p, _f64p, _i64p, ctypes.c_int,
                                         _i64, _i64, ctypes.c_int, _i64p]
        L.lo_dsc_chunks_full.restype = None
        L.lo_dsc_chunks_full.argtypes = [_u32p, _u32p, _u32p, _f64p, _f64p,
                                         _f64p, _f64p, _i64p, ctypes.c_int,
                                         _i64, _i64, ctypes.c_int, _i64p]
        L.lo_wc_chunks.restype = None
        L.lo_wc_chunks.argtypes = [_u32p, _u32p, _u32p, _f64p, _f64p, _f64p,
                                   _f64p, _i64p, ctypes.c_int, _i64, _i64,
                                   ctypes.c_int]
        L.lo_stable_argsort_u32.restype = ctypes.c_int
        L.lo_stable_argsort_u32.argtypes = [_u32p, _i64, _i64p]
        L.lo_detect_runs.restype = _i64
        L.lo_detect_runs.argtypes = [_u32p, _i64, _i64p, _u32p]
        L.lo_snap.restype = None
        L.lo_snap.argtypes = [_u32p, _i64, _i64p, ctypes.c_int]
        L.lo_max_threads.restype = ctypes.c_int
        L.lo_set_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def set_threads(n):
    lib().lo_set_threads(int(n))


def max_threads():
    return int(lib().lo_max_threads())


# --------------------------------------------------------------------------
# Problem container: a plain dict of arrays keeps the oracle independent of
# any host type in the product package.
#   atoms, voxels, fibers : u32[Nc]; values : f64[Nc]; dict : f64[Na*Nd]
#   y : f64[Nv*Nd] or None;  w_true : f64[Nf] or None
#   dims : (Na, Nv, Nf, Nd, Nc);  ordering : "unsorted"|"by_atom"|...
# --------------------------------------------------------------------------


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _geometric_runs(rng, nc, mean):
    """Truncated geometric run lengths summing to nc (datagen.py:65-80).

    Draws whole batches exactly as the reference loop does (the batch is
    always drawn in full, the loop stops inside it), so the PCG64 stream
    advances identically."""
    if nc == 0:
        return np.empty(0, dtype=np.int64)
    p = 1.0 / mean
    parts = []
    left = nc
    while left > 0:
        batch = rng.geometric(p, size=max(16, int(left * p) + 1)).astype(np.int64)
        csum = np.cumsum(batch)
        stop = int(np.searchsorted(csum, left, side="left"))
        if stop < len(batch):
            take = batch[:stop + 1].copy()
            take[-1] = left - (csum[stop - 1] if stop > 0 else 0)
            parts.append(take)
            left = 0
        else:
            parts.append(batch)
            left -= int(csum[-1])
    return np.concatenate(parts)


def draw(dims, mean_run_length=4.0, weight_density=0.5, noise_sigma=0.0,
         seed=0):
    """The random part of datagen.generate (datagen.py:83-113, 117-118):
    tensor, dictionary, w_true and the noise vector, in the reference's
    PCG64 call order.  y itself needs a DSC; see ``generate``."""
    na, nv, nf, nd, nc = dims
    rng = np.random.default_rng(seed)
    lengths = _geometric_runs(rng, nc, mean_run_length)
    n_runs = len(lengths)
    if n_runs <= nv:
        run_voxels = rng.choice(nv, size=n_runs, replace=False)
    else:
        run_voxels = rng.integers(0, nv, size=n_runs)
    voxels = np.repeat(run_voxels.astype(np.uint32), lengths)
    atoms = rng.integers(0, na, size=nc, dtype=np.uint32)
    fibers = rng.integers(0, nf, size=nc, dtype=np.uint32)
    values = 1.0 - rng.random(nc)
    order = rng.permutation(nc)
    rows = rng.standard_normal((na, nd))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    n_active = max(1, round(weight_density * nf))
    w_true = np.zeros(nf)
    active = rng.choice(nf, size=n_active, replace=False)
    w_true[active] = 1.0 - rng.random(n_active)
    noise = None
    if noise_sigma > 0.0:
        noise = noise_sigma * rng.standard_normal(nv * nd)
    return dict(atoms=_u32(atoms[order]), voxels=_u32(voxels[order]),
                fibers=_u32(fibers[order]), values=_f64(values[order]),
                dict=_f64(rows.ravel()), w_true=w_true, noise=noise,
                dims=tuple(int(x) for x in dims), ordering="unsorted")


def generate(dims, mean_run_length=4.0, weight_density=0.5, noise_sigma=0.0,
             seed=0):
    """Bit-identical restatement of lifespmv.generate (datagen.py:83-123)."""
    p = draw(dims, mean_run_length, weight_density, noise_sigma, seed)
    y = np.zeros(p["dims"][1] * p["dims"][3])
    dsc(p, p["w_true"], y)
    if p["noise"] is not None:
        y += p["noise"]
    p["y"] = y
    return p


def small_problem(seed, noise=0.1, **over):
    """tests/conftest.py:20-36 restated (desk-scale seeded instance)."""
    rng = np.random.default_rng(seed)
    d = dict(n_atoms=int(rng.integers(1, 31)), n_voxels=int(rng.integers(1, 51)),
             n_fibers=int(rng.integers(1, 41)),
             n_dirs=int(rng.choice([1, 8, 16])),
             n_coeffs=int(rng.integers(1, 501)))
    d.update(over)
    d["n_coeffs"] = min(d["n_coeffs"],
                        d["n_atoms"] * d["n_voxels"] * d["n_fibers"])
    mean_run = float(rng.uniform(1.0, min(8.0, d["n_coeffs"])))
    dims = (d["n_atoms"], d["n_voxels"], d["n_fibers"], d["n_dirs"],
            d["n_coeffs"])
    return generate(dims, mean_run, 0.5, noise, seed)


# ---- kernels ------------------------------------------------------------


def dsc(p, w, y, skip_zero=True, start=0, end=None):
    """y += M w over coefficients [start, end) in storage order; returns the
    zero-skip count (engine.dsc_sequential, engine.py:218-233)."""
    end = p["dims"][4] if end is None else end
    return int(lib().lo_dsc_range(p["atoms"], p["voxels"], p["fibers"],
                                  p["values"], p["dict"], _f64(w), y, start,
                                  end, p["dims"][3], int(bool(skip_zero))))


def wc(p, y, w, start=0, end=None):
    """w += M^T y over [start, end) (engine.wc_sequential, engine.py:236-244)."""
    end = p["dims"][4] if end is None else end
    lib().lo_wc_range(p["atoms"], p["voxels"], p["fibers"], p["values"],
                      p["dict"], _f64(y), w, start, end, p["dims"][3])


def _flat_chunks(chunks):
    return np.ascontiguousarray(np.asarray(chunks, dtype=np.int64).reshape(-1))


def _on_runs(keys, chunks):
    n = len(keys)
    for s, _ in chunks[1:]:
        if 0 < s < n and keys[s - 1] == keys[s]:
            return False
    return True


def dsc_chunks(p, w, y, chunks, aligned, skip_zero=True):
    """engine.dsc_parallel regimes (engine.py:263-273); returns skip total."""
    nc, nd = p["dims"][4], p["dims"][3]
    flat = _flat_chunks(chunks)
    skips = np.zeros(len(chunks), dtype=np.int64)
    args = (p["atoms"], p["voxels"], p["fibers"], p["values"], p["dict"],
            _f64(w), y, flat, len(chunks))
    if aligned:
        lib().lo_dsc_chunks_owned(*args, nd, int(bool(skip_zero)), skips)
    elif p["ordering"] == "by_voxel":
        lib().lo_dsc_chunks_edge(*args, nc, nd, int(bool(skip_zero)), skips)
    else:
        lib().lo_dsc_chunks_full(*args, len(y), nd, int(bool(skip_zero)), skips)
    return int(skips.sum())


def wc_chunks(p, y, w, chunks, kind="coefficient"):
    """engine.wc_parallel (engine.py:387-413)."""
    owned = kind == "fiber" or (p["ordering"] == "by_fiber"
                                and _on_runs(p["fibers"], chunks))
    lib().lo_wc_chunks(p["atoms"], p["voxels"], p["fibers"], p["values"],
                       p["dict"], _f64(y), w, _flat_chunks(chunks), len(chunks),
                       p["dims"][2], p["dims"][3], int(owned))


# ---- restructuring ------------------------------------------------------


def stable_argsort(keys):
    keys = _u32(keys)
    perm = np.empty(len(keys), dtype=np.int64)
    if lib().lo_stable_argsort_u32(keys, len(keys), perm) != 0:
        raise MemoryError("oracle argsort")
    return perm


def sort_by(p, key):
    """restructure.sort_by (restructure.py:54-73): (sorted problem, perm)."""
    perm = stable_argsort(p[key + "s"])
    q = dict(p)
    for name in ("atoms", "voxels", "fibers", "values"):
        q[name] = np.ascontiguousarray(p[name][perm])
    q["ordering"] = "by_" + key
    return q, perm


def detect_runs(keys):
    keys = _u32(keys)
    n = len(keys)
    b = np.empty(n + 1, dtype=np.int64)
    k = np.empty(max(n, 1), dtype=np.uint32)
    r = int(lib().lo_detect_runs(keys, n, b, k))
    return b[:r + 1].copy(), k[:r].copy()


def build_plan(p, kind, sync_free, threads):
    """engine.build_plan chunk boundaries (engine.py:139-184)."""
    nc = p["dims"][4]
    if kind == "coefficient":
        size = math.ceil(nc / threads) if nc else 0
        bounds = [min(i * size, nc) for i in range(threads + 1)]
        if sync_free:
            b = np.asarray(bounds, dtype=np.int64)
            lib().lo_snap(p["voxels"], nc, b, len(b))
            bounds = b.tolist()
    else:
        keys = p[kind + "s"]
        if nc == 0:
            bounds = [0] * (threads + 1)
        else:
            starts, _ = detect_runs(keys)
            n_runs = len(starts) - 1
            per = math.ceil(n_runs / threads)
            bounds = [int(starts[min(i * per, n_runs)]) for i in range(threads + 1)]
    return tuple((int(bounds[i]), int(bounds[i + 1])) for i in range(threads))


# ---- SBBNNLS (sbbnnls.py:102-291) ----------------------------------------


def project_gradient(g, w):
    out = g.copy()
    out[(w == 0.0) & (g > 0.0)] = 0.0
    return out


def solve(p, w0=None, max_iters=500, grad_tol=1e-12, threads=1,
          dsc_key="voxel", wc_key="atom", skip_zero=True):
    """Alg. 1 with the reference's default operator pairing: DSC on the
    voxel-sorted copy with the sync-free coefficient plan, WC on the
    atom-sorted copy with the coefficient plan (sbbnnls.py:47-48,
    restructure.py:95-104).  Returns (w, trace dict)."""
    b = p["y"]
    nv, nf, nd = p["dims"][1], p["dims"][2], p["dims"][3]
    ops = {}
    for op, key in (("dsc", dsc_key), ("wc", wc_key)):
        q = p if key == "none" else sort_by(p, key)[0]
        sync_free = op == "dsc" and key == "voxel"
        ops[op] = (q, build_plan(q, "coefficient", sync_free, threads), sync_free)
    calls = {"dsc": 0, "wc": 0}
    last_skip = [0]

    def mv(w):
        q, chunks, aligned = ops["dsc"]
        y = np.zeros(nv * nd)
        last_skip[0] = dsc_chunks(q, w, y, chunks, aligned, skip_zero)
        calls["dsc"] += 1
        return y

    def mtv(y):
        q, chunks, _ = ops["wc"]
        w = np.zeros(nf)
        wc_chunks(q, y, w, chunks)
        calls["wc"] += 1
        return w

    if w0 is None:
        ones = np.ones(nf)
        scale = np.linalg.norm(b) / max(np.linalg.norm(mv(ones)), 1e-300)
        w = ones * scale
    else:
        w = np.maximum(np.asarray(w0, dtype=np.float64), 0.0)
    recs = []
    term = ""
    init_obj = final_obj = float("nan")
    for i in range(1, max_iters + 1):
        c0 = (calls["dsc"], calls["wc"])
        r = mv(w) - b
        skipped = last_skip[0]
        obj = 0.5 * float(np.dot(r, r))
        if i == 1:
            init_obj = obj
        gt = project_gradient(mtv(r), w)
        gnorm = float(np.linalg.norm(gt))
        if gnorm < grad_tol:
            term, final_obj = "grad_tol", obj
            break
        mg = mv(gt)
        if i % 2 == 1:
            num, den = float(np.dot(gt, gt)), float(np.dot(mg, mg))
        else:
            mtmg = mtv(mg)
            num, den = float(np.dot(mg, mg)), float(np.dot(mtmg, mtmg))
        if den == 0.0:
            term, final_obj = "degenerate_step", obj
            break
        alpha = num / den
        w = np.maximum(w - alpha * gt, 0.0)
        recs.append(dict(iteration=i, objective=obj, alpha=alpha,
                         grad_norm=gnorm, zeros=int(np.count_nonzero(w == 0.0)),
                         dsc_calls=calls["dsc"] - c0[0],
                         wc_calls=calls["wc"] - c0[1], dsc_skipped=skipped,
                         w_min=float(w.min()) if len(w) else 0.0,
                         t=time.perf_counter()))
    else:
        term = "max_iters"
        r = mv(w) - b
        final_obj = 0.5 * float(np.dot(r, r))
    return w, dict(records=recs, termination=term, initial_objective=init_obj,
                   final_objective=final_obj, total_dsc_calls=calls["dsc"],
                   total_wc_calls=calls["wc"])
