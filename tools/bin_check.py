"""Binned two-phase products on the GPU: accuracy vs the fp64 bit-exact
kernels and timing (CUDA events) on a set of shapes, incl. duplicate-heavy
voxels (split rows), long fascicles (split virtual slots) and C1/C2.

    python tools/bin_check.py [--c2] [--skew] [--layouts bin,sparse]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_06234_b200 as L  # noqa: E402
from paper_1905_06234_b200 import _native as N, device  # noqa: E402


def custom(na, nv, nf, nt, nc, seed, zipf=None, hot_voxel=None):
    rng = np.random.default_rng(seed)
    a = rng.integers(0, na, nc, dtype=np.uint32)
    v = rng.integers(0, nv, nc, dtype=np.uint32)
    if zipf:
        f = (rng.zipf(zipf, nc) - 1) % nf
        f = f.astype(np.uint32)
    else:
        f = rng.integers(0, nf, nc, dtype=np.uint32)
    if hot_voxel:
        k = int(hot_voxel * nc)
        v[:k] = 7
    val = 1.0 - rng.random(nc)
    d = L.Dims(n_atoms=na, n_voxels=nv, n_fibers=nf, n_dirs=nt, n_coeffs=nc)
    rows = rng.standard_normal((na, nt))
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    t = L.PhiTensor(atoms=a, voxels=v, fibers=f, values=val, dims=d)
    return t, L.Dictionary(data=rows.ravel(), dims=d)


def check(name, tensor, dic, layout, reps=10):
    d = tensor.dims
    device.set_layout(layout)
    t0 = time.time()
    op = device.DeviceOperator(tensor, dic, exact=True)
    setup = time.time() - t0
    rng = np.random.default_rng(1)
    w64 = rng.random(d.n_fibers)
    w64[rng.random(d.n_fibers) < 0.3] = 0.0
    y64 = rng.standard_normal(d.signal_len)
    cu = lambda x, dt: torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dt)
    # fp64 exact references on the device
    yr = torch.zeros(d.signal_len, dtype=torch.float64, device="cuda")
    sk = torch.zeros(1, dtype=torch.int64, device="cuda")
    op.dsc_f64(cu(w64, torch.float64), yr, N.SKIP_ZERO, sk)
    wr = torch.zeros(d.n_fibers, dtype=torch.float64, device="cuda")
    op.wc_f64(cu(y64, torch.float64), wr)
    # fp32 products
    w32, yin = cu(w64, torch.float32), cu(y64, torch.float32)
    y = torch.empty(d.signal_len, dtype=torch.float32, device="cuda")
    w = torch.empty(d.n_fibers, dtype=torch.float32, device="cuda")
    sk32 = torch.zeros(1, dtype=torch.int64, device="cuda")
    sq = torch.zeros(1, dtype=torch.float64, device="cuda")
    op.dsc_f32(w32, y, None, N.SKIP_ZERO, sk32, sq)
    op.wc_f32(yin, w)
    torch.cuda.synchronize()
    e_d = (torch.linalg.norm(y.double() - yr) / torch.linalg.norm(yr)).item()
    e_w = (torch.linalg.norm(w.double() - wr) / torch.linalg.norm(wr)).item()
    sq_err = abs(sq.item() - (y.double() ** 2).sum().item()) / max(sq.item(), 1e-300)
    # repeatability
    y2 = torch.empty_like(y)
    w2 = torch.empty_like(w)
    op.dsc_f32(w32, y2, None, N.SKIP_ZERO)
    op.wc_f32(yin, w2)
    torch.cuda.synchronize()
    rep = bool(torch.equal(y, y2)) and bool(torch.equal(w, w2))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    for _ in range(3):
        op.dsc_f32(w32, y, None, N.SKIP_ZERO)
        op.wc_f32(yin, w)
    ev[0].record()
    for _ in range(reps):
        op.dsc_f32(w32, y, None, N.SKIP_ZERO)
    ev[1].record()
    for _ in range(reps):
        op.wc_f32(yin, w)
    ev[2].record()
    torch.cuda.synchronize()
    td = ev[0].elapsed_time(ev[1]) / reps
    tw = ev[1].elapsed_time(ev[2]) / reps
    print(f"{name:24s} {layout:6s} kind={op.kind:6s} dsc_err={e_d:.2e} wc_err={e_w:.2e} "
          f"skip={int(sk32.item())}/{int(sk.item())} sq_rel={sq_err:.1e} repeat={rep} "
          f"dsc={td:.3f}ms wc={tw:.3f}ms setup={setup:.2f}s", flush=True)
    ok = e_d < 1e-5 and e_w < 1e-5 and int(sk32.item()) == int(sk.item()) and rep
    op.close()
    return ok


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c2", action="store_true")
    ap.add_argument("--layouts", default="bin")
    ap.add_argument("--skew", action="store_true", help="16M/100M uniform vs Zipf fascicles vs one 5%% voxel")
    args = ap.parse_args()
    cases = [
        ("tiny", custom(64, 500, 800, 96, 40_000, 3)),
        ("dups(na=12)", custom(12, 300, 900, 96, 60_000, 4)),
        ("nt=32", custom(200, 2000, 3000, 32, 200_000, 5)),
        ("nt=45", custom(200, 2000, 3000, 45, 200_000, 6)),
        ("nt=150", custom(300, 2000, 3000, 150, 300_000, 7)),
        ("nt=192", custom(300, 2000, 3000, 192, 300_000, 8)),
        ("zipf-fascicles", custom(1057, 4000, 20_000, 96, 2_000_000, 9, zipf=1.3)),
        ("hot-voxel-5%", custom(1057, 30_000, 80_000, 96, 4_000_000, 10, hot_voxel=0.05)),
    ]
    c1 = L.generate(L.GenConfig(dims=L.Dims(1057, 10_000, 20_000, 96, 5_000_000),
                                mean_run_length=520.0, weight_density=0.5, noise_sigma=0.1, seed=0))
    cases.append(("C1", (c1.tensor, c1.dictionary)))
    if args.c2:
        c2 = L.generate(L.GenConfig(dims=L.Dims(1057, 200_000, 500_000, 96, 100_000_000),
                                    mean_run_length=520.0, weight_density=0.5, noise_sigma=0.1, seed=0))
        cases.append(("C2", (c2.tensor, c2.dictionary)))
    if args.skew:
        cases = [
            ("16M-uniform", custom(1057, 40_000, 100_000, 96, 16_000_000, 11)),
            ("16M-zipf1.3", custom(1057, 40_000, 100_000, 96, 16_000_000, 11, zipf=1.3)),
            ("16M-hot-voxel-5%", custom(1057, 40_000, 100_000, 96, 16_000_000, 11, hot_voxel=0.05)),
            ("100M-uniform", custom(1057, 200_000, 500_000, 96, 100_000_000, 12)),
            ("100M-zipf1.3", custom(1057, 200_000, 500_000, 96, 100_000_000, 12, zipf=1.3)),
        ]
    bad = 0
    for name, (t, dic) in cases:
        for lay in args.layouts.split(","):
            try:
                bad += 0 if check(name, t, dic, lay) else 1
            except Exception as e:  # report and continue
                print(f"{name:24s} {lay:6s} FAILED: {e}", flush=True)
                bad += 1
    print("bad cases:", bad)


if __name__ == "__main__":
    main()
