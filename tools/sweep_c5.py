"""C5 (BASELINE.json configs[4]): isolated DSC and WC bandwidth over nnz
1M..1B with skewed fascicle lengths, on one B200.

The reference generator cannot skew fascicle lengths (datagen.py:97) and is
too slow at 1B, so the problem is drawn on the device (torch, seeded):
Nθ=96, Na=1057, Nv=Nc/500, Nf=Nc/200; fascicle segment lengths lognormal
(sigma 1.0) or Zipf-like, scaled to sum to Nc; voxels and atoms uniform;
values in (0, 1].  Each nnz is built with from_device (no host copies),
timed as the median of --reps CUDA-event-timed calls after warm-up, and
reported as algorithmic GB/s (same formula as bench.py) and
as a fraction of the measured HBM peak.  Up to --parity-max nnz the fp32
products are checked against the device fp64 bit-exact family (relative L2
<= 1e-5, the north_star tolerance).  One JSON line per (nnz, op).

  python tools/sweep_c5.py --nnz 1e6,4e6,16e6,64e6,256e6,1e9 [--skew lognormal|zipf]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402  (spmv_bytes, peaks)
import paper_1905_06234_b200 as L  # noqa: E402
from paper_1905_06234_b200 import _native, datagen, device  # noqa: E402


def draw(nc, skew, seed):
    return datagen.draw_skewed_device(nc, skew, seed)


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--nnz", default="1e6,4e6,16e6,64e6,256e6,1e9")
    ap.add_argument("--skew", choices=["lognormal", "zipf"], default="lognormal")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--parity-max", type=float, default=16e6)
    ap.add_argument("--layout", default="auto")
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    peak, src = bench.peaks()
    device.set_layout(args.layout)
    for nc in [int(float(x)) for x in args.nnz.split(",")]:
        t0 = time.time()
        dims, a, v, f, val, dic, fmax = draw(nc, args.skew, args.seed)
        exact = nc <= args.parity_max
        op = L.DeviceOperator.from_device(dims, a, v, f, val, dic, exact=exact)
        del a, v, f, val
        torch.cuda.synchronize()
        build_s = time.time() - t0
        w = torch.rand(dims.n_fibers, device="cuda")
        w[torch.rand(dims.n_fibers, device="cuda") < 0.5] = 0.0  # half-zero w (zero skip active)
        y = torch.empty(dims.signal_len, device="cuda")
        g = torch.empty(dims.n_fibers, device="cuda")
        ymax = torch.empty(1, device="cuda")
        dsc_ms = timed(lambda: op.dsc_f32(w, y, flags=_native.SKIP_ZERO, absmax=ymax), args.reps)
        wc_ms = timed(lambda: op.wc_f32(y, g, y_absmax=ymax), args.reps)
        # binned layout: 2-byte cell + 2-byte slot + 4-byte value per coefficient
        # for both products (SURVEY 8(d) under compression, as bench.py)
        ib = 2 if op.kind == "bin" else 4
        bd, bw = bench.spmv_bytes((dims.n_atoms, dims.n_voxels, dims.n_fibers, dims.n_dirs, nc), idx_bytes=ib)
        parity = None
        if exact:
            y64 = torch.zeros(dims.signal_len, dtype=torch.float64, device="cuda")
            op.dsc_f64(w.double(), y64)
            g64 = torch.zeros(dims.n_fibers, dtype=torch.float64, device="cuda")
            op.wc_f64(y.double(), g64)
            rel = lambda a_, b_: float((a_.double() - b_).norm() / b_.norm())  # noqa: E731
            parity = {"dsc_rel_l2": rel(y, y64), "wc_rel_l2": rel(g, g64), "tol": 1e-5}
        base = {"config": "C5", "nnz": nc, "n_voxels": dims.n_voxels, "n_fibers": dims.n_fibers,
                "n_atoms": dims.n_atoms, "n_dirs": dims.n_dirs, "skew": args.skew,
                "max_fascicle_len": fmax, "kernels": op.kind, "tensor_cores": list(op.tensor_ops), "build_s": round(build_s, 3),
                "peak_gbs": peak, "peak_source": src}
        for name, ms, b in (("dsc", dsc_ms, bd), ("wc", wc_ms, bw)):
            gbs = b / ms / 1e6
            line = dict(base, op=name, ms=round(ms, 4), bytes=b, gbs=round(gbs, 1),
                        frac=round(gbs / peak, 4))
            if parity:
                line["parity"] = parity
            print(json.dumps(line), flush=True)
        op.close()
        del op, w, y, g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
