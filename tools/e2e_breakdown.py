"""Where bench.py's e2e time goes at C2: the device-timed session first (as
bench.py runs it), then public solve() calls from fresh PhiTensor objects,
each followed by the same solve spelled out through the session API with
host timestamps per phase.

    python tools/e2e_breakdown.py [--steps 20] [--c1]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1905_06234_b200 as L  # noqa: E402
from paper_1905_06234_b200 import _native as N, device, sbbnnls  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--c1", action="store_true")
args = ap.parse_args()
dims = L.Dims(1057, 10_000, 20_000, 96, 5_000_000) if args.c1 else \
    L.Dims(1057, 200_000, 500_000, 96, 100_000_000)
p = L.generate(L.GenConfig(dims=dims, mean_run_length=1.04 * dims.n_coeffs / dims.n_voxels,
                           weight_density=0.5, noise_sigma=0.1, seed=0))
t = p.tensor

# the device-timed part of bench.py
op = device.DeviceOperator(t, p.dictionary)
b = torch.from_numpy(p.y).to(device="cuda", dtype=torch.float32)
w = torch.empty(dims.n_fibers, dtype=torch.float32, device="cuda")
sess = sbbnnls.SolverSession(op, b, w, L.SolverConfig(max_iters=30, grad_tol=0.0))
sess.iterate(30)
sess.finish()
sess.close()
del op, sess
torch.cuda.synchronize()


def fresh():
    return L.Problem(tensor=L.PhiTensor(atoms=t.atoms, voxels=t.voxels, fibers=t.fibers,
                                        values=t.values, dims=t.dims),
                     dictionary=p.dictionary, y=p.y)


def spelled_out(prob, steps):
    cfg = L.SolverConfig(max_iters=steps, grad_tol=0.0)
    marks = [("start", time.perf_counter())]

    def mark(what):
        torch.cuda.synchronize()
        marks.append((what, time.perf_counter()))
    sbbnnls.check_restructure_pairs(prob.tensor.ordering, cfg)
    mark("checks")
    o = device.operator_for(prob.tensor, prob.dictionary, exact=False)
    mark("operator")
    bb = device.upload(np.asarray(prob.y, dtype=np.float64), torch.float32)
    ww = torch.empty(dims.n_fibers, dtype=torch.float32, device="cuda")
    mark("b upload")
    s = sbbnnls.SolverSession(o, bb, ww, cfg)
    mark("session create (w0 DSC, graph)")
    s.iterate(steps)
    mark(f"{steps} iterations")
    s.poll()
    mark("poll")
    s.finish()
    mark("finish (final DSC, records)")
    s.close()
    mark("session destroy")
    ww.double().cpu().numpy()
    mark("w D2H")
    o.close()
    mark("operator destroy (not in solve)")
    prev = marks[0][1]
    out = []
    for what, tm in marks[1:]:
        out.append(f"{what} {1e3 * (tm - prev):.1f}")
        prev = tm
    total = 1e3 * (marks[-2][1] - marks[0][1])
    print(f"  spelled out: total {total:.1f} ms | " + " | ".join(out), flush=True)


for rep in range(3):
    prob = fresh()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    w_host, tr = L.solve(prob, config=L.SolverConfig(max_iters=args.steps, grad_tol=0.0))
    dt = time.perf_counter() - t0
    print(f"solve {rep}: {dt * 1e3:.1f} ms = setup {tr.setup_seconds * 1e3:.1f} + loop "
          f"{tr.loop_seconds * 1e3:.1f} + other {1e3 * (dt - tr.setup_seconds - tr.loop_seconds):.1f}"
          f" -> e2e {args.steps / dt:.1f} it/s", flush=True)
    prob.tensor.__dict__.get("_device_cache", {}).get("op", [None])[0].close()
    spelled_out(fresh(), args.steps)
