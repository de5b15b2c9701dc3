"""Benchmark: SBBNNLS iterations/sec on the STN96-shaped problem (C2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one SBBNNLS iteration (2 DSC + 1.5 WC on average, Alg. 1) over
the whole synthetic problem of BASELINE.json configs[1]: N_theta=96,
Na=1057, Nv=200k, Nf=500k, Nc=100M (data: the reference generator's
algorithm, seed 0, noise 0.1).  ``value`` times exactly K iterations with
the problem resident in HBM (CUDA events, max over ranks); ``e2e`` times a
public ``solve()`` of K iterations from host numpy arrays (H2D of Phi/D/b,
device restructuring, the iterations, D2H of w).  The reference arm
(``--impl reference``) times the CPU oracle port of the reference's
sbbnnls.solve on the full C2 workload on this host's cores: W untimed
iterations, then exactly K timed ones of the same solve.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (Na, Nv, Nf, Ntheta, Nc)
    "c2": (1057, 200_000, 500_000, 96, 100_000_000),
    "c1": (1057, 10_000, 20_000, 96, 5_000_000),
    "c2s": (1057, 50_000, 125_000, 96, 25_000_000),
    # one rank's share of C3 at 8 GPUs (an eighth of C2's voxels, all fascicles)
    "c2x8": (1057, 25_000, 500_000, 96, 12_500_000),
    # BASELINE.json configs[3] (quoted on 8 GPUs; Nv assumed):
    # N_theta = 150 takes the 160-wide register-tiled kernels
    "c4": (1057, 250_000, 1_000_000, 150, 400_000_000),
}
WORKLOADS = {
    "c2": "C2 STN96-shaped synthetic LiFE problem (BASELINE.json configs[1])",
    "c1": "C1 synthetic STD LiFE problem (BASELINE.json configs[0])",
    "c2s": "C2 at quarter scale",
    "c2x8": "one rank's share of C3 at 8 GPUs (C2 voxels / 8, all fascicles) on 1 GPU",
    "c4": "C4 probabilistic-tractography scale, N_theta=150 (BASELINE.json configs[3])",
}
METRIC = "SBBNNLS iters/sec"
UNIT = "it/s"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        return float(m["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def spmv_bytes(dims, val_bytes=4, idx_bytes=4, vec_bytes=4):
    """Algorithmic (compulsory) bytes per call, SURVEY.md 8(d)."""
    na, nv, nf, nt, nc = dims
    dsc = nc * (2 * idx_bytes + val_bytes) + (nv + 1) * 4 + nf * vec_bytes \
        + nv * nt * vec_bytes + na * nt * vec_bytes
    wc = nc * (2 * idx_bytes + val_bytes) + (nv + 1) * 4 + nv * nt * vec_bytes \
        + nf * vec_bytes + na * nt * vec_bytes
    return dsc, wc


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML
    polled every 2 ms from a thread (the timed region of K=20 iterations is
    ~35 ms, shorter than nvidia-smi's 100 ms period); nvidia-smi when NVML
    is unavailable."""

    REASONS = (("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20),
               ("hw_thermal_slowdown", 0x40), ("sw_power_cap", 0x4))

    def __init__(self, device_index):
        self.dev = device_index
        self.samples = []   # (sm_mhz, reasons bitmask)
        self.max_mhz = None
        self.proc = None
        self._stop = threading.Event()
        self._nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = int(vis.split(",")[self.dev]) if vis and vis.split(",")[0].isdigit() else self.dev
            h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self._nvml = (pynvml, h)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:
            self._nvml = None
            self._start_smi()
        time.sleep(0.01)  # the first samples precede the timed region's start
        return self

    def _poll(self):
        pynvml, h = self._nvml
        reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            pynvml.nvmlDeviceGetCurrentClocksThrottleReasons
        while True:
            try:
                self.samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                     reasons(h)))
            except Exception:
                pass
            if self._stop.wait(0.002):
                break

    def _start_smi(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read_smi, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read_smi(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            try:
                self.max_mhz = float(parts[1])
                self.samples.append((float(parts[0]), int(parts[2], 16)))
            except (ValueError, IndexError):
                continue

    def __exit__(self, *exc):
        self._stop.set()
        if self._nvml is not None:
            self.t.join(timeout=1)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        mask = 0
        for _, r in self.samples:
            mask |= int(r)
        return {"sm_mhz": statistics.median(m for m, _ in self.samples),
                "sm_max_mhz": self.max_mhz,
                "reasons": sorted(n for n, bit in self.REASONS if mask & bit),
                "samples": len(self.samples),
                "source": "nvml 2 ms" if self._nvml is not None else "nvidia-smi 100 ms"}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------
# reference arm: CPU oracle port on the full workload
# ---------------------------------------------------------------------------


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_problem(problem):
    """The oracle's dict view of a generated Problem (same arrays, no copy)."""
    t = problem.tensor
    d = t.dims
    return dict(atoms=t.atoms, voxels=t.voxels, fibers=t.fibers, values=t.values,
                dict=problem.dictionary.data, y=problem.y, ordering="unsorted",
                dims=(d.n_atoms, d.n_voxels, d.n_fibers, d.n_dirs, d.n_coeffs))


def time_oracle_iterations(p, warm, steps, threads):
    """Seconds for exactly `steps` SBBNNLS iterations of the oracle port of
    sbbnnls.solve at full size, after `warm` untimed iterations, read from
    the per-iteration timestamps of ONE solve (its sorting setup and the w0
    DSC fall before iteration 1 ends and are excluded)."""
    from oracle import oracle as O
    O.set_threads(threads)
    _, tr = O.solve(p, max_iters=warm + steps, grad_tol=0.0, threads=threads)
    recs = tr["records"]
    if len(recs) < warm + steps:
        raise RuntimeError(f"oracle solve stopped after {len(recs)} iterations ({tr['termination']})")
    return recs[warm + steps - 1]["t"] - recs[warm - 1]["t"]


def cpu_reference(problem, dims, warm=1, steps=2, threads=None):
    """Per-iteration rate of the oracle port of sbbnnls.solve on the FULL
    workload (iterations warm+1 .. warm+steps of one solve)."""
    threads = threads or os.cpu_count()
    sec = time_oracle_iterations(oracle_problem(problem), warm, steps, threads)
    return {"value": steps / sec, "unit": UNIT, "cores": threads, "kind": "port",
            "cpu_model": cpu_model(),
            "sample": (f"oracle port (C + numpy, OpenMP) of sbbnnls.solve on the full workload "
                       f"Nc={dims[4]}: iterations {warm + 1}..{warm + steps} of one solve "
                       f"({steps} iterations, {sec:.1f} s), sorting setup excluded")}


def run_reference(args, dims):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    from oracle import oracle as O
    threads = os.cpu_count()
    O.set_threads(threads)
    na, nv, nf, nt, nc = dims
    t0 = time.perf_counter()
    p = O.generate(dims, 1.04 * nc / nv, 0.5, 0.1, 0)
    t_gen = time.perf_counter() - t0
    # a step is one SBBNNLS iteration of the reference algorithm on the full
    # workload: W untimed iterations, then exactly K timed ones
    sec = time_oracle_iterations(p, args.warmup, args.steps, threads)
    value = args.steps / sec
    line = {"metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * sec / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(dims, args, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "cpu_model": cpu_model(),
                             "sample": f"oracle port (C + numpy, OpenMP) of sbbnnls.solve on "
                                       f"the full workload Nc={nc}: iterations "
                                       f"{args.warmup + 1}..{args.warmup + args.steps} of one "
                                       f"solve timed from its per-iteration timestamps "
                                       f"(generation {t_gen:.0f} s and sorting setup excluded)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def workload_config(dims, args, world):
    na, nv, nf, nt, nc = dims
    return {"workload": WORKLOADS.get(args.config, args.config),
            "n_atoms": na, "n_voxels": nv, "n_fibers": nf, "n_dirs": nt, "n_coeffs": nc,
            "mean_run_length": round(1.04 * nc / nv, 3), "noise_sigma": 0.1, "seed": 0,
            "parallelism": f"voxel-shard x{world}" if world > 1 else "1 GPU",
            "l2": f"inputs larger than L2 (Phi alone {nc * 12 / 1e9:.1f} GB vs 126 MB L2)"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------


def run_ours(args, dims):
    import torch

    import paper_1905_06234_b200 as L
    from paper_1905_06234_b200 import _native, datagen

    world, rank, local = dist_env()
    # the sharded code path also at world 1 (a one-GPU check of the N > 1 path)
    sharded = world > 1 or os.environ.get("LIFE_BENCH_SHARDED") == "1"
    torch.cuda.set_device(local)
    from paper_1905_06234_b200 import device as _dev
    _dev.set_layout(args.layout)
    if sharded:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    na, nv, nf, nt, nc = dims
    cfg = L.GenConfig(dims=L.Dims(*dims), mean_run_length=1.04 * nc / nv,
                      weight_density=0.5, noise_sigma=0.1, seed=0)
    t_gen = time.perf_counter()
    problem = L.generate(cfg)
    t_gen = time.perf_counter() - t_gen
    info = {"generate_s": round(t_gen, 2)}

    # ---- device-resident timing of exactly K iterations ---------------------
    total_iters = args.warmup + args.steps
    comm = None
    if sharded:
        from paper_1905_06234_b200 import distributed as D
        comm = D.NcclComm()  # the library's own NCCL communicator (graphs on)
        # each rank uploads 1/N of the coefficient list; shards are routed
        # to their owners over NVLink (all_to_all), see shard_from_slices
        op, b, (v0, v1), _ = D.shard_from_slices(problem)
        local_dims = (na, op.dims.n_voxels, nf, nt, op.dims.n_coeffs)
        info["shard"] = {"voxels": [int(v0), int(v1)], "n_coeffs": int(op.dims.n_coeffs)}
    else:
        op = L.DeviceOperator(problem.tensor, problem.dictionary)
        b = torch.from_numpy(problem.y).to(device="cuda", dtype=torch.float32)
        local_dims = dims
    info["restructure_ms"] = round(op.info.sort_ms, 1)
    info["atom_groups"] = op.info.atom_groups
    info["kernels"] = op.kind
    info["tensor_cores"] = list(op.tensor_ops)
    w = torch.empty(nf, dtype=torch.float32, device="cuda")
    scfg = L.SolverConfig(max_iters=total_iters, grad_tol=0.0)
    sess = L.sbbnnls.SolverSession(op, b, w, scfg, comm=comm)
    sess.iterate(args.warmup)
    torch.cuda.synchronize()
    if sharded:
        torch.distributed.barrier()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = _native.launch_count()
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize()
        start.record()
        sess.iterate(args.steps)
        stop.record()
        torch.cuda.synchronize()
    launches = _native.launch_count() - launches0
    ms = start.elapsed_time(stop)
    if sharded:
        t = torch.tensor([ms], device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    res, recs = sess.finish()
    if res.iterations < total_iters:
        raise RuntimeError(f"solver stopped after {res.iterations} < {total_iters} iterations "
                           f"({res.termination}); timed region would contain no-op steps")
    value = args.steps / (ms * 1e-3)

    # ---- kernel-level timing (DSC / WC) for the roofline -------------------
    # (this rank's shard when N > 1: local bytes over local kernel time)
    dsc_b, wc_b = spmv_bytes(local_dims)
    if op.kind == "bin":
        # binned layout: per coefficient a 2-byte tile cell, a 2-byte bin slot
        # and a 4-byte value, for both products (SURVEY 8(d) counts the
        # actual sizes under compression); the tile<->bin exchange through
        # the scratch is design overhead and shows up in `traffic`
        dsc_b, wc_b = spmv_bytes(local_dims, idx_bytes=2)

    y = torch.empty(local_dims[1] * nt, dtype=torch.float32, device="cuda")
    g = torch.empty(nf, dtype=torch.float32, device="cuda")
    ymax = torch.zeros(1, dtype=torch.float32, device="cuda")
    iso = max(5, min(20, args.steps))
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(iso)]
    for _ in range(2):
        op.dsc_f32(w, y, flags=_native.SKIP_ZERO, absmax=ymax)
    for e0, e1 in ev:
        e0.record()
        op.dsc_f32(w, y, flags=_native.SKIP_ZERO, absmax=ymax)
        e1.record()
    torch.cuda.synchronize()
    t_dsc = statistics.mean(e0.elapsed_time(e1) for e0, e1 in ev) * 1e-3
    for _ in range(2):
        op.wc_f32(y, g, y_absmax=ymax)
    for e0, e1 in ev:
        e0.record()
        op.wc_f32(y, g, y_absmax=ymax)
        e1.record()
    torch.cuda.synchronize()
    t_wc = statistics.mean(e0.elapsed_time(e1) for e0, e1 in ev) * 1e-3
    peak, peak_kind = peaks()
    dsc_gbs, wc_gbs = dsc_b / t_dsc / 1e9, wc_b / t_wc / 1e9
    if 2 * t_dsc >= 1.5 * t_wc:
        dom, ach, traffic_key = "dsc", dsc_gbs, "dsc"
    else:
        dom, ach, traffic_key = "wc", wc_gbs, "wc"
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof) and args.config == "c2" and world == 1:  # captured on C2, 1 GPU
        try:
            with open(prof) as f:
                traffic = json.load(f).get(traffic_key)
        except Exception:
            traffic = None

    # ---- end to end through the public API from host buffers ---------------
    e2e = None
    if not args.no_e2e:
        t = problem.tensor
        fresh = L.PhiTensor(atoms=t.atoms, voxels=t.voxels, fibers=t.fibers, values=t.values,
                            dims=t.dims)
        p2 = L.Problem(tensor=fresh, dictionary=problem.dictionary, y=problem.y)
        sess.close()
        del op, sess
        torch.cuda.synchronize()
        if sharded:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        if sharded:
            # the communicator of the device-timed run is reused (NCCL init is
            # a one-time job cost, not a per-solve one)
            w_host, tr = D.solve_sharded(p2, L.SolverConfig(max_iters=args.steps, grad_tol=0.0),
                                         comm=comm)
        else:
            w_host, tr = L.solve(p2, config=L.SolverConfig(max_iters=args.steps, grad_tol=0.0))
        e2e_s = time.perf_counter() - t0
        if sharded:
            tt = torch.tensor([e2e_s], device="cuda")
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            e2e_s = float(tt.item())
        # bytes crossing PCIe (life_phi_create with LIFE_PHI_HOST_INPUT): atom and
        # voxel packed into one u32 when both fields fit (else atoms u16 / u32 +
        # voxels u32), fibers u32, values f32 (fp32-only operator); the
        # dictionary as f64, b as f32 (rounded while staging)
        bits = lambda x: max(1, int(x).bit_length())  # field width with an all-ones spare
        av = 4 if bits(na) + bits(nv) <= 32 else (2 if na < 65535 else 4) + 4
        h2d = nc * (av + 4 + 4) + na * nt * 8 + nv * nt * 4
        if sharded:  # whole job: each rank's 1/N slice (u32 indices, f64 values), D per rank
            h2d = nc * (4 + 4 + 4 + 8) + world * na * nt * 8 + nv * nt * 4
        cached = fresh.__dict__.get("_device_cache", {}).get("op")
        e2e = {"value": args.steps / e2e_s, "unit": UNIT,
               "setup_s": round(tr.setup_seconds, 3), "loop_s": round(tr.loop_seconds, 4),
               "create_ms": round(cached[0].info.sort_ms, 1) if cached else None,
               "other_s": round(e2e_s - tr.setup_seconds - tr.loop_seconds, 3),
               "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": nf * 8 // args.steps,
               "seconds": round(e2e_s, 3),
               "what": f"one solve() of {args.steps} iterations from host numpy arrays: "
                       "H2D of Phi/D/b + device restructuring + iterations + D2H of w "
                       "(bytes spread over the steps)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:  # the CPU baseline is a 1-GPU figure
        cpu = cpu_reference(problem, dims)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f32", "data": "synthetic",
                "config": workload_config(dims, args, world),
                "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                             "frac": ach / peak, "traffic": traffic, "kernel": dom,
                             "peak_source": peak_kind},
                "spmv": {"dsc_ms": t_dsc * 1e3, "wc_ms": t_wc * 1e3,
                         "dsc_gbs": dsc_gbs, "wc_gbs": wc_gbs,
                         "dsc_bytes": dsc_b, "wc_bytes": wc_b,
                         "dsc_frac": dsc_gbs / peak, "wc_frac": wc_gbs / peak},
                "e2e": e2e, "cpu_baseline": cpu, "clocks": clocks.summary(),
                "gpu_launches": int(launches), "info": info}
        print(json.dumps(line), flush=True)
    if sharded:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--layout", default="auto", choices=["auto", "sparse", "bin"])
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    dims = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, dims)
    else:
        run_ours(args, dims)


if __name__ == "__main__":
    main()
