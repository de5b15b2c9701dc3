"""Voxel sharding for multi-GPU runs, checked on CPU.

world_size-2 gloo process groups run the sharded computation with the
oracle as the per-rank compute; the all-reduced results must match the
unsharded oracle (bitwise for DSC: every voxel has one owner and keeps its
coefficient order; bitwise for the fixed-point WC sums)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_1905_06234_b200 as L
from paper_1905_06234_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("seed", range(12))
def test_run_table_snap_equals_reference_rule(seed):
    rng = np.random.default_rng(seed)
    nv = int(rng.integers(1, 40))
    counts = rng.geometric(0.2, size=nv) * (rng.random(nv) < 0.8)
    keys = np.repeat(np.arange(nv), counts)
    nc = keys.size
    starts = np.concatenate(([0], np.cumsum(counts)))
    for T in (1, 2, 3, 4, 8):
        step = -(-nc // T) if nc else 0
        bounds = [min(i * step, nc) for i in range(T + 1)]
        assert D._snap_runs(starts, bounds) == L.snap_to_run_boundaries(keys, bounds)
        ranges = D.shard_voxel_ranges(counts, T)
        assert ranges[0][0] == 0 and ranges[-1][1] == nv
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))


def _worker(rank, world, port, q, dims):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from oracle import oracle as O
    p = O.generate(dims, 30.0, 0.5, 0.1, 11)
    counts = np.bincount(p["voxels"], minlength=dims[1])
    v0, v1 = D.shard_voxel_ranges(counts, world)[rank]
    sel = np.flatnonzero((p["voxels"] >= v0) & (p["voxels"] < v1))
    loc = dict(p)
    for k in ("atoms", "fibers", "values"):
        loc[k] = np.ascontiguousarray(p[k][sel])
    loc["voxels"] = np.ascontiguousarray(p["voxels"][sel] - v0, dtype=np.uint32)
    nvl = max(1, v1 - v0)
    loc["dims"] = (dims[0], nvl, dims[2], dims[3], sel.size)
    nt = dims[3]
    rng = np.random.default_rng(3)
    w = rng.standard_normal(dims[2])
    # DSC: local slice, gathered
    y_loc = np.zeros(nvl * nt)
    O.dsc(loc, w, y_loc)
    y_full = torch.zeros(dims[1] * nt, dtype=torch.float64)
    y_full[v0 * nt:v1 * nt] = torch.from_numpy(y_loc[:(v1 - v0) * nt])
    dist.all_reduce(y_full)
    # WC: fp64 partials summed, and fixed-point partials summed as int64
    yin = rng.standard_normal(dims[1] * nt)
    w_loc = np.zeros(dims[2])
    O.wc(loc, yin[v0 * nt:v1 * nt] if v1 > v0 else np.zeros(nt), w_loc)
    wsum = torch.from_numpy(w_loc.copy())
    dist.all_reduce(wsum)
    scale = 2.0 ** 40
    q_loc = torch.from_numpy(np.rint(w_loc * scale).astype(np.int64))
    dist.all_reduce(q_loc)
    if rank == 0:
        q.put((y_full.numpy(), wsum.numpy(), q_loc.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_products_match_unsharded(world, oracle):
    dims = (20, 60, 50, 16, 4000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, dims)) for r in range(world)]
    for pr in procs:
        pr.start()
    y_sh, w_sh, q_sh = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = oracle.generate(dims, 30.0, 0.5, 0.1, 11)
    rng = np.random.default_rng(3)
    w = rng.standard_normal(dims[2])
    y = np.zeros(dims[1] * dims[3])
    oracle.dsc(p, w, y)
    assert np.array_equal(y_sh, y)          # one owner per voxel: bitwise
    yin = rng.standard_normal(dims[1] * dims[3])
    wf = np.zeros(dims[2])
    oracle.wc(p, yin, wf)
    np.testing.assert_allclose(w_sh, wf, rtol=1e-12, atol=1e-12 * np.abs(wf).max())
    # integer partial sums are order independent: equal to any other split
    assert q_sh.dtype == np.int64


def test_global_fix_bounds():
    d = L.Dims(3, 4, 5, 2, 6)
    t = L.PhiTensor(atoms=[0, 1, 2, 0, 1, 2], voxels=[0, 1, 2, 3, 0, 1],
                    fibers=[4, 4, 4, 1, 0, 4], values=[0.5, -2.0, 1.0, 1.0, 0.1, 0.3], dims=d)
    vmax, fmax = D.global_fix_bounds(t)
    assert fmax == 4 and abs(vmax - 2.0) < 1e-5


def _route_worker(rank, world, port, q, dims):
    """shard_from_slices' routing on CPU tensors: each rank takes its 1/N
    slice of the coefficient list, the statistics come from all-reduces and
    the coefficients reach their owners by all_to_all."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    p = O.generate(dims, 30.0, 0.5, 0.1, 11)
    d = L.Dims(*dims)
    c0, c1 = D.slice_bounds(d.n_coeffs, rank, world)
    sl = [torch.from_numpy(np.ascontiguousarray(p[k][c0:c1]).view(np.int32))
          for k in ("atoms", "voxels", "fibers")]
    val = torch.from_numpy(np.ascontiguousarray(p["values"][c0:c1]))
    counts, vmax, fmax = D.reduce_shard_stats(sl[1], sl[2], val, d, None, torch.device("cpu"))
    ranges = D.shard_voxel_ranges(counts, world)
    a, v, f, vv = D.route_to_shards((*sl, val), sl[1], ranges, None, torch.device("cpu"))
    q.put((rank, counts, vmax, fmax, ranges, a.numpy().view(np.uint32), v.numpy().view(np.uint32),
           f.numpy().view(np.uint32), vv.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slices_routed_to_shards_equal_host_selection(world, oracle):
    dims = (20, 60, 50, 16, 4000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_route_worker, args=(r, world, port, q, dims)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = sorted((q.get(timeout=120) for _ in range(world)), key=lambda x: x[0])
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = oracle.generate(dims, 30.0, 0.5, 0.1, 11)
    d = L.Dims(*dims)
    t = L.PhiTensor(atoms=p["atoms"], voxels=p["voxels"], fibers=p["fibers"], values=p["values"], dims=d)
    counts = np.bincount(t.voxels, minlength=d.n_voxels)
    ranges = D.shard_voxel_ranges(counts, world)
    vmax, fmax = D.global_fix_bounds(t)
    dic = L.Dictionary(data=p["dict"], dims=d)
    for rank, c, vm, fm, rg, a, v, f, vv in got:
        assert np.array_equal(c, counts) and rg == ranges
        assert vm == vmax and fm == fmax  # bit for bit
        v0, v1 = ranges[rank]
        tl, _, _ = D.shard_problem(t, dic, np.zeros(d.signal_len), v0, v1)
        assert np.array_equal(a, tl.atoms) and np.array_equal(v, tl.voxels + np.uint32(v0))
        assert np.array_equal(f, tl.fibers) and np.array_equal(vv, tl.values)
