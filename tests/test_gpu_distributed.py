"""Voxel-sharded SBBNNLS: two and three ranks on one GPU through the C-ABI
comm hook (gloo process group, host-staged all-reduce), and the library's
own NCCL communicator at world 1 through the graph path, against the
single-GPU solve."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem():
    import paper_1905_06234_b200 as L
    dims = L.Dims(n_atoms=300, n_voxels=2000, n_fibers=3000, n_dirs=96, n_coeffs=400_000)
    return L.generate(L.GenConfig(dims=dims, mean_run_length=208.0, weight_density=0.5,
                                  noise_sigma=0.1, seed=5))


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_1905_06234_b200 as L
    from paper_1905_06234_b200 import distributed as D
    p = _problem()
    w, tr = D.solve_sharded(p, L.SolverConfig(max_iters=12, grad_tol=0.0))
    q.put((rank, w, tr.final_objective, [r.objective for r in tr.records],
           [r.dsc_skipped for r in tr.records], tr.termination))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_solve_matches_single_gpu(world):
    import paper_1905_06234_b200 as L
    p = _problem()
    w1, tr1 = L.solve(p, config=L.SolverConfig(max_iters=12, grad_tol=0.0))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    outs = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    ws = [o[1] for o in outs]
    for other in ws[1:]:
        assert np.array_equal(other, ws[0])       # replicated state: identical on all ranks
    rel = np.linalg.norm(ws[0] - w1) / np.linalg.norm(w1)
    assert rel <= 1e-5, rel
    fo = outs[0][2]
    assert abs(fo - tr1.final_objective) <= 1e-5 * tr1.final_objective
    assert outs[0][4] == [r.dsc_skipped for r in tr1.records]  # global skip counts
    assert outs[0][5] == tr1.termination


def test_nccl_comm_world1_through_graphs():
    """The library's own NCCL communicator (life_comm_init_nccl) at world 1,
    the only shape one GPU allows: the sharded iteration (bound-scaled WC,
    DSC scalars in the tail of the WC all-reduce, odd-iteration scalar
    all-reduce) runs as CUDA graphs and matches the single-GPU solve."""
    import torch

    import paper_1905_06234_b200 as L
    from paper_1905_06234_b200 import _native as N
    from paper_1905_06234_b200 import device
    from paper_1905_06234_b200 import distributed as D
    from paper_1905_06234_b200.sbbnnls import SolverSession, trace_from

    p = _problem()
    cfg = L.SolverConfig(max_iters=12, grad_tol=0.0)
    w1, tr1 = L.solve(p, config=cfg)
    comm = D.NcclComm(rank=0, nranks=1)
    assert comm.c.capturable == 1 and comm.c.nranks == 1
    op = device.DeviceOperator(p.tensor, p.dictionary)
    b = device.upload(np.asarray(p.y, dtype=np.float64), torch.float32)
    w = torch.empty(p.dims.n_fibers, dtype=torch.float32, device="cuda")
    launches0 = N.launch_count()
    sess = SolverSession(op, b, w, cfg, comm=comm)
    sess.iterate(cfg.max_iters)
    res, recs = sess.finish()
    sess.close()
    assert N.launch_count() > launches0
    tr = trace_from(res, recs)
    wn = w.double().cpu().numpy()
    rel = np.linalg.norm(wn - w1) / np.linalg.norm(w1)
    assert rel <= 1e-5, rel
    assert abs(tr.final_objective - tr1.final_objective) <= 1e-5 * tr1.final_objective
    assert [r.dsc_skipped for r in tr.records] == [r.dsc_skipped for r in tr1.records]
    # bitwise repeatable through the communicator
    w2 = torch.empty_like(w)
    sess = SolverSession(op, b, w2, cfg, comm=comm)
    sess.iterate(cfg.max_iters)
    sess.finish()
    sess.close()
    assert torch.equal(w, w2)
    comm.close()


def _nccl_world1_worker(port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    import paper_1905_06234_b200 as L
    from paper_1905_06234_b200 import _native as N
    from paper_1905_06234_b200 import distributed as D
    p = _problem()
    cfg = L.SolverConfig(max_iters=12, grad_tol=0.0)
    # shards from 1/N host slices, routed with NCCL all_to_all on the device
    op, b, rng, bounds = D.shard_from_slices(p)
    # against the host selection of the same voxel range
    t, dic, b_host = D.shard_problem(p.tensor, p.dictionary, p.y, *rng)
    ref = L.DeviceOperator(t, dic)
    vmax, fmax = D.global_fix_bounds(p.tensor)
    N.check(N.lib().life_phi_set_fix_bounds(ref.handle, vmax, 0.0, fmax))
    w = torch.from_numpy(p.w_true).to("cuda", torch.float32)
    ys = []
    gs = []
    for o in (op, ref):
        y = torch.zeros(o.dims.signal_len, dtype=torch.float32, device="cuda")
        g = torch.zeros(p.dims.n_fibers, dtype=torch.float32, device="cuda")
        o.dsc_f32(w, y, flags=N.SKIP_ZERO)
        o.wc_f32(y, g)
        ys.append(y.cpu().numpy())
        gs.append(g.cpu().numpy())
    same_ops = bool(np.array_equal(ys[0], ys[1]) and np.array_equal(gs[0], gs[1]))
    same_b = bool(np.array_equal(b.cpu().numpy(), b_host.astype(np.float32)))
    w_dev, tr_dev = D.solve_sharded(p, cfg)                         # device routing
    w_host, tr_host = D.solve_sharded(p, cfg, ranges=[(0, p.dims.n_voxels)])  # host selection
    q.put((rng, bounds, D.global_fix_bounds(p.tensor), same_ops, same_b,
           bool(np.array_equal(w_dev, w_host)), tr_dev.final_objective, tr_host.final_objective))
    dist.destroy_process_group()


def test_shards_from_slices_over_nccl_world1():
    """shard_from_slices through an NCCL process group (world 1: the
    statistics all-reduces and the all_to_all run on the device): the
    operator, b and the sharded solve equal the host-selected shard's."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_nccl_world1_worker, args=(_free_port(), q))
    pr.start()
    rng, bounds, host_bounds, same_ops, same_b, same_w, fo_dev, fo_host = q.get(timeout=300)
    pr.join(timeout=60)
    assert pr.exitcode == 0
    assert rng == (0, 2000) and bounds == host_bounds
    assert same_ops and same_b and same_w and fo_dev == fo_host
