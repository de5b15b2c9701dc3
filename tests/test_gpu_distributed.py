"""Voxel-sharded SBBNNLS through the C-ABI comm hook: two ranks on one GPU
(gloo process group, host-staged all-reduce) against the single-GPU solve.
The NCCL path differs only in the transport of the same all-reduce calls."""

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
