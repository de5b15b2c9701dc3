"""Voxel-sharded SBBNNLS over several GPUs.

One process per GPU.  Phi is cut into contiguous voxel ranges balanced by
coefficient count; a boundary never splits a voxel's coefficients -- exactly
the reference's synchronization-free rule (engine.build_plan with
PartitionStrategy("coefficient", sync_free=True), engine.py:113-184) with
one "thread" per GPU.  Each rank holds its Phi slice (voxels renumbered
from 0), the full dictionary, its slice of the signal and the replicated
weights.

Per iteration the exchange is: DSC local (one all-reduce of two doubles:
sum of squares and skip count), WC local partial sums of the Nf fascicle
weights in 64-bit fixed point followed by one all-reduce (int64 sum, so the
result is bit-identical on all ranks and independent of the reduction
order).  All Nf-space solver work (projection, step size, update) then runs
redundantly and identically on every rank: there is no broadcast.

The collectives are torch.distributed calls (NCCL over NVLink/NVSwitch for
the CUDA backend; gloo works too, for tests) enqueued on the solver's stream
from a ctypes callback that liblife_b200 invokes between its kernels.
"""

import ctypes
import math

import numpy as np

from . import _native as N
from .errors import ConfigInvalid
from .tensor import Dictionary, Dims, PhiTensor


def shard_voxel_ranges(voxel_counts, nranks):
    """Contiguous voxel ranges [v0, v1) per rank.

    The coefficient range of the voxel-sorted tensor is split into
    ceil(Nc/nranks) chunks whose interior boundaries are snapped to voxel-run
    boundaries (engine.snap_to_run_boundaries), then mapped back to voxels.
    ``voxel_counts[v]`` is the number of coefficients of voxel v."""
    counts = np.asarray(voxel_counts, dtype=np.int64)
    nv = counts.size
    nc = int(counts.sum())
    if nranks < 1:
        raise ConfigInvalid("nranks must be >= 1")
    starts = np.concatenate(([0], np.cumsum(counts)))
    step = math.ceil(nc / nranks) if nc else 0
    bounds = [min(i * step, nc) for i in range(nranks + 1)]
    # the voxel key array of the sorted tensor, implicitly: run v covers
    # [starts[v], starts[v+1]); snap on that run table (same result as
    # snap_to_run_boundaries on the expanded key array, tested)
    bounds = _snap_runs(starts, bounds)
    # coefficient boundary -> voxel boundary (first voxel starting at it)
    vb = [0]
    for b in bounds[1:-1]:
        vb.append(int(np.searchsorted(starts, b, side="left")))
    vb.append(nv)
    for i in range(1, len(vb)):
        vb[i] = max(vb[i], vb[i - 1])
    return [(vb[i], vb[i + 1]) for i in range(nranks)]


def _snap_runs(starts, bounds):
    """snap_to_run_boundaries on the run table (no per-coefficient keys)."""
    nc = int(starts[-1])
    out = list(bounds)
    for i in range(1, len(out) - 1):
        b = out[i]
        if 0 < b < nc:
            v = int(np.searchsorted(starts, b, side="right")) - 1  # run containing b
            lo, hi = int(starts[v]), int(starts[v + 1])
            if lo < b < hi:
                out[i] = lo if (b - lo) <= (hi - b) else hi
    for i in range(1, len(out)):
        out[i] = max(out[i], out[i - 1])
    return out


def shard_problem(tensor, dictionary, y, v0, v1):
    """The local problem of voxel range [v0, v1): (PhiTensor, Dictionary, b)."""
    d = tensor.dims
    sel = (tensor.voxels >= v0) & (tensor.voxels < v1)
    idx = np.flatnonzero(sel)
    local = Dims(n_atoms=d.n_atoms, n_voxels=max(1, v1 - v0), n_fibers=d.n_fibers,
                 n_dirs=d.n_dirs, n_coeffs=int(idx.size))
    t = PhiTensor(atoms=tensor.atoms[idx], voxels=tensor.voxels[idx] - np.uint32(v0),
                  fibers=tensor.fibers[idx], values=tensor.values[idx], dims=local)
    dic = Dictionary(data=dictionary.data, dims=local)
    b = np.zeros(local.signal_len)
    if v1 > v0:
        b[:] = np.asarray(y)[v0 * d.n_dirs:v1 * d.n_dirs]
    return t, dic, b


def global_fix_bounds(tensor):
    """(max |value|, longest fascicle) over the whole problem: every rank must
    derive the same fixed-point exponent for the WC all-reduce."""
    vmax = float(np.max(np.abs(tensor.values))) if tensor.dims.n_coeffs else 0.0
    fmax = int(np.bincount(tensor.fibers, minlength=1).max()) if tensor.dims.n_coeffs else 1
    return vmax * (1.0 + 1e-6), max(fmax, 1)


def slice_bounds(n, rank, nranks):
    """The contiguous 1/nranks slice of the coefficient list a rank uploads."""
    return rank * n // nranks, (rank + 1) * n // nranks


def reduce_shard_stats(voxels, fibers, values, dims, group, xdev):
    """Whole-problem statistics from every rank's coefficient slice (torch
    tensors): per-voxel coefficient counts (the shard rule's input), and the
    fixed-point bounds of ``global_fix_bounds`` -- computed as slice-local
    bincounts / max|value| followed by one SUM and one MAX all-reduce, equal
    to the host computation bit for bit."""
    import torch
    import torch.distributed as dist
    cnt = torch.bincount(voxels.long(), minlength=dims.n_voxels)
    fcnt = torch.bincount(fibers.long(), minlength=dims.n_fibers)
    vm = values.abs().max().reshape(1) if values.numel() else \
        torch.zeros(1, dtype=torch.float64, device=values.device)
    both = torch.cat((cnt, fcnt)).to(xdev)
    vm = vm.to(xdev)
    dist.all_reduce(both, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(vm, op=dist.ReduceOp.MAX, group=group)
    counts = both[:dims.n_voxels].cpu().numpy()
    nc = int(counts.sum())
    vmax = float(vm.item()) if nc else 0.0
    fmax = int(both[dims.n_voxels:].max().item()) if nc else 1
    return counts, vmax * (1.0 + 1e-6), max(fmax, 1)


def route_to_shards(arrays, voxels, ranges, group, xdev):
    """Send every coefficient of this rank's slice to the rank owning its
    voxel (one all_to_all per array over the group: NVLink with NCCL).  A
    rank receives its voxel range's coefficients in their original relative
    order (senders' slices are in rank order and each sender's partition is
    stable), i.e. exactly what ``shard_problem`` selects on the host."""
    import torch
    import torch.distributed as dist
    world = len(ranges)
    dev = voxels.device
    ends = torch.tensor([r[1] for r in ranges], dtype=torch.int64, device=dev)
    dest = torch.searchsorted(ends, voxels.long(), right=True)
    order = torch.argsort(dest, stable=True)
    send = torch.bincount(dest, minlength=world).to(xdev)
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    sl, rl = send.cpu().tolist(), recv.cpu().tolist()
    out = []
    for a in arrays:
        src = a[order].to(xdev)
        dst = torch.empty(int(sum(rl)), dtype=a.dtype, device=xdev)
        dist.all_to_all_single(dst, src, output_split_sizes=rl, input_split_sizes=sl, group=group)
        out.append(dst)
    return out


def shard_from_slices(problem, group=None):
    """Each rank's voxel shard built on the GPUs: the rank uploads only its
    1/N slice of the coefficient list (staged H2D), the statistics and the
    shard ranges come from two all-reduces, and the coefficients are routed
    to their owners by all_to_all.  Host work per rank is O(Nc/N), against
    three full passes over the host arrays for ``shard_problem`` +
    ``global_fix_bounds`` (2.5 s at C2).  Returns (DeviceOperator, b as a
    CUDA f32 tensor, (v0, v1), (vmax, fmax)); the operator equals the one
    built from ``shard_problem`` (same coefficients in the same order)."""
    import torch
    import torch.distributed as dist

    from . import device
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    xdev = torch.device("cuda") if dist.get_backend(group) == "nccl" else torch.device("cpu")
    t = problem.tensor
    d = t.dims
    c0, c1 = slice_bounds(d.n_coeffs, rank, world)
    a, v, f = (device.upload(x[c0:c1]) for x in (t.atoms, t.voxels, t.fibers))
    val = device.upload(np.asarray(t.values[c0:c1], dtype=np.float64))
    counts, vmax, fmax = reduce_shard_stats(v, f, val, d, group, xdev)
    ranges = shard_voxel_ranges(counts, world)
    v0, v1 = ranges[rank]
    a, v, f, val = (x.to("cuda") for x in route_to_shards((a, v, f, val), v, ranges, group, xdev))
    v -= v0
    local = Dims(n_atoms=d.n_atoms, n_voxels=max(1, v1 - v0), n_fibers=d.n_fibers,
                 n_dirs=d.n_dirs, n_coeffs=int(v.numel()))
    dic = device.upload(np.asarray(problem.dictionary.data, dtype=np.float64))
    op = device.DeviceOperator.from_device(local, a, v, f, val, dic)
    N.check(N.lib().life_phi_set_fix_bounds(op.handle, vmax, 0.0, fmax))
    y = np.asarray(problem.y, dtype=np.float64)
    b = device.upload(y[v0 * d.n_dirs:v1 * d.n_dirs], torch.float32) if v1 > v0 else \
        torch.zeros(local.signal_len, dtype=torch.float32, device="cuda")
    return op, b, (v0, v1), (vmax, fmax)


class _CudaArray:
    """Zero-copy torch view of a raw device pointer (__cuda_array_interface__)."""

    _TYPES = {N.DT_F64: "<f8", N.DT_F32: "<f4", N.DT_I64: "<i8"}

    def __init__(self, ptr, count, dtype):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": self._TYPES[dtype],
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


class TorchComm:
    """life_comm backed by torch.distributed (NCCL on GPUs, gloo in tests)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        self.error = None
        self.host_staged = dist.get_backend(group) == "gloo"

        def _allreduce(buf, count, dtype, op, stream, ctx):
            try:
                import torch
                t = torch.as_tensor(_CudaArray(buf, count, dtype), device="cuda")
                red = dist.ReduceOp.SUM if op == N.OP_SUM else dist.ReduceOp.MAX
                s = torch.cuda.ExternalStream(stream) if stream else torch.cuda.default_stream()
                with torch.cuda.stream(s):
                    if self.host_staged:  # gloo (tests): through host memory
                        h = t.cpu()
                        dist.all_reduce(h, op=red, group=self.group)
                        t.copy_(h)
                    else:                 # NCCL: enqueued, stream-ordered
                        dist.all_reduce(t, op=red, group=self.group)
                return 0
            except Exception as exc:  # reported by the C side as LIFE_ERR_NCCL
                self.error = exc
                return 1

        self._fn = N.ALLREDUCE_FN(_allreduce)
        self.c = N.CommC(allreduce=self._fn, ctx=None, rank=self.rank, nranks=self.nranks)


class NcclComm:
    """life_comm over the library's own NCCL communicator (life_comm_init_nccl):
    ncclAllReduce enqueued by the C side on the solver stream, capturable, so
    sharded iterations run as CUDA graphs.  The 128-byte ncclUniqueId is made
    on rank 0 and broadcast over the torch.distributed group (any backend)."""

    def __init__(self, group=None, rank=None, nranks=None):
        import torch
        if rank is None or nranks is None:
            import torch.distributed as dist
            rank, nranks = dist.get_rank(group), dist.get_world_size(group)
            uid = torch.zeros(128, dtype=torch.uint8)
            if rank == 0:
                buf = ctypes.create_string_buffer(128)
                N.check(N.lib().life_nccl_unique_id(buf))
                uid = torch.frombuffer(bytearray(buf.raw), dtype=torch.uint8)
            if dist.get_backend(group) == "nccl":
                uid = uid.cuda()
                dist.broadcast(uid, src=dist.get_global_rank(group, 0) if group else 0, group=group)
                uid = uid.cpu()
            else:
                dist.broadcast(uid, src=0, group=group)
            raw = bytes(uid.numpy().tobytes())
        else:  # single process (world 1): a local id
            buf = ctypes.create_string_buffer(128)
            N.check(N.lib().life_nccl_unique_id(buf))
            raw = buf.raw
        self.rank, self.nranks, self.error = int(rank), int(nranks), None
        self.c = N.CommC()
        idbuf = ctypes.create_string_buffer(raw, 128)
        N.check(N.lib().life_comm_init_nccl(idbuf, self.rank, self.nranks, ctypes.byref(self.c)))

    def close(self):
        if self.c is not None and self.c.ctx:
            N.lib().life_comm_destroy_nccl(ctypes.byref(self.c))

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_sharded(problem, config=None, group=None, w0=None, ranges=None, comm=None):
    """SBBNNLS with Phi voxel-sharded over the ranks of a torch.distributed
    group (every rank calls it with the same problem).  Returns (w, trace);
    both are identical on all ranks.  `comm` reuses a communicator
    (NcclComm / TorchComm) across calls; by default one is made per call."""
    import torch

    from . import device
    from .sbbnnls import SolverConfig, SolverSession, trace_from

    config = config or SolverConfig()
    if config.precision != "fp32":
        raise ConfigInvalid("voxel-sharded solves run the fp32 path")
    import torch.distributed as dist
    # NCCL process groups: the library's own capturable NCCL communicator
    # (graphs on); other backends (gloo in tests): the torch callback
    if comm is None:
        comm = NcclComm(group) if dist.get_backend(group) == "nccl" else TorchComm(group)
    if ranges is None:
        # shards built on the GPUs from 1/N host slices (shard_from_slices)
        op, b, _, _ = shard_from_slices(problem, group)
    else:  # caller-chosen ranges: host selection
        v0, v1 = ranges[comm.rank]
        t, dic, b_host = shard_problem(problem.tensor, problem.dictionary, problem.y, v0, v1)
        op = device.DeviceOperator(t, dic)
        vmax, fmax = global_fix_bounds(problem.tensor)
        N.check(N.lib().life_phi_set_fix_bounds(op.handle, vmax, 0.0, fmax))
        b = torch.from_numpy(b_host).to(device="cuda", dtype=torch.float32)
    if w0 is None:
        w = torch.empty(problem.dims.n_fibers, dtype=torch.float32, device="cuda")
    else:
        w = torch.from_numpy(np.asarray(w0, dtype=np.float64)).to(device="cuda",
                                                                  dtype=torch.float32)
    sess = SolverSession(op, b, w, config, has_w0=w0 is not None, comm=comm)
    done = False
    while not done:
        sess.iterate(config.poll_every)
        done = sess.poll()
    if comm.error is not None:
        raise comm.error
    res, recs = sess.finish()
    sess.close()
    return w.cpu().numpy().astype(np.float64), trace_from(res, recs)


__all__ = ["NcclComm", "TorchComm", "global_fix_bounds", "shard_problem", "shard_voxel_ranges",
           "solve_sharded"]
