"""DSC / WC entry points with the reference engine's signatures.

Drop-in for /root/reference/pkg/src/lifespmv/engine.py:45-434.  Plans,
strategies and their validation are host logic and behave exactly like the
reference (same chunk boundaries, same exceptions).  The products
themselves always run on the B200 through liblife_b200 -- a plan's chunks
are validated, then honoured trivially: on the device every output row has
exactly one writer (a warp owns a voxel range for DSC; WC accumulates per
fascicle in order-independent fixed point), so every regime of the
reference (ownership, edge- and full-privatization) gives the sequential
result.
"""

import math
from dataclasses import dataclass

import numpy as np

from . import device
from .errors import (
    ConfigInvalid,
    DimensionMismatch,
    PlanTensorMismatch,
    StrategyRequiresSorted,
)
from .tensor import OffsetPhiTensor

PARTITION_KINDS = ("coefficient", "atom", "voxel", "fiber")
_NEEDS = {"atom": "by_atom", "voxel": "by_voxel", "fiber": "by_fiber"}


@dataclass(frozen=True)
class PartitionStrategy:
    """How a coefficient range is split (engine.py:45-61)."""

    kind: str = "coefficient"
    sync_free: bool = False

    def __post_init__(self):
        if self.kind not in PARTITION_KINDS:
            raise ConfigInvalid(f"unknown partition kind {self.kind!r}")


@dataclass(frozen=True)
class ExecutionPlan:
    """Strategy bound to half-open chunks (engine.py:64-75)."""

    strategy: PartitionStrategy
    threads: int
    chunks: tuple


@dataclass
class KernelStats:
    """Zero-weight skips and elapsed seconds of one call (engine.py:78-83).

    ``elapsed`` is the device time of the kernels (CUDA events)."""

    skipped_coefficients: int = 0
    elapsed: float = 0.0


def _phi(t):
    return t.tensor if isinstance(t, OffsetPhiTensor) else t


def snap_to_run_boundaries(key_array, boundaries):
    """Move interior split points off runs (engine.py:113-136): to the run
    end adding fewer coefficients to the gaining worker, ties to the later
    worker (the run start), then restore monotonicity."""
    keys = np.asarray(key_array)
    n = len(keys)
    out = [int(b) for b in boundaries]
    for i in range(1, len(out) - 1):
        b = out[i]
        if 0 < b < n and keys[b - 1] == keys[b]:
            lo = int(np.searchsorted(keys, keys[b], side="left"))
            hi = int(np.searchsorted(keys, keys[b], side="right"))
            out[i] = lo if (b - lo) <= (hi - b) else hi
    for i in range(1, len(out)):
        out[i] = max(out[i], out[i - 1])
    return out


def _equal_split(nc, threads):
    step = math.ceil(nc / threads) if nc else 0
    return [min(i * step, nc) for i in range(threads + 1)]


def _whole_runs(keys, nc, threads):
    if nc == 0:
        return [0] * (threads + 1)
    starts = np.concatenate(([0], np.flatnonzero(np.diff(keys)) + 1, [nc]))
    n_runs = len(starts) - 1
    per = math.ceil(n_runs / threads)
    return [int(starts[min(i * per, n_runs)]) for i in range(threads + 1)]


def check_strategy_ordering(strategy, ordering):
    """The ordering requirements build_plan enforces (engine.py:166-180),
    raised in the same order with the same messages; usable without a
    tensor (the solver validates its restructure/strategy pairs up front)."""
    if strategy.kind == "coefficient":
        if strategy.sync_free and ordering != "by_voxel":
            raise StrategyRequiresSorted("sync_free requires a voxel-sorted tensor")
        return
    want = _NEEDS[strategy.kind]
    if ordering != want:
        raise StrategyRequiresSorted(
            f"{strategy.kind} partitioning requires ordering {want!r}, "
            f"tensor is {ordering!r}")
    if strategy.sync_free and strategy.kind != "voxel":
        raise StrategyRequiresSorted("sync_free applies to voxel-run splits")


def build_plan(tensor, strategy, threads):
    """Chunk boundaries for a strategy on this tensor (engine.py:155-184)."""
    if threads < 1:
        raise ConfigInvalid("threads must be >= 1")
    phi = _phi(tensor)
    nc = phi.dims.n_coeffs
    check_strategy_ordering(strategy, phi.ordering)
    if strategy.kind == "coefficient":
        bounds = _equal_split(nc, threads)
        if strategy.sync_free:
            bounds = snap_to_run_boundaries(phi.voxels, bounds)
    else:
        bounds = _whole_runs(phi.key_array(strategy.kind), nc, threads)
    chunks = tuple((bounds[i], bounds[i + 1]) for i in range(threads))
    return ExecutionPlan(strategy=strategy, threads=threads, chunks=chunks)


def _check_coverage(plan, nc):
    pos = 0
    for s, e in plan.chunks:
        if s != pos or e < s:
            raise PlanTensorMismatch("chunks do not tile the coefficient range")
        pos = e
    if pos != nc:
        raise PlanTensorMismatch(f"plan covers [0, {pos}), tensor has {nc} coefficients")


def _on_runs(keys, plan):
    n = len(keys)
    return all(not (0 < s < n and keys[s - 1] == keys[s]) for s, _ in plan.chunks[1:])


def _length(x):
    return int(x.shape[0]) if hasattr(x, "shape") else len(x)


def _check_args(tensor, dictionary, weights, signal):
    d = tensor.dims
    if _length(tensor.values) != d.n_coeffs:
        raise DimensionMismatch("tensor arrays disagree with dims.n_coeffs")
    if _length(dictionary.data) != d.dict_len:
        raise DimensionMismatch("dictionary length != n_atoms * n_dirs")
    if _length(weights) != d.n_fibers:
        raise DimensionMismatch("w length != n_fibers")
    if _length(signal) != d.signal_len:
        raise DimensionMismatch("y length != n_voxels * n_dirs")


def dsc_sequential(tensor, dictionary, w, y_out, *, skip_zero=True, precision=None):
    """y_out += M w (engine.py:218-233) on the B200.

    ``precision`` ("fp32" default / "fp64" bit-exact) selects the kernel
    family; see :mod:`paper_1905_06234_b200.device`."""
    _check_args(tensor, dictionary, w, y_out)
    if tensor.dims.n_coeffs == 0:
        return KernelStats(0, 0.0)
    skipped, secs = device.dsc_accumulate(tensor, dictionary, w, y_out, skip_zero, precision)
    return KernelStats(skipped, secs)


def wc_sequential(tensor, dictionary, y, w_out, *, precision=None):
    """w_out += M^T y (engine.py:236-244) on the B200."""
    _check_args(tensor, dictionary, w_out, y)
    if tensor.dims.n_coeffs == 0:
        return KernelStats(0, 0.0)
    secs = device.wc_accumulate(tensor, dictionary, y, w_out, precision)
    return KernelStats(0, secs)


def dsc_parallel(tensor, dictionary, w, y_out, plan, *, skip_zero=True, precision=None):
    """y_out += M w following a plan (engine.py:247-274): the plan is
    validated exactly as the reference does; the device computes every voxel
    block with a single writer."""
    phi = _phi(tensor)
    _check_args(tensor, dictionary, w, y_out)
    _check_coverage(plan, phi.dims.n_coeffs)
    if plan.strategy.sync_free or plan.strategy.kind == "voxel":
        if phi.ordering != "by_voxel":
            raise PlanTensorMismatch("run-aligned DSC plan needs a voxel-sorted tensor")
        if not _on_runs(phi.voxels, plan):
            raise PlanTensorMismatch("plan chunk straddles a voxel run")
    return dsc_sequential(tensor, dictionary, w, y_out, skip_zero=skip_zero,
                          precision=precision)


def wc_parallel(tensor, dictionary, y, w_out, plan, *, precision=None):
    """w_out += M^T y following a plan (engine.py:372-413)."""
    phi = _phi(tensor)
    _check_args(tensor, dictionary, w_out, y)
    _check_coverage(plan, phi.dims.n_coeffs)
    if plan.strategy.kind == "fiber" and not (
            phi.ordering == "by_fiber" and _on_runs(phi.fibers, plan)):
        raise PlanTensorMismatch("fiber plan needs fiber-run-aligned chunks")
    return wc_sequential(tensor, dictionary, y, w_out, precision=precision)


def inner_axpy(scale, src, dst):
    """dst += scale * src over a direction span (engine.py:416-425)."""
    if scale == 0.0:
        return
    dst += scale * src


def inner_dot(a, b):
    """Dot product over a span (engine.py:428-434)."""
    return float(np.dot(a, b))
