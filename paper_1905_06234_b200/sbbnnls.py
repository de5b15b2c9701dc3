"""SBBNNLS (Alg. 1) driven entirely on the B200.

Drop-in for /root/reference/pkg/src/lifespmv/sbbnnls.py:34-291.  The whole
iteration (DSC -> WC -> projection -> step size -> update) runs on the device
through the C-ABI ``life_solve``: scalars never leave HBM, iteration pairs
are replayed as one CUDA graph, and the host polls the termination flag
every ``poll_every`` iterations.  Control flow, termination reasons, call
counts and trace fields follow the reference exactly.
"""

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from . import device, engine
from .errors import ConfigInvalid, DegenerateStep

DEFAULT_MAX_ITERS = 500


@dataclass
class SolverConfig:
    """Solver controls (sbbnnls.py:34-62) plus device options.

    ``threads``, the restructure keys and strategies are validated exactly
    as the reference's ``_runners`` would (``solve`` raises
    StrategyRequiresSorted / ConfigInvalid for incompatible pairs before any
    device work); the device then uses its own voxel-major tile layout for
    both products.  ``precision``: "fp32" (fast) or "fp64" (bit-exact
    kernels)."""

    max_iters: int = DEFAULT_MAX_ITERS
    grad_tol: float = 1e-12
    threads: int = 1
    dsc_restructure: str = "voxel"
    wc_restructure: str = "atom"
    dsc_strategy: engine.PartitionStrategy = None
    wc_strategy: engine.PartitionStrategy = None
    skip_zero: bool = True
    precision: str = "fp32"
    use_graph: bool = True
    poll_every: int = 16

    def __post_init__(self):
        if self.max_iters < 1:
            raise ConfigInvalid("max_iters must be >= 1")
        if self.grad_tol < 0:
            raise ConfigInvalid("grad_tol must be >= 0")
        if self.threads < 1:
            raise ConfigInvalid("threads must be >= 1")
        for key in (self.dsc_restructure, self.wc_restructure):
            if key not in ("none", "atom", "voxel", "fiber"):
                raise ConfigInvalid(f"unknown restructure key {key!r}")
        if self.precision not in ("fp32", "fp64"):
            raise ConfigInvalid(f"unknown precision {self.precision!r}")


@dataclass
class TraceRecord:
    """One completed iteration (sbbnnls.py:65-85)."""

    iteration: int
    objective: float
    alpha: float
    grad_norm: float
    zeros: int
    dsc_seconds: float
    wc_seconds: float
    dsc_calls: int
    wc_calls: int
    dsc_skipped: int
    w_min: float


@dataclass
class SolverTrace:
    records: list = field(default_factory=list)
    termination: str = ""
    initial_objective: float = float("nan")
    final_objective: float = float("nan")
    total_dsc_calls: int = 0
    total_wc_calls: int = 0
    loop_seconds: float = 0.0
    setup_seconds: float = 0.0   # operator build (H2D + restructuring) + uploads

    @property
    def iterations(self):
        return len(self.records)


def project_nonneg(v):
    """Clamp to the nonnegative orthant (sbbnnls.py:102-104)."""
    return np.maximum(v, 0.0)


def project_gradient(g, w):
    """Zero the components at active coordinates that point outward
    (sbbnnls.py:107-116)."""
    out = np.array(g, dtype=np.float64, copy=True)
    out[(np.asarray(w) == 0.0) & (out > 0.0)] = 0.0
    return out


def _mv(problem, precision):
    def mv(w):
        y = np.zeros(problem.dims.signal_len)
        engine.dsc_sequential(problem.tensor, problem.dictionary, w, y, precision=precision)
        return y
    return mv


def _mtv(problem, precision):
    def mtv(y):
        w = np.zeros(problem.dims.n_fibers)
        engine.wc_sequential(problem.tensor, problem.dictionary, y, w, precision=precision)
        return w
    return mtv


def gradient(problem, w, *, precision=None):
    """M^T (M w - y) (sbbnnls.py:186-189)."""
    return _mtv(problem, precision)(_mv(problem, precision)(w) - problem.y)


def objective(problem, w, *, precision=None):
    """0.5 ||M w - y||^2 (sbbnnls.py:192-196)."""
    r = _mv(problem, precision)(w) - problem.y
    return 0.5 * engine.inner_dot(r, r)


def step_size(iter_index, g_tilde, problem, *, precision=None):
    """Barzilai-Borwein step for the iteration parity (sbbnnls.py:199-220)."""
    mg = _mv(problem, precision)(g_tilde)
    if iter_index % 2 == 1:
        num, den = engine.inner_dot(g_tilde, g_tilde), engine.inner_dot(mg, mg)
    else:
        mtmg = _mtv(problem, precision)(mg)
        num, den = engine.inner_dot(mg, mg), engine.inner_dot(mtmg, mtmg)
    if den == 0.0:
        raise DegenerateStep(f"zero step denominator at iteration {iter_index}")
    return num / den


def check_restructure_pairs(ordering, config):
    """Validate (op, restructure key, strategy) the way the reference's
    ``_runners`` do (sbbnnls.py:119-167): the strategy defaults to
    ``best_partition(op, key)`` and must suit the ordering of the copy the
    key produces (``sort_by`` tags ``by_<key>``; "none" keeps the tensor's
    own).  Only metadata is involved, no sort runs."""
    from .restructure import best_partition
    if config.threads < 1:
        raise ConfigInvalid("threads must be >= 1")
    for op, key, strategy in (("dsc", config.dsc_restructure, config.dsc_strategy),
                              ("wc", config.wc_restructure, config.wc_strategy)):
        if strategy is None:
            strategy = best_partition(op, key)
        engine.check_strategy_ordering(strategy, ordering if key == "none" else f"by_{key}")


def solve_device(op, b, w, config, stream=None):
    """Run ``life_solve`` on device tensors: b (signal) and w (in: w0 when
    ``w`` is given initialised, out: final weights).  Returns the raw C result
    and records.  ``w0_given`` is signalled by ``config._w0`` (internal)."""
    torch = N.require_cuda()
    cfg = N.SolverConfigC(max_iters=config.max_iters, skip_zero=int(config.skip_zero),
                          exact_f64=int(config.precision == "fp64"),
                          has_w0=int(getattr(config, "_has_w0", False)),
                          grad_tol=float(config.grad_tol), poll_every=int(config.poll_every),
                          use_graph=int(config.use_graph), comm=None)
    recs = (N.TraceRecordC * config.max_iters)()
    res = N.SolverResultC()
    N.check(N.lib().life_solve(op.handle, ctypes.c_void_p(b.data_ptr()),
                               ctypes.c_void_p(w.data_ptr()), ctypes.byref(cfg), recs,
                               ctypes.byref(res), N.stream_ptr(stream)))
    del torch
    return res, recs


class SolverSession:
    """Stepwise device solver over an operator (C-ABI life_sbb_*).

    ``b`` and ``w`` are CUDA tensors of the session precision; ``w`` holds
    w0 when ``has_w0`` and receives the iterates.  Used by bench.py to time
    exactly N iterations, and by the multi-GPU driver."""

    def __init__(self, op, b, w, config, has_w0=False, stream=None, comm=None):
        N.require_cuda()
        self.config = config
        self._b, self._w, self._stream = b, w, stream
        self._comm = comm  # keeps the ctypes callback alive for the session
        cfg = N.SolverConfigC(max_iters=config.max_iters, skip_zero=int(config.skip_zero),
                              exact_f64=int(config.precision == "fp64"), has_w0=int(has_w0),
                              grad_tol=float(config.grad_tol),
                              poll_every=int(config.poll_every),
                              use_graph=int(config.use_graph),
                              comm=ctypes.pointer(comm.c) if comm is not None else None)
        h = ctypes.c_void_p()
        N.check(N.lib().life_sbb_create(op.handle, ctypes.c_void_p(b.data_ptr()),
                                        ctypes.c_void_p(w.data_ptr()), ctypes.byref(cfg),
                                        N.stream_ptr(stream), ctypes.byref(h)))
        self._h = h
        self._op = op  # keep the operator alive

    def iterate(self, n):
        N.check(N.lib().life_sbb_iterate(self._h, int(n), N.stream_ptr(self._stream)))

    def poll(self):
        done = ctypes.c_int(0)
        N.check(N.lib().life_sbb_poll(self._h, ctypes.byref(done), N.stream_ptr(self._stream)))
        return bool(done.value)

    def finish(self):
        recs = (N.TraceRecordC * self.config.max_iters)()
        res = N.SolverResultC()
        N.check(N.lib().life_sbb_finish(self._h, recs, ctypes.byref(res),
                                        N.stream_ptr(self._stream)))
        return res, recs

    def close(self):
        if self._h:
            N.lib().life_sbb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover - interpreter shutdown
            pass


def trace_from(res, recs, setup_seconds=0.0):
    """SolverTrace from the C result and trace records."""
    trace = SolverTrace(termination=N.TERM_NAMES.get(res.termination, "max_iters"),
                        initial_objective=res.initial_objective,
                        final_objective=res.final_objective,
                        total_dsc_calls=int(res.total_dsc_calls),
                        total_wc_calls=int(res.total_wc_calls),
                        loop_seconds=res.loop_seconds, setup_seconds=setup_seconds)
    for i in range(res.iterations):
        r = recs[i]
        trace.records.append(TraceRecord(
            iteration=r.iteration, objective=r.objective, alpha=r.alpha,
            grad_norm=r.grad_norm, zeros=r.zeros, dsc_seconds=r.dsc_seconds,
            wc_seconds=r.wc_seconds, dsc_calls=r.dsc_calls, wc_calls=r.wc_calls,
            dsc_skipped=int(r.dsc_skipped), w_min=r.w_min))
    return trace


def solve(problem, w0=None, config=None):
    """Run the solver on the B200; returns (weights, trace) like
    sbbnnls.solve (sbbnnls.py:223-291)."""
    if config is None:
        config = SolverConfig()
    if problem.y is None:
        raise ConfigInvalid("problem has no signal vector to fit")
    check_restructure_pairs(problem.tensor.ordering, config)
    torch = N.require_cuda()
    t_setup = time.perf_counter()
    exact = config.precision == "fp64"
    dtype = torch.float64 if exact else torch.float32
    op = device.operator_for(problem.tensor, problem.dictionary, exact=exact)
    b = device.upload(np.asarray(problem.y, dtype=np.float64), dtype)
    if w0 is None:
        w = torch.empty(problem.dims.n_fibers, dtype=dtype, device="cuda")
    else:
        w = device.upload(np.asarray(w0, dtype=np.float64), dtype)
    config._has_w0 = w0 is not None
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t_setup
    res, recs = solve_device(op, b, w, config)
    # D2H in the solve's own dtype, widened on the host (exact)
    return w.cpu().numpy().astype(np.float64), trace_from(res, recs, t_setup)
