"""ctypes binding of liblife_b200.so (the C ABI in include/life_b200.h).

The shared library is built in-tree (``make -C paper_1905_06234_b200/csrc``
or ``python __graft_entry__.py``).  There is no fallback: if the library or a
CUDA device is missing, every compute entry point raises.
"""

import ctypes
import os

from .errors import DeviceError, raise_for_status

_HERE = os.path.dirname(os.path.abspath(__file__))
# LIFE_B200_LIB overrides the path (diagnostic builds, tools/ only)
LIB_PATH = os.environ.get("LIFE_B200_LIB") or os.path.join(_HERE, "liblife_b200.so")

c_i32, c_i64, c_u32, c_u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64
c_void_p, c_double = ctypes.c_void_p, ctypes.c_double

# flags (life_b200.h)
PHI_HOST_INPUT = 0x1
PHI_EXACT_F64 = 0x2
PHI_NO_FAST_F32 = 0x4
PHI_FORCE_SPARSE = 0x8
PHI_FORCE_DENSE = 0x10
PHI_NO_TENSOR = 0x20
PHI_TENSOR = 0x40
PHI_NO_BIN = 0x80
PHI_VALUES_F32 = 0x100
ACCUMULATE = 0x01
SKIP_ZERO = 0x02
SUBTRACT_B = 0x04
PROJECT_GRAD = 0x08
TERM_NAMES = {1: "max_iters", 2: "grad_tol", 3: "degenerate_step"}


class Dims(ctypes.Structure):
    _fields_ = [("n_atoms", c_i64), ("n_voxels", c_i64), ("n_fibers", c_i64),
                ("n_dirs", c_i64), ("n_coeffs", c_i64)]


class PhiInfo(ctypes.Structure):
    _fields_ = [("dims", Dims), ("atom_groups", c_i32), ("atoms_per_group", c_i32),
                ("n_warps", c_i32), ("has_exact", c_i32), ("n_voxel_runs", c_i64),
                ("n_fiber_runs", c_i64), ("max_fiber_run", c_i64),
                ("max_voxel_run", c_i64), ("device_bytes", c_i64), ("sort_ms", c_double),
                ("tensor_ops", c_i32), ("reserved", c_i32)]


class SpmvOut(ctypes.Structure):
    _fields_ = [("skipped", c_void_p), ("sumsq", c_void_p), ("absmax", c_void_p)]


# int (*)(void *buf, int64_t count, int dtype, int op, void *stream, void *ctx)
ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, c_void_p, c_i64, ctypes.c_int, ctypes.c_int,
                                c_void_p, c_void_p)
DT_F64, DT_F32, DT_I64 = 0, 1, 2
OP_SUM, OP_MAX = 0, 1


class CommC(ctypes.Structure):
    _fields_ = [("allreduce", ALLREDUCE_FN), ("ctx", c_void_p), ("rank", c_i32),
                ("nranks", c_i32), ("capturable", c_i32), ("reserved", c_i32)]


class SolverConfigC(ctypes.Structure):
    _fields_ = [("max_iters", c_i32), ("skip_zero", c_i32), ("exact_f64", c_i32),
                ("has_w0", c_i32), ("grad_tol", c_double), ("poll_every", c_i32),
                ("use_graph", c_i32), ("comm", ctypes.POINTER(CommC))]


class TraceRecordC(ctypes.Structure):
    _fields_ = [("iteration", c_i32), ("zeros", c_i32), ("dsc_skipped", c_i64),
                ("objective", c_double), ("alpha", c_double), ("grad_norm", c_double),
                ("w_min", c_double), ("dsc_seconds", c_double), ("wc_seconds", c_double),
                ("dsc_calls", c_i32), ("wc_calls", c_i32)]


class SolverResultC(ctypes.Structure):
    _fields_ = [("termination", c_i32), ("iterations", c_i32),
                ("initial_objective", c_double), ("final_objective", c_double),
                ("total_dsc_calls", c_i64), ("total_wc_calls", c_i64),
                ("loop_seconds", c_double)]


# every symbol the header declares: name -> (restype, argtypes)
SIGNATURES = {
    "life_abi_version": (ctypes.c_int, []),
    "life_status_string": (ctypes.c_char_p, [ctypes.c_int]),
    "life_last_error": (ctypes.c_char_p, []),
    "life_launch_count": (c_u64, []),
    "life_phi_create": (ctypes.c_int, [ctypes.POINTER(Dims), c_void_p, c_void_p, c_void_p,
                                       c_void_p, c_void_p, c_u32, c_void_p,
                                       ctypes.POINTER(c_void_p), ctypes.POINTER(c_i64)]),
    "life_phi_destroy": (ctypes.c_int, [c_void_p]),
    "life_release_cached_memory": (ctypes.c_int, []),
    "life_cached_memory_bytes": (ctypes.c_int, [ctypes.POINTER(c_i64)]),
    "life_copy_h2d": (ctypes.c_int, [c_void_p, c_void_p, c_i64, c_void_p]),
    "life_copy_h2d_f32": (ctypes.c_int, [c_void_p, c_void_p, c_i64, c_void_p]),
    "life_phi_get_info": (ctypes.c_int, [c_void_p, ctypes.POINTER(PhiInfo)]),
    "life_stable_argsort_u32": (ctypes.c_int, [c_void_p, c_i64, c_void_p, c_void_p]),
    "life_detect_runs_u32": (ctypes.c_int, [c_void_p, c_i64, c_void_p, c_void_p,
                                            ctypes.POINTER(c_i64), c_void_p]),
    "life_gather_coo": (ctypes.c_int, [c_void_p, c_i64, c_void_p, c_void_p, c_void_p,
                                       c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                       c_void_p]),
    "life_dsc_f32": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_u32,
                                    ctypes.POINTER(SpmvOut), c_void_p]),
    "life_wc_f32": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                                   c_u32, ctypes.POINTER(SpmvOut), c_void_p]),
    "life_dsc_f64": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_u32, c_void_p,
                                    c_void_p]),
    "life_wc_f64": (ctypes.c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "life_solve": (ctypes.c_int, [c_void_p, c_void_p, c_void_p,
                                  ctypes.POINTER(SolverConfigC),
                                  ctypes.POINTER(TraceRecordC),
                                  ctypes.POINTER(SolverResultC), c_void_p]),
    "life_sbb_create": (ctypes.c_int, [c_void_p, c_void_p, c_void_p,
                                       ctypes.POINTER(SolverConfigC), c_void_p,
                                       ctypes.POINTER(c_void_p)]),
    "life_sbb_iterate": (ctypes.c_int, [c_void_p, ctypes.c_int, c_void_p]),
    "life_sbb_poll": (ctypes.c_int, [c_void_p, ctypes.POINTER(ctypes.c_int), c_void_p]),
    "life_sbb_finish": (ctypes.c_int, [c_void_p, ctypes.POINTER(TraceRecordC),
                                       ctypes.POINTER(SolverResultC), c_void_p]),
    "life_sbb_destroy": (ctypes.c_int, [c_void_p]),
    "life_phi_set_fix_bounds": (ctypes.c_int, [c_void_p, c_double, c_double, c_i64]),
    "life_nccl_unique_id": (ctypes.c_int, [c_void_p]),
    "life_comm_init_nccl": (ctypes.c_int, [c_void_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(CommC)]),
    "life_comm_destroy_nccl": (ctypes.c_int, [ctypes.POINTER(CommC)]),
    "life_phi_get_fix_bounds": (ctypes.c_int, [c_void_p, ctypes.POINTER(c_double),
                                               ctypes.POINTER(c_double),
                                               ctypes.POINTER(c_i64)]),
}

_lib = None


class NativeUnavailable(DeviceError):
    """liblife_b200.so is missing or cannot be loaded."""


def lib():
    """Load (once) and return the bound library.  Raises, never falls back."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(
            f"{LIB_PATH} is not built; run `make -C {os.path.join(_HERE, 'csrc')}` "
            "or `python __graft_entry__.py`")
    try:
        handle = ctypes.CDLL(LIB_PATH)
    except OSError as exc:  # pragma: no cover - environment specific
        raise NativeUnavailable(f"cannot load {LIB_PATH}: {exc}") from exc
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    _lib = handle
    return _lib


def check(status, position=None):
    """Raise the LifeError matching a nonzero status (with the C message)."""
    if status != 0:
        msg = lib().life_last_error().decode(errors="replace")
        raise_for_status(status, msg, position)


def launch_count():
    return int(lib().life_launch_count())


def cached_memory_bytes():
    """Device bytes of destroyed operators / sessions kept for reuse."""
    n = c_i64(0)
    check(lib().life_cached_memory_bytes(ctypes.byref(n)))
    return int(n.value)


def release_cached_memory():
    """Hand the library's cached device blocks back to the driver."""
    check(lib().life_release_cached_memory())


def require_cuda():
    """Fail loudly when no CUDA device is visible (no CPU fallback exists)."""
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the LiFE B200 path has no CPU fallback")
    lib()
    return torch


def stream_ptr(stream=None):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)
