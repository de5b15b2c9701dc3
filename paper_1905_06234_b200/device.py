"""Device-resident operator: a life_phi handle plus its call wrappers.

``DeviceOperator`` owns the restructured copies of Phi and D in HBM
(C-ABI ``life_phi_create``).  ``dsc``/``wc`` run one product through the
C ABI on either host arrays (numpy: copied in and out) or CUDA tensors
(used in place).  Two precisions:

* ``"fp32"`` -- the fast path: tile-shaped operators run the binned
  two-phase products (tcgen05 tile contraction + shared-memory fascicle
  bins, exact integer reductions; ~5e-7 relative L2 of the reference),
  operators whose voxels carry few atoms the voxel-segment kernels.
* ``"fp64"`` -- the bit-exact path: same rounding and per-output order as
  the reference loops (_kernels.py:14-68), equal to
  ``dsc_sequential``/``wc_sequential`` bit for bit.
"""

import ctypes
import warnings
import weakref

import numpy as np

from . import _native as N
from .errors import ConfigInvalid, DimensionMismatch
from .tensor import OffsetPhiTensor

_DEFAULT_PRECISION = ["fp32"]
# Frozen (read-only) numpy arrays are only ever copied to the device.
warnings.filterwarnings("ignore", message="The given NumPy array is not writable")


_LAYOUT = ["auto"]


_LAYOUTS = ("auto", "sparse", "dense", "bin")


def set_layout(name):
    """fp32 kernel family for operators built from now on: "auto" (density
    heuristic: "bin" for tile-shaped operators, else "sparse"), "sparse"
    (voxel-segment kernels) or "bin" / "dense" (binned two-phase products:
    tcgen05 tile side + shared-memory fascicle bins, n_dirs <= 192; larger
    direction counts take the voxel-segment kernels).  The round-1
    single-pass tile families ("fma", "tensor") were retired in round 2."""
    if name not in _LAYOUTS:
        raise ConfigInvalid(f"layout must be one of {'/'.join(_LAYOUTS)}, got {name!r}")
    _LAYOUT[0] = name


def layout():
    return _LAYOUT[0]


def set_default_precision(precision):
    if precision not in ("fp32", "fp64"):
        raise ConfigInvalid(f"precision must be 'fp32' or 'fp64', got {precision!r}")
    _DEFAULT_PRECISION[0] = precision


def default_precision():
    return _DEFAULT_PRECISION[0]


def _phi(tensor):
    return tensor.tensor if isinstance(tensor, OffsetPhiTensor) else tensor


def upload(arr, dtype=None, stream=None):
    """Host numpy array -> new CUDA tensor through the library's pinned
    staging copy (life_copy_h2d: ~50 GB/s against ~7 GB/s for a pageable
    torch .to("cuda")); `dtype` converts on the device afterwards."""
    torch = N.require_cuda()
    a = np.ascontiguousarray(arr)
    if a.dtype == np.float64 and dtype == torch.float32:  # rounded while staging
        t = torch.empty(a.shape, dtype=torch.float32, device="cuda")
        N.check(N.lib().life_copy_h2d_f32(ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(a.ctypes.data),
                                          a.size, N.stream_ptr(stream)))
        return t
    tdt = {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32,
           np.dtype(np.uint32): torch.int32, np.dtype(np.int32): torch.int32,
           np.dtype(np.int64): torch.int64}[a.dtype]
    t = torch.empty(a.shape, dtype=tdt, device="cuda")
    N.check(N.lib().life_copy_h2d(ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(a.ctypes.data),
                                  a.nbytes, N.stream_ptr(stream)))
    return t if dtype is None or dtype == tdt else t.to(dtype)


class DeviceOperator:
    """The operator M = Phi x_1 D resident on the current CUDA device."""

    def __init__(self, tensor, dictionary, exact=False, fast=True, stream=None):
        torch = N.require_cuda()
        phi = _phi(tensor)
        d = phi.dims
        if dictionary.data.shape[0] != d.dict_len:
            raise DimensionMismatch("dictionary length != n_atoms * n_dirs")
        self.dims = d
        self.exact = bool(exact)
        self.fast = bool(fast)
        nc = d.n_coeffs
        # host arrays straight into life_phi_create (LIFE_PHI_HOST_INPUT):
        # the library stages them through pinned buffers
        u32 = (lambda x: np.ascontiguousarray(x, dtype=np.uint32) if nc else None)
        a, v, f = u32(phi.atoms), u32(phi.voxels), u32(phi.fibers)
        val = np.ascontiguousarray(phi.values, dtype=np.float64) if nc else None
        dic = np.ascontiguousarray(dictionary.data, dtype=np.float64)
        self._create(d, a, v, f, val, dic, stream, host=True)

    @classmethod
    def from_device(cls, dims, atoms, voxels, fibers, values, dictionary,
                    exact=False, fast=True, stream=None):
        """Build from CUDA tensors (u32 indices viewed as int32, f64 values)."""
        self = cls.__new__(cls)
        N.require_cuda()
        self.dims, self.exact, self.fast = dims, bool(exact), bool(fast)
        self._create(dims, atoms, voxels, fibers, values, dictionary, stream)
        return self

    def _create(self, d, a, v, f, val, dic, stream, host=False):
        flags = (N.PHI_EXACT_F64 if self.exact else 0) | (0 if self.fast else N.PHI_NO_FAST_F32)
        # host input: the fp32-only operator lets values cross PCIe as f32
        flags |= (N.PHI_HOST_INPUT | (0 if self.exact else N.PHI_VALUES_F32)) if host else 0
        flags |= {"auto": 0, "sparse": N.PHI_FORCE_SPARSE, "dense": N.PHI_FORCE_DENSE,
                  "bin": N.PHI_FORCE_DENSE}[_LAYOUT[0]]
        dims = N.Dims(d.n_atoms, d.n_voxels, d.n_fibers, d.n_dirs, d.n_coeffs)
        handle = ctypes.c_void_p()
        bad = ctypes.c_int64(-1)
        ptr = (lambda t: None if t is None else ctypes.c_void_p(
            t.ctypes.data if isinstance(t, np.ndarray) else t.data_ptr()))
        st = N.stream_ptr(stream)
        rc = N.lib().life_phi_create(ctypes.byref(dims), ptr(a), ptr(v), ptr(f), ptr(val),
                                     ptr(dic), flags, st, ctypes.byref(handle),
                                     ctypes.byref(bad))
        N.check(rc, bad.value)
        self._handle = handle
        self._finalizer = weakref.finalize(self, N.lib().life_phi_destroy, handle)
        info = N.PhiInfo()
        N.check(N.lib().life_phi_get_info(handle, ctypes.byref(info)))
        self.info = info

    @property
    def kind(self):
        """"bin" (binned two-phase products) or "sparse" (voxel-segment
        kernels): the fp32 kernel family this operator uses."""
        return "bin" if self.info.atom_groups == -2 else "sparse"

    @property
    def tensor_ops(self):
        """Products running on the tcgen05 tensor cores: subset of {"dsc", "wc"}."""
        t = self.info.tensor_ops
        return tuple(n for b, n in ((1, "dsc"), (2, "wc")) if t & b)

    @property
    def handle(self):
        return self._handle

    def close(self):
        self._finalizer()

    # ---- products on device tensors -------------------------------------
    def dsc_f32(self, w, y, b=None, flags=0, skipped=None, sumsq=None, absmax=None,
                stream=None):
        out = N.SpmvOut(_p(skipped), _p(sumsq), _p(absmax))
        N.check(N.lib().life_dsc_f32(self._handle, _p(w), _p(y), _p(b), flags,
                                     ctypes.byref(out), N.stream_ptr(stream)))

    def wc_f32(self, y, w, w_ref=None, y_absmax=None, flags=0, sumsq=None, stream=None):
        out = N.SpmvOut(None, _p(sumsq), None)
        N.check(N.lib().life_wc_f32(self._handle, _p(y), _p(w), _p(w_ref), _p(y_absmax),
                                    flags, ctypes.byref(out), N.stream_ptr(stream)))

    def dsc_f64(self, w, y, flags=0, skipped=None, stream=None):
        N.check(N.lib().life_dsc_f64(self._handle, _p(w), _p(y), flags, _p(skipped),
                                     N.stream_ptr(stream)))

    def wc_f64(self, y, w, stream=None):
        N.check(N.lib().life_wc_f64(self._handle, _p(y), _p(w), N.stream_ptr(stream)))


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def operator_for(tensor, dictionary, exact=False):
    """Cached DeviceOperator for (tensor, dictionary) on the current device.

    The cache entry is keyed on the dictionary object, the fp32 layout
    selected by set_layout() and the CUDA device; a change of any of them,
    or a request for the exact layout the cached operator lacks, rebuilds
    it (the old handle is released)."""
    import torch
    phi = _phi(tensor)
    cache = phi.__dict__.setdefault("_device_cache", {})
    key = (id(dictionary), _LAYOUT[0], torch.cuda.current_device())
    entry = cache.get("op")
    if entry is not None:
        op, dic, k = entry
        if dic is dictionary and k == key and (op.exact or not exact):
            return op
        op.close()
        del cache["op"]
    op = DeviceOperator(phi, dictionary, exact=exact, fast=True)
    cache["op"] = (op, dictionary, key)
    return op


# ---- reference-shaped products (accumulate into caller buffers) ------------


def _aligned(t):
    """The fp32 kernels move vectors in 16-byte units (life_b200.h): views
    at odd offsets (e.g. ``buf[1:]``) are copied to a fresh allocation."""
    return t if t.data_ptr() % 16 == 0 else t.clone()


def _in_place_ok(torch, t, dtype):
    return (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == dtype
            and t.is_contiguous() and t.data_ptr() % 16 == 0
            and t.device.index == torch.cuda.current_device())


def _as_device(torch, x, dtype):
    if isinstance(x, torch.Tensor):
        if not x.is_cuda:
            return x.to(device="cuda", dtype=dtype).contiguous()
        return _aligned(x.to(device="cuda", dtype=dtype).contiguous())
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(
        device="cuda", dtype=dtype)


def _accumulate_into(torch, dst, add):
    """dst += add, keeping dst's own storage and dtype."""
    if isinstance(dst, torch.Tensor):
        dst.add_(add.to(device=dst.device, dtype=dst.dtype))
    else:
        dst += add.double().cpu().numpy()


def dsc_accumulate(tensor, dictionary, w, y_out, skip_zero=True, precision=None):
    """y_out += M w; returns (skipped, gpu_seconds)."""
    torch = N.require_cuda()
    precision = precision or default_precision()
    op = operator_for(tensor, dictionary, exact=(precision == "fp64"))
    d = op.dims
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    skipped = torch.zeros(1, dtype=torch.int64, device="cuda")
    flags = N.SKIP_ZERO if skip_zero else 0
    if precision == "fp64":
        wd = _as_device(torch, w, torch.float64)
        if _in_place_ok(torch, y_out, torch.float64):
            yd = y_out
        else:
            yd = _as_device(torch, y_out, torch.float64)
        start.record()
        op.dsc_f64(wd, yd, flags, skipped)
        stop.record()
        if yd is not y_out:
            if isinstance(y_out, torch.Tensor):
                y_out.copy_(yd)
            else:
                y_out[...] = yd.cpu().numpy()
    else:
        wd = _as_device(torch, w, torch.float32)
        if _in_place_ok(torch, y_out, torch.float32):
            start.record()
            op.dsc_f32(wd, y_out, None, flags | N.ACCUMULATE, skipped)
            stop.record()
        else:
            yd = torch.empty(d.signal_len, dtype=torch.float32, device="cuda")
            start.record()
            op.dsc_f32(wd, yd, None, flags, skipped)
            stop.record()
            _accumulate_into(torch, y_out, yd)
    torch.cuda.synchronize()
    return int(skipped.item()), start.elapsed_time(stop) * 1e-3


def wc_accumulate(tensor, dictionary, y, w_out, precision=None):
    """w_out += M^T y; returns gpu_seconds."""
    torch = N.require_cuda()
    precision = precision or default_precision()
    op = operator_for(tensor, dictionary, exact=(precision == "fp64"))
    d = op.dims
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if precision == "fp64":
        yd = _as_device(torch, y, torch.float64)
        if _in_place_ok(torch, w_out, torch.float64):
            wd = w_out
        else:
            wd = _as_device(torch, w_out, torch.float64)
        start.record()
        op.wc_f64(yd, wd)
        stop.record()
        if wd is not w_out:
            if isinstance(w_out, torch.Tensor):
                w_out.copy_(wd)
            else:
                w_out[...] = wd.cpu().numpy()
    else:
        yd = _as_device(torch, y, torch.float32)
        if _in_place_ok(torch, w_out, torch.float32):
            start.record()
            op.wc_f32(yd, w_out, flags=N.ACCUMULATE)
            stop.record()
        else:
            wd = torch.empty(d.n_fibers, dtype=torch.float32, device="cuda")
            start.record()
            op.wc_f32(yd, wd)
            stop.record()
            _accumulate_into(torch, w_out, wd)
    torch.cuda.synchronize()
    return start.elapsed_time(stop) * 1e-3


def autotune_layout(problem, trials=3, candidates=("sparse", "bin")):
    """Pick the fp32 kernel family for a problem by timing one DSC + one WC
    per candidate on the device (the paper's runtime selection between
    kernel variants, restructure.py:107-144 for
    the reference's CPU analogue).  Returns (best name, {name: mean seconds}).
    A candidate whose layout cannot be built for the problem (e.g. the
    tensor layout above 128 directions) is skipped."""
    torch = N.require_cuda()
    d = problem.dims
    w = torch.from_numpy(np.asarray(problem.w_true if problem.w_true is not None
                                    else np.ones(d.n_fibers))).float().cuda()
    y = torch.zeros(d.signal_len, device="cuda")
    g = torch.zeros(d.n_fibers, device="cuda")
    ymax = torch.ones(1, device="cuda")
    saved, times = _LAYOUT[0], {}
    try:
        for name in candidates:
            set_layout(name)
            op = DeviceOperator(problem.tensor, problem.dictionary)
            if name != "sparse" and op.kind == "sparse":
                continue  # no tile layout for this problem
            run = lambda: (op.dsc_f32(w, y), op.wc_f32(y, g, y_absmax=ymax))  # noqa: E731
            run()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(trials):
                run()
            e1.record()
            torch.cuda.synchronize()
            times[name] = e0.elapsed_time(e1) / 1e3 / trials
            op.close()
    finally:
        set_layout(saved)
    best = min(times, key=times.get)
    return best, times
