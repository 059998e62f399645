"""Plan: one stencil problem resident on one GPU, driven through the C ABI.

A plan owns two device buffers (ping-pong) in a private pitched layout,
chooses the kernel (fused temporal-blocking kernel for the stencil class, or
the generic one-step kernel) and its fusion depth k.  Host grids use the
compact halo-inclusive box convention of include/sb200.h.
"""

from __future__ import annotations

import ctypes
import threading
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from . import _abi
from .core import GridError, SpecError, canonical, validate

_DTYPES = {"f64": (_abi.SB_F64, np.float64), "f32": (_abi.SB_F32, np.float32)}
_ARITH = {"exact": _abi.SB_ARITH_EXACT, "fma": _abi.SB_ARITH_FMA}
_KERNEL = {"auto": _abi.SB_KERNEL_AUTO, "generic": _abi.SB_KERNEL_GENERIC,
           "fused": _abi.SB_KERNEL_FUSED}


@dataclass
class Timing:
    device_ms: float
    kernel_ms: float
    launches: int
    point_updates: int
    k_used: int
    kernel_name: str


def host_shape(d: int, r: int, dims, ghost=(0, 0)) -> tuple[int, ...]:
    """Shape of the compact host box for interior ``dims`` (slowest first)."""
    dims = tuple(int(n) for n in dims)
    if len(dims) != d:
        raise GridError(f"need {d} extents, got {len(dims)}")
    lo = ghost[0] if ghost[0] else r
    hi = ghost[1] if ghost[1] else r
    return (dims[0] + lo + hi,) + tuple(n + 2 * r for n in dims[1:])


class Plan:
    """A device-resident sweep of ``spec`` over interior ``dims``.

    ``dtype`` 'f64' or 'f32'; ``arith`` 'exact' (bit-identical to the
    reference oracle) or 'fma'; ``k`` fused steps per launch (0 = auto);
    ``kernel`` 'auto' | 'generic' | 'fused'; ``ghost`` = (lo, hi) ghost depths
    of slab sides (0 = physical Dirichlet halo).
    """

    def __init__(self, spec, dims, *, dtype="f64", arith="fma", k=0, kernel="auto",
                 device=0, ghost=(0, 0)):
        validate(spec)
        if dtype not in _DTYPES:
            raise ValueError(f"dtype must be one of {list(_DTYPES)}")
        if arith not in _ARITH:
            raise ValueError(f"arith must be one of {list(_ARITH)}")
        if kernel not in _KERNEL:
            raise ValueError(f"kernel must be one of {list(_KERNEL)}")
        self.spec = spec
        self.d, self.r = spec.d, spec.r
        self.dims = tuple(int(n) for n in dims)
        if len(self.dims) != self.d:
            raise GridError(f"{getattr(spec, 'name', 'spec')} needs {self.d} extents, "
                            f"got {len(self.dims)}")
        self.dtype_name = dtype
        self.np_dtype = _DTYPES[dtype][1]
        self.ghost = (int(ghost[0]), int(ghost[1]))
        self.shape = host_shape(self.d, self.r, self.dims, self.ghost)
        offs, ws = canonical(spec)
        self._offs = (ctypes.c_int32 * (len(offs) * self.d))(*[c for o in offs for c in o])
        self._ws = (ctypes.c_double * len(ws))(*ws)
        prob = _abi.SbProblem()
        prob.d, prob.r = self.d, self.r
        prob.shape = _abi.SB_STAR if spec.shape == "star" else _abi.SB_BOX
        prob.nw = len(ws)
        prob.offsets = ctypes.cast(self._offs, ctypes.POINTER(ctypes.c_int32))
        prob.weights = ctypes.cast(self._ws, ctypes.POINTER(ctypes.c_double))
        for a in range(3):
            prob.dims[a] = self.dims[a] if a < self.d else 1
        prob.dtype = _DTYPES[dtype][0]
        prob.arith = _ARITH[arith]
        prob.k = int(k)
        prob.kernel = _KERNEL[kernel]
        prob.device = int(device)
        prob.ghost_lo, prob.ghost_hi = self.ghost
        self._lib = _abi.load()
        handle = ctypes.c_void_p()
        _abi.check(self._lib.sb_plan_create(ctypes.byref(handle), ctypes.byref(prob)))
        self._h = handle
        kk = ctypes.c_int32()
        _abi.check(self._lib.sb_plan_k(self._h, ctypes.byref(kk)))
        self.k = int(kk.value)

    # -- lifecycle
    def close(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.sb_plan_destroy(h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- data movement
    def _check_box(self, box: np.ndarray):
        if box.shape != self.shape:
            raise GridError(f"host box shape {box.shape}, expected {self.shape}")
        if box.dtype != self.np_dtype:
            raise GridError(f"host box dtype {box.dtype}, expected {np.dtype(self.np_dtype)}")
        if not box.flags.c_contiguous:
            raise GridError("host box must be C-contiguous")

    def upload(self, box: np.ndarray) -> None:
        self._check_box(box)
        _abi.check(self._lib.sb_upload(self._h, box.ctypes.data, box.nbytes))

    def download(self, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.shape, dtype=self.np_dtype)
        self._check_box(out)
        _abi.check(self._lib.sb_download(self._h, out.ctypes.data, out.nbytes))
        return out

    def upload_pitched(self, first_row: int, pitch_bytes: int) -> None:
        """Upload a host box given as uniformly pitched rows (``first_row``: address
        of row 0; see ``sb_upload_pitched``) -- a NATURAL GridBuffer in place."""
        _abi.check(self._lib.sb_upload_pitched(self._h, ctypes.c_void_p(first_row), int(pitch_bytes)))

    def download_pitched(self, first_row: int, pitch_bytes: int) -> None:
        """Write the current box back into pitched host rows (``sb_download_pitched``)."""
        _abi.check(self._lib.sb_download_pitched(self._h, ctypes.c_void_p(first_row), int(pitch_bytes)))

    def sweep_host(self, box: np.ndarray, steps: int, out: np.ndarray | None = None) -> np.ndarray:
        """``steps`` steps from the host box ``box`` into ``out`` (default: a new array),
        transfers overlapped with the sweep where the plan allows it (``sb_sweep_host``)."""
        self._check_box(box)
        if out is None:
            out = np.empty(self.shape, dtype=self.np_dtype)
        self._check_box(out)
        _abi.check(self._lib.sb_sweep_host(self._h, box.ctypes.data, 0, out.ctypes.data, 0, int(steps)))
        return out

    def sweep_host_pitched(self, first_in: int, in_pitch: int, first_out: int, out_pitch: int, steps: int) -> None:
        """:meth:`sweep_host` on pitched host rows (addresses of row 0; may coincide)."""
        _abi.check(self._lib.sb_sweep_host(self._h, ctypes.c_void_p(first_in), int(in_pitch),
                                           ctypes.c_void_p(first_out), int(out_pitch), int(steps)))

    def upload_async(self, box: np.ndarray) -> None:
        """Stream-ordered upload: returns once enqueued; `box` (ideally pinned
        memory) must stay alive and unmodified until :meth:`synchronize`."""
        self._check_box(box)
        _abi.check(self._lib.sb_upload_async(self._h, box.ctypes.data, box.nbytes))

    def download_async(self, out: np.ndarray) -> np.ndarray:
        """Stream-ordered download into `out`; valid after :meth:`synchronize`."""
        self._check_box(out)
        _abi.check(self._lib.sb_download_async(self._h, out.ctypes.data, out.nbytes))
        return out

    def upload_storage(self, grid) -> None:
        """Upload a reference-storage grid (``GridBuffer.data`` in NATURAL,
        BLOCK_TRANSPOSE or DLT layout, any vl) and un-permute it on the device."""
        data, st = self._storage(grid)
        _abi.check(self._lib.sb_upload_storage(self._h, data.ctypes.data, data.nbytes, ctypes.byref(st)))

    def download_storage(self, grid, out: np.ndarray | None = None) -> np.ndarray:
        """The current grid, permuted on the device into ``grid``'s layout, as a
        full storage array (default: a new array shaped like ``grid.data``);
        non-interior cells keep the values of the last :meth:`upload_storage`."""
        data, st = self._storage(grid)
        if out is None:
            out = np.empty_like(data)
        if out.shape != data.shape or out.dtype != data.dtype or not out.flags.c_contiguous:
            raise GridError("storage output must match the grid's storage array")
        _abi.check(self._lib.sb_download_storage(self._h, out.ctypes.data, out.nbytes, ctypes.byref(st)))
        return out

    def _storage(self, grid):
        data = np.ascontiguousarray(grid.data, dtype=self.np_dtype)
        return data, storage_descriptor(grid)

    def synchronize(self) -> None:
        _abi.check(self._lib.sb_synchronize(self._h))

    # -- compute
    def run(self, steps: int) -> Timing:
        t = _abi.SbTiming()
        _abi.check(self._lib.sb_run(self._h, int(steps), ctypes.byref(t)))
        return Timing(t.device_ms, t.kernel_ms, t.launches, t.point_updates, t.k_used,
                      t.kernel_name.decode())

    def step_box(self, ranges) -> None:
        """One step over the interior sub-box ``ranges`` = [(lo, hi)] per axis
        (the reference's ``scalar_step(..., ranges=...)``); only that box of
        the new current buffer is valid."""
        if len(ranges) != self.d:
            raise _abi.GridError(f"ranges has {len(ranges)} axes, grid has {self.d}")
        lo = (ctypes.c_int64 * 3)(*[int(r[0]) for r in ranges], *([0] * (3 - self.d)))
        hi = (ctypes.c_int64 * 3)(*[int(r[1]) for r in ranges], *([0] * (3 - self.d)))
        _abi.check(self._lib.sb_step_box(self._h, lo, hi))

    def launch(self, steps: int) -> None:
        _abi.check(self._lib.sb_launch(self._h, int(steps)))

    def launch_repeat(self, steps: int, repeats: int, per_sweep_events: bool = False) -> None:
        """``repeats`` back-to-back sweeps of ``steps`` steps enqueued natively
        (see :meth:`repeat_times`).  Asynchronous."""
        _abi.check(self._lib.sb_launch_repeat(self._h, int(steps), int(repeats), 1 if per_sweep_events else 0))

    def repeat_times(self) -> list[float]:
        """Durations (ms) of the last :meth:`launch_repeat` (waits for it): one
        per sweep with per-sweep events, else one for the whole run."""
        buf = (ctypes.c_float * 65536)()
        n = self._lib.sb_repeat_times(self._h, buf, 65536)
        if n < 0:
            _abi.check(n)
        return [float(buf[i]) for i in range(min(n, 65536))]

    def launch_range(self, steps: int, lo: int, hi: int, finish: bool) -> None:
        """One fused launch writing only slowest-axis interior positions [lo, hi);
        ``finish`` completes the step (swaps buffers).  Asynchronous."""
        _abi.check(self._lib.sb_launch_range(self._h, int(steps), int(lo), int(hi), 1 if finish else 0))

    def set_stream(self, stream_ptr: int | None) -> None:
        _abi.check(self._lib.sb_set_stream(self._h, ctypes.c_void_p(stream_ptr or 0)))

    def kernel_count(self) -> int:
        """Kernels this plan has launched so far (main, boundary and generic)."""
        c = ctypes.c_int64()
        _abi.check(self._lib.sb_kernel_count(self._h, ctypes.byref(c)))
        return int(c.value)

    def device_view(self, which: int = 0):
        """(base pointer, origin element offset, element strides) of a buffer."""
        base = ctypes.c_void_p()
        origin = ctypes.c_int64()
        strides = (ctypes.c_int64 * 3)()
        _abi.check(self._lib.sb_device_view(self._h, which, ctypes.byref(base),
                                            ctypes.byref(origin), strides))
        return int(base.value or 0), int(origin.value), tuple(strides[: self.d])


_LAYOUT_CODES = {"natural": _abi.SB_LAYOUT_NATURAL, "block_transpose": _abi.SB_LAYOUT_BLOCK_TRANSPOSE,
                 "dlt": _abi.SB_LAYOUT_DLT}


def storage_descriptor(grid) -> _abi.SbStorage:
    """C-ABI ``sb_storage`` of a (reference or sb200) GridBuffer."""
    from .grid import layout_value
    st = _abi.SbStorage()
    st.layout = _LAYOUT_CODES[layout_value(grid)]
    st.vl = int(getattr(grid, "vl", 4))
    st.unit_n = int(grid.unit_n)
    st.unit_np = int(grid.unit_np)
    st.halo_unit = int(grid.halo_unit)
    return st


def _problem(spec, dims, dtype, arith, k, kernel, device, ghost=(0, 0)):
    """(sb_problem, keep-alive arrays) for a spec over interior ``dims``."""
    offs, ws = canonical(spec)
    d = spec.d
    c_offs = (ctypes.c_int32 * (len(offs) * d))(*[c for o in offs for c in o])
    c_ws = (ctypes.c_double * len(ws))(*ws)
    prob = _abi.SbProblem()
    prob.d, prob.r = d, spec.r
    prob.shape = _abi.SB_STAR if spec.shape == "star" else _abi.SB_BOX
    prob.nw = len(ws)
    prob.offsets = ctypes.cast(c_offs, ctypes.POINTER(ctypes.c_int32))
    prob.weights = ctypes.cast(c_ws, ctypes.POINTER(ctypes.c_double))
    for a in range(3):
        prob.dims[a] = int(dims[a]) if a < d else 1
    prob.dtype = _DTYPES[dtype][0]
    prob.arith = _ARITH[arith]
    prob.k = int(k)
    prob.kernel = _KERNEL[kernel]
    prob.device = int(device)
    prob.ghost_lo, prob.ghost_hi = ghost
    return prob, (c_offs, c_ws)


class MultiPlan:
    """One grid over several GPUs of this node (include/sb200.h sb_multi_*).

    The interior is split along the slowest axis into ``ngpu`` slabs, one
    slab plan per device of ``devices`` (default 0 .. ngpu-1; repeating a
    device emulates the decomposition on one GPU).  Ghost planes (depth r*k)
    are peer-copied between neighbours after every launch of k fused steps,
    overlapped with the slab interiors; the result is bit-identical to one
    device.  Host boxes are the GLOBAL compact halo-inclusive box.
    """

    def __init__(self, spec, dims, *, ngpu, devices=None, dtype="f64", arith="fma", k=0, kernel="auto"):
        validate(spec)
        if dtype not in _DTYPES or arith not in _ARITH or kernel not in _KERNEL:
            raise ValueError("bad dtype / arith / kernel")
        self.spec = spec
        self.d, self.r = spec.d, spec.r
        self.dims = tuple(int(n) for n in dims)
        if len(self.dims) != self.d:
            raise GridError(f"{getattr(spec, 'name', 'spec')} needs {self.d} extents, got {len(self.dims)}")
        self.np_dtype = _DTYPES[dtype][1]
        self.shape = host_shape(self.d, self.r, self.dims)
        prob, self._keep = _problem(spec, self.dims, dtype, arith, k, kernel, 0)
        devs = list(range(ngpu)) if devices is None else [int(x) for x in devices]
        if len(devs) != ngpu:
            raise ValueError(f"devices has {len(devs)} entries, ngpu is {ngpu}")
        c_devs = (ctypes.c_int32 * ngpu)(*devs)
        self._lib = _abi.load()
        h = ctypes.c_void_p()
        _abi.check(self._lib.sb_multi_create(ctypes.byref(h), ctypes.byref(prob), int(ngpu), c_devs))
        self._h = h
        g, kk = ctypes.c_int32(), ctypes.c_int32()
        _abi.check(self._lib.sb_multi_info(self._h, ctypes.byref(g), ctypes.byref(kk)))
        self.ngpu, self.k = int(g.value), int(kk.value)

    def slabs(self):
        """[(start, end, device)] of every slab (global interior planes)."""
        out = []
        for i in range(self.ngpu):
            a, b, dv = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
            _abi.check(self._lib.sb_multi_slab(self._h, i, ctypes.byref(a), ctypes.byref(b), ctypes.byref(dv)))
            out.append((int(a.value), int(b.value), int(dv.value)))
        return out

    def close(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.sb_multi_destroy(h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check_box(self, box):
        if box.shape != self.shape or box.dtype != self.np_dtype or not box.flags.c_contiguous:
            raise GridError(f"host box must be C-contiguous {np.dtype(self.np_dtype)} of shape {self.shape}")

    def upload(self, box: np.ndarray) -> None:
        self._check_box(box)
        _abi.check(self._lib.sb_multi_upload(self._h, box.ctypes.data, box.nbytes))

    def download(self, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.shape, dtype=self.np_dtype)
        self._check_box(out)
        _abi.check(self._lib.sb_multi_download(self._h, out.ctypes.data, out.nbytes))
        return out

    def run(self, steps: int) -> Timing:
        t = _abi.SbTiming()
        _abi.check(self._lib.sb_multi_run(self._h, int(steps), ctypes.byref(t)))
        return Timing(t.device_ms, t.kernel_ms, t.launches, t.point_updates, t.k_used, t.kernel_name.decode())


_CACHE = threading.local()
PLAN_CACHE_SIZE = 8           # plans kept per host thread (device memory stays allocated)
PLAN_CACHE_BYTES = 24 << 30   # ... and their device memory, least recently used evicted first


def _plan_bytes(spec, dims, dtype) -> int:
    """Device memory of a plan, roughly: two pitched halo-inclusive buffers."""
    n = 1
    for a, d in enumerate(dims):
        n *= int(d) + 2 * spec.r + (32 if a == len(dims) - 1 else 0)
    return 2 * n * (4 if dtype == "f32" else 8)


def cached_plan(spec, dims, *, dtype="f64", arith="fma", k=0, kernel="auto", device=0) -> "Plan":
    """A Plan for this problem from the calling thread's LRU cache.

    Repeated single steps / tiles / sweeps of one geometry (the reference's
    ``_execute`` loop and tile runner call a step function once per time step
    and tile) reuse the device buffers, streams and schedules instead of
    allocating them per call.  Plans are per host thread (a plan serves one
    host thread at a time, include/sb200.h), so concurrent callers -- the
    reference's ThreadPoolExecutor tile workers -- never share one.
    """
    offs, ws = canonical(spec)
    key = (spec.d, spec.r, spec.shape, tuple(offs), tuple(ws), tuple(int(n) for n in dims),
           dtype, arith, int(k), kernel, int(device))
    cache = getattr(_CACHE, "plans", None)
    if cache is None:
        cache = _CACHE.plans = OrderedDict()
    p = cache.get(key)
    if p is not None and p._h:
        cache.move_to_end(key)
        return p
    p = Plan(spec, dims, dtype=dtype, arith=arith, k=k, kernel=kernel, device=device)
    p._cache_bytes = _plan_bytes(spec, dims, dtype)
    cache[key] = p
    while len(cache) > 1 and (len(cache) > PLAN_CACHE_SIZE or
                              sum(q._cache_bytes for q in cache.values()) > PLAN_CACHE_BYTES):
        _, old = cache.popitem(last=False)
        old.close()
    return p


def clear_plan_cache() -> None:
    """Release the calling thread's cached plans (their device memory)."""
    cache = getattr(_CACHE, "plans", None)
    while cache:
        _, p = cache.popitem()
        p.close()


def sweep(spec, box: np.ndarray, steps: int, *, arith="fma", k=0, kernel="auto",
          device=0, dtype=None, ngpu=1, devices=None) -> np.ndarray:
    """``steps`` Jacobi steps of ``spec`` over a compact halo-inclusive ``box``.

    Returns a new box (halo preserved).  The grid-in/grid-out entry point of
    the drop-in (stencil shape and coefficients, input grid, timestep count).
    ``ngpu`` > 1 splits the grid into slabs over that many devices of this
    node (``devices``: their ordinals, default 0 .. ngpu-1) -- see MultiPlan.
    """
    validate(spec)
    box = np.asarray(box)
    if dtype is None:
        dtype = "f32" if box.dtype == np.float32 else "f64"
    np_dtype = _DTYPES[dtype][1]
    if box.ndim != spec.d:
        raise GridError(f"box has {box.ndim} axes, spec needs {spec.d}")
    dims = tuple(s - 2 * spec.r for s in box.shape)
    if any(n <= 0 for n in dims):
        raise GridError(f"box shape {box.shape} too small for order {spec.r}")
    if ngpu > 1 or devices is not None:
        n = ngpu if devices is None else len(devices)
        with MultiPlan(spec, dims, ngpu=n, devices=devices, dtype=dtype, arith=arith, k=k, kernel=kernel) as p:
            p.upload(np.ascontiguousarray(box, dtype=np_dtype))
            p.run(steps)
            return p.download()
    if _plan_bytes(spec, dims, dtype) <= PLAN_CACHE_BYTES // 2:
        # the calling thread's cached plan: creating and freeing the two grid buffers costs
        # 10-550 ms around a 100 ms sweep (C5); clear_plan_cache() releases the memory
        p = cached_plan(spec, dims, dtype=dtype, arith=arith, k=k, kernel=kernel, device=device)
        return p.sweep_host(np.ascontiguousarray(box, dtype=np_dtype), steps)
    with Plan(spec, dims, dtype=dtype, arith=arith, k=k, kernel=kernel, device=device) as p:
        return p.sweep_host(np.ascontiguousarray(box, dtype=np_dtype), steps)


__all__ = ["Plan", "MultiPlan", "Timing", "sweep", "cached_plan", "clear_plan_cache", "host_shape", "storage_descriptor", "SpecError", "GridError"]
