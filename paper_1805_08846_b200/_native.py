"""ctypes binding of the C ABI (include/clawb200.h) -> libclawb200.so.

The product path has no CPU fallback: if the library is missing, or no CUDA
device is available, every entry point raises :class:`DeviceError`.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from .errors import DeviceError

HERE = os.path.dirname(os.path.abspath(__file__))
#: CLB_LIB_VARIANT=<tag> loads libclawb200_<tag>.so (tuning experiments built
#: by `python -m paper_1805_08846_b200.build --variant <tag> -D...`)
_VARIANT = os.environ.get("CLB_LIB_VARIANT")
LIB_PATH = os.path.join(HERE, f"libclawb200_{_VARIANT}.so" if _VARIANT else "libclawb200.so")

CLB_OK = 0
CLB_EINVAL = -1
CLB_ECUDA = -2
CLB_ENOMEM = -3
CLB_EUNSUPPORTED = -4

SOLVER_IDS = {"advection": 0, "acoustics": 1, "shallow_water": 2, "vc_acoustics": 3}

#: every symbol include/clawb200.h declares
EXPORTS = (
    "clb_create", "clb_destroy", "clb_last_error", "clb_version", "clb_set_stream",
    "clb_set_segments", "clb_upload", "clb_download", "clb_upload_padded",
    "clb_download_padded", "clb_set_boundary", "clb_sweep", "clb_sweep_async", "clb_fetch",
    "clb_attempt_step", "clb_first_nonfinite", "clb_halo_layout", "clb_halo_copy", "clb_solve_pairs",
    "clb_enable_timing", "clb_timing", "clb_host_alloc", "clb_host_free", "clb_memory_info",
    "clb_selftest_arith", "clb_run_batch", "clb_frame_size", "clb_write_frame",
    "clb_sweep_segments", "clb_sweep_async_range", "clb_set_x_variant", "clb_x_variant",
    "clb_x_activity",
    "clb_register_device_solver", "clb_sweep_args_size", "clb_nccl_unique_id",
    "clb_attach_comm", "clb_halo_exchange", "clb_results_allreduce",
)

#: x-sweep kernel variants (clb_set_x_variant)
XVAR_AUTO, XVAR_MARCH, XVAR_TMA, XVAR_PAIR, XVAR_TMA_STREAM, XVAR_TMA_ADAPT = 0, 1, 2, 3, 4, 5

#: clb_run_batch statuses (include/clawb200.h)
BATCH_STOP, BATCH_MAXSTEPS, BATCH_LOGFULL, BATCH_BLOWUP, BATCH_UNSTABLE, BATCH_DTERR = range(6)


class ClbDesc(ctypes.Structure):
    _fields_ = [
        ("ndim", ctypes.c_int32),
        ("num_states", ctypes.c_int32),
        ("itemsize", ctypes.c_int32),
        ("solver_id", ctypes.c_int32),
        ("limiter_id", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("cells", ctypes.c_int64 * 3),
        ("spacing", ctypes.c_double * 3),
        ("params", ctypes.c_double * 8),
        ("bc", (ctypes.c_int32 * 2) * 3),
        ("normal_velocity", ctypes.c_int32 * 3),
    ]


class ClbBatch(ctypes.Structure):
    _fields_ = [
        ("t", ctypes.c_double), ("last_max_speed", ctypes.c_double),
        ("prev_nu", ctypes.c_double), ("nu_max", ctypes.c_double),
        ("prev_reverted", ctypes.c_int32),
        ("cur", ctypes.c_int32), ("scratch0", ctypes.c_int32), ("scratch1", ctypes.c_int32),
        ("stop", ctypes.c_double), ("cfl_target", ctypes.c_double), ("cfl_max", ctypes.c_double),
        ("dt_cap", ctypes.c_double), ("min_spacing", ctypes.c_double),
        ("max_accepted", ctypes.c_int64),
        ("n_attempts", ctypes.c_int64), ("n_accepted", ctypes.c_int64),
        ("status", ctypes.c_int32), ("fail_sweep", ctypes.c_int32),
        ("fail_dt", ctypes.c_double),
    ]


class ClbAttempt(ctypes.Structure):
    _fields_ = [
        ("t_start", ctypes.c_double), ("dt", ctypes.c_double), ("max_speed", ctypes.c_double),
        ("nu", ctypes.c_double), ("dt_retry", ctypes.c_double),
        ("accepted", ctypes.c_int32), ("landed", ctypes.c_int32),
    ]


_lib = None

_vp = ctypes.c_void_p
_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_int = ctypes.c_int
_dbl = ctypes.c_double
_sz = ctypes.c_size_t


def lib():
    """Load libclawb200.so once (raises DeviceError if it is not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (or python paper_1805_08846_b200/build.py); there is no CPU fallback"
        )
    L = ctypes.CDLL(LIB_PATH)
    sig = {
        "clb_create": (_int, [ctypes.POINTER(ClbDesc), ctypes.POINTER(_vp)]),
        "clb_destroy": (_int, [_vp]),
        "clb_last_error": (ctypes.c_char_p, [_vp]),
        "clb_version": (_int, []),
        "clb_set_stream": (_int, [_vp, _vp]),
        "clb_set_segments": (_int, [_vp, _int, _int]),
        "clb_set_x_variant": (_int, [_vp, _int]),
        "clb_register_device_solver": (_int, [_int, _int, _int, _int, _sz, _vp, _vp, _vp, _vp]),
        "clb_sweep_args_size": (_sz, []),
        "clb_nccl_unique_id": (_int, [_vp]),
        "clb_attach_comm": (_int, [_vp, _vp, _int, _int, _int, _int]),
        "clb_halo_exchange": (_int, [_vp, _int]),
        "clb_results_allreduce": (_int, [_vp]),
        "clb_x_variant": (_int, [_vp, ctypes.POINTER(_i32)]),
        "clb_x_activity": (_int, [_vp, ctypes.POINTER(ctypes.c_uint64),
                                  ctypes.POINTER(ctypes.c_uint64)]),
        "clb_upload": (_int, [_vp, _int, _vp, _sz]),
        "clb_download": (_int, [_vp, _int, _vp, _sz]),
        "clb_upload_padded": (_int, [_vp, _int, _vp, _sz]),
        "clb_download_padded": (_int, [_vp, _int, _vp, _sz]),
        "clb_set_boundary": (_int, [_vp, _int, _int, _int]),
        "clb_sweep": (_int, [_vp, _int, _dbl, _int, _int, ctypes.POINTER(_dbl), ctypes.POINTER(_i32)]),
        "clb_sweep_async": (_int, [_vp, _int, _dbl, _int, _int, _int, _int]),
        "clb_fetch": (_int, [_vp, _int, ctypes.POINTER(_dbl), ctypes.POINTER(_i32)]),
        "clb_attempt_step": (_int, [_vp, _dbl, _int, _int, _int, ctypes.POINTER(_dbl),
                                    ctypes.POINTER(_i32)]),
        "clb_first_nonfinite": (_int, [_vp, _int, ctypes.POINTER(_i32), ctypes.POINTER(_i32),
                                       ctypes.POINTER(_i64)]),
        "clb_halo_layout": (_int, [_vp, _int, _int, ctypes.POINTER(_vp), ctypes.POINTER(_vp),
                                   ctypes.POINTER(_sz), ctypes.POINTER(_sz)]),
        "clb_halo_copy": (_int, [_vp, _int, _int, _int, _vp]),
        "clb_solve_pairs": (_int, [_vp, _int, _i64, _vp, _vp, _vp, _vp]),
        "clb_enable_timing": (_int, [_vp, _int]),
        "clb_timing": (_int, [_vp, ctypes.POINTER(_dbl), ctypes.POINTER(_i64)]),
        "clb_host_alloc": (_vp, [_sz]),
        "clb_host_free": (None, [_vp]),
        "clb_memory_info": (_int, [_vp, ctypes.POINTER(_sz), ctypes.POINTER(_i64)]),
        "clb_selftest_arith": (_int, [_int, _i64, _vp, _vp, ctypes.POINTER(_i64)]),
        "clb_run_batch": (_int, [_vp, ctypes.POINTER(ClbBatch), ctypes.POINTER(ClbAttempt), _i64]),
        "clb_frame_size": (_int, [_vp, ctypes.POINTER(_sz)]),
        "clb_sweep_segments": (_int, [_vp, _int, ctypes.POINTER(_i32), ctypes.POINTER(_i32)]),
        "clb_sweep_async_range": (_int, [_vp, _int, _dbl, _int, _int, _int, _int, _int, _int]),
        "clb_write_frame": (_int, [_vp, _int, _dbl, ctypes.c_uint64, _vp, _sz]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _check(code: int, handle=None):
    if code == CLB_OK:
        return
    msg = lib().clb_last_error(handle)
    msg = msg.decode() if msg else "unknown error"
    if code in (CLB_EINVAL, CLB_EUNSUPPORTED):
        raise ValueError(msg)
    raise DeviceError(msg)


class DeviceGrid:
    """Owning wrapper of one clb handle: three device buffers of one grid."""

    def __init__(self, *, ndim, cells, spacing, num_states, dtype, solver_id, limiter_id,
                 params, bc, normal_velocity, device=0):
        d = ClbDesc()
        d.ndim = ndim
        d.num_states = num_states
        self.dtype = np.dtype(dtype)
        d.itemsize = self.dtype.itemsize
        d.solver_id = solver_id
        d.limiter_id = limiter_id
        d.device = device
        for ax in range(3):
            d.cells[ax] = int(cells[ax]) if ax < ndim else 1
            d.spacing[ax] = float(spacing[ax]) if ax < ndim else 1.0
            d.normal_velocity[ax] = -1
            d.bc[ax][0] = 0
            d.bc[ax][1] = 0
        for ax in range(ndim):
            d.bc[ax][0], d.bc[ax][1] = bc[ax]
            nv = normal_velocity[ax]
            d.normal_velocity[ax] = -1 if nv is None else int(nv)
        pv = np.asarray(params, dtype=self.dtype)
        for i in range(min(8, pv.shape[0])):
            d.params[i] = float(pv[i])  # T-packed value widened exactly
        self.desc = d
        self.ndim = ndim
        self.cells = tuple(int(c) for c in cells[:ndim])
        self.num_states = num_states
        h = _vp()
        L = lib()
        code = L.clb_create(ctypes.byref(d), ctypes.byref(h))
        _check(code, None)
        self.handle = h

    # -- lifecycle ----------------------------------------------------------
    def close(self):
        if getattr(self, "handle", None):
            lib().clb_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- transfers ------------------------------------------------------------
    @property
    def interior_shape(self):
        return (self.num_states,) + tuple(reversed(self.cells))

    @property
    def padded_shape(self):
        return (self.num_states,) + tuple(c + 4 for c in reversed(self.cells))

    def upload(self, buf: int, interior: np.ndarray):
        a = np.ascontiguousarray(interior, dtype=self.dtype)
        if a.shape != self.interior_shape:
            raise ValueError(f"interior shape {a.shape} != {self.interior_shape}")
        _check(lib().clb_upload(self.handle, buf, a.ctypes.data, a.nbytes), self.handle)

    def download(self, buf: int, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.interior_shape, dtype=self.dtype)
        assert out.flags.c_contiguous and out.dtype == self.dtype
        _check(lib().clb_download(self.handle, buf, out.ctypes.data, out.nbytes), self.handle)
        return out

    def upload_padded(self, buf: int, padded: np.ndarray):
        a = np.ascontiguousarray(padded, dtype=self.dtype)
        if a.shape != self.padded_shape:
            raise ValueError(f"padded shape {a.shape} != {self.padded_shape}")
        _check(lib().clb_upload_padded(self.handle, buf, a.ctypes.data, a.nbytes), self.handle)

    def download_padded(self, buf: int, out: np.ndarray | None = None) -> np.ndarray:
        if out is None:
            out = np.empty(self.padded_shape, dtype=self.dtype)
        _check(lib().clb_download_padded(self.handle, buf, out.ctypes.data, out.nbytes),
               self.handle)
        return out

    # -- compute --------------------------------------------------------------
    def set_boundary(self, axis: int, lo: int, hi: int):
        _check(lib().clb_set_boundary(self.handle, axis, lo, hi), self.handle)

    def set_segments(self, axis: int, seg_len: int):
        _check(lib().clb_set_segments(self.handle, axis, seg_len), self.handle)

    def set_x_variant(self, variant: int):
        """x-sweep kernel: XVAR_AUTO, XVAR_MARCH (warp-march), XVAR_TMA, XVAR_PAIR,
        XVAR_TMA_STREAM or XVAR_TMA_ADAPT (the last two: fp64 2-D shallow water)."""
        _check(lib().clb_set_x_variant(self.handle, int(variant)), self.handle)

    def x_variant(self) -> int:
        """The kernel variant the next x sweep launches (XVAR_MARCH .. XVAR_TMA_ADAPT)."""
        v = _i32(0)
        _check(lib().clb_x_variant(self.handle, ctypes.byref(v)), self.handle)
        return int(v.value)

    def x_activity(self) -> tuple[int, int]:
        """(computed strided warp groups since the last x sweep, threshold):
        the geometry pair runs its streaming twin next while computed <
        threshold (XVAR_TMA_ADAPT handles only)."""
        c, t = ctypes.c_uint64(0), ctypes.c_uint64(0)
        _check(lib().clb_x_activity(self.handle, ctypes.byref(c), ctypes.byref(t)), self.handle)
        return int(c.value), int(t.value)

    def attach_comm(self, uid: bytes, nranks: int, rank: int, lo_nbr, hi_nbr):
        """Device-resident slab exchange over NCCL (clb_attach_comm)."""
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        _check(lib().clb_attach_comm(self.handle, buf, int(nranks), int(rank),
                                     -1 if lo_nbr is None else int(lo_nbr),
                                     -1 if hi_nbr is None else int(hi_nbr)), self.handle)

    def halo_exchange(self, buf: int):
        _check(lib().clb_halo_exchange(self.handle, int(buf)), self.handle)

    def results_allreduce(self):
        _check(lib().clb_results_allreduce(self.handle), self.handle)

    def set_stream(self, stream_ptr: int | None):
        _check(lib().clb_set_stream(self.handle, stream_ptr or None), self.handle)

    def sweep(self, axis: int, dt: float, src: int, dst: int):
        s = _dbl(0.0)
        nf = _i32(0)
        _check(lib().clb_sweep(self.handle, axis, float(dt), src, dst, ctypes.byref(s),
                               ctypes.byref(nf)), self.handle)
        return s.value, bool(nf.value)

    def sweep_async(self, axis: int, dt: float, src: int, dst: int, slot: int,
                    literal: bool = False):
        _check(lib().clb_sweep_async(self.handle, axis, float(dt), src, dst, slot,
                                     1 if literal else 0), self.handle)

    def segments(self, axis: int):
        """(nseg, seg_len) of the sweep along `axis`."""
        n, L = _i32(0), _i32(0)
        _check(lib().clb_sweep_segments(self.handle, axis, ctypes.byref(n), ctypes.byref(L)),
               self.handle)
        return int(n.value), int(L.value)

    def sweep_async_range(self, axis: int, dt: float, src: int, dst: int, slot: int,
                          seg_begin: int, seg_end: int, literal: bool = False):
        _check(lib().clb_sweep_async_range(self.handle, axis, float(dt), src, dst, slot,
                                           1 if literal else 0, seg_begin, seg_end), self.handle)

    def fetch(self, nslots: int):
        s = (_dbl * 4)()
        nf = (_i32 * 4)()
        _check(lib().clb_fetch(self.handle, nslots, s, nf), self.handle)
        return [s[i] for i in range(nslots)], [bool(nf[i]) for i in range(nslots)]

    def attempt_step(self, dt: float, src: int, s0: int, s1: int):
        s = (_dbl * 4)()
        nf = (_i32 * 4)()
        _check(lib().clb_attempt_step(self.handle, float(dt), src, s0, s1, s, nf), self.handle)
        return [s[i] for i in range(self.ndim)], [bool(nf[i]) for i in range(self.ndim)]

    def first_nonfinite(self, buf: int):
        found = _i32(0)
        state = _i32(0)
        cell = (_i64 * 3)()
        _check(lib().clb_first_nonfinite(self.handle, buf, ctypes.byref(found),
                                         ctypes.byref(state), cell), self.handle)
        if not found.value:
            return None
        return int(state.value), tuple(int(cell[i]) for i in range(self.ndim))

    def halo_layout(self, buf: int, side: int):
        sp = _vp()
        rp = _vp()
        bb = _sz()
        ss = _sz()
        _check(lib().clb_halo_layout(self.handle, buf, side, ctypes.byref(sp), ctypes.byref(rp),
                                     ctypes.byref(bb), ctypes.byref(ss)), self.handle)
        return sp.value, rp.value, bb.value, ss.value

    def halo_read(self, buf: int, side: int) -> np.ndarray:
        """The 2 owned boundary rows/planes of `side`, every state, as bytes."""
        _, _, nbytes, _ = self.halo_layout(buf, side)
        out = np.empty((self.num_states, nbytes), dtype=np.uint8)
        _check(lib().clb_halo_copy(self.handle, buf, side, 1, out.ctypes.data), self.handle)
        return out

    def halo_write(self, buf: int, side: int, data: np.ndarray) -> None:
        """Write neighbour rows into the ghost layers of `side`."""
        a = np.ascontiguousarray(data, dtype=np.uint8)
        _check(lib().clb_halo_copy(self.handle, buf, side, 0, a.ctypes.data), self.handle)

    def solve_pairs(self, axis: int, ql: np.ndarray, qr: np.ndarray, num_waves: int):
        ql = np.ascontiguousarray(ql, dtype=self.dtype)
        qr = np.ascontiguousarray(qr, dtype=self.dtype)
        n = ql.shape[0]
        W = np.empty((n, num_waves, self.num_states), dtype=self.dtype)
        s = np.empty((n, num_waves), dtype=self.dtype)
        _check(lib().clb_solve_pairs(self.handle, axis, n, ql.ctypes.data, qr.ctypes.data,
                                     W.ctypes.data, s.ctypes.data), self.handle)
        return W, s

    def run_batch(self, batch: "ClbBatch", log_cap: int = 4096):
        """Device-resident attempt loop (clb_run_batch): updates `batch` in
        place and returns the logged attempts."""
        log = (ClbAttempt * log_cap)()
        _check(lib().clb_run_batch(self.handle, ctypes.byref(batch), log, log_cap), self.handle)
        return [log[i] for i in range(batch.n_attempts)]

    def frame_size(self) -> int:
        n = _sz()
        _check(lib().clb_frame_size(self.handle, ctypes.byref(n)), self.handle)
        return n.value

    def write_frame(self, buf: int, time: float, step: int, out) -> None:
        """CLAWFRM1 frame of buffer `buf` into the writable buffer `out`
        (e.g. a PinnedBuffer's array) of exactly frame_size() bytes."""
        mv = memoryview(out).cast("B")
        addr = ctypes.addressof(ctypes.c_char.from_buffer(mv))
        _check(lib().clb_write_frame(self.handle, buf, float(time), int(step), addr, mv.nbytes),
               self.handle)

    def enable_timing(self, on: bool = True):
        _check(lib().clb_enable_timing(self.handle, 1 if on else 0), self.handle)

    def timing(self):
        ms = (_dbl * 3)()
        cnt = (_i64 * 3)()
        _check(lib().clb_timing(self.handle, ms, cnt), self.handle)
        return [ms[i] for i in range(3)], [cnt[i] for i in range(3)]

    def memory_info(self):
        b = _sz()
        p = _i64()
        _check(lib().clb_memory_info(self.handle, ctypes.byref(b), ctypes.byref(p)), self.handle)
        return b.value, p.value


def nccl_unique_id() -> bytes:
    """A fresh 128-byte ncclUniqueId (clb_nccl_unique_id)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().clb_nccl_unique_id(buf))
    return buf.raw


def selftest_arith(a, b, device: int = 0):
    """Branch-free div/sqrt of the sweep kernels vs div.rn/sqrt.rn on the
    device: (div mismatches, sqrt mismatches, div fallbacks, sqrt fallbacks)
    for fp64, the same four for fp32 (low words of a, b as floats), then
    (mismatches, fallbacks) of the limiter-ratio division and of the Roe
    division (b in [2^-485, 2^513])."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError("a and b must have the same shape")
    out = (_i64 * 12)()
    _check(lib().clb_selftest_arith(device, a.size, a.ctypes.data, b.ctypes.data, out))
    return tuple(int(out[i]) for i in range(12))


class PinnedBuffer:
    """Page-locked host array from clb_host_alloc (for end-to-end copies)."""

    def __init__(self, shape, dtype):
        dtype = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * dtype.itemsize
        self.ptr = lib().clb_host_alloc(max(nbytes, 1))
        if not self.ptr:
            raise DeviceError("pinned host allocation failed")
        buf = (ctypes.c_char * max(nbytes, 1)).from_address(self.ptr)
        self.array = np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape))).reshape(shape)

    def free(self):
        if self.ptr:
            lib().clb_host_free(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass
