"""ctypes binding of include/sdeb200.h (libsdeb200.so, built in-tree).

There is deliberately no fallback: if the library is missing, or no CUDA
device is visible, every device entry point raises.  ctypes releases the GIL
for the duration of each call (the reference's worker pool, engine.py:265-274,
becomes per-device host threads inside the library).
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SDEB200_LIB", os.path.join(_HERE, "libsdeb200.so"))

SDB_OK, SDB_ERR_CONFIG, SDB_ERR_UNSUPPORTED, SDB_ERR_CUDA, SDB_ERR_ARGUMENT = range(5)
SDB_MODEL_KURAMOTO = 1
SDB_MODEL_EXPRESSION = 2
SOLVER_IDS = {"em": 0, "euler": 1, "rk4": 2}
STREAM_IDS = {"philox": 0, "sfc64": 1, "xoshiro256pp": 2}
COUPLING_IDS = {"meanfield": 0, "pairwise": 1}

_c_double_p = ctypes.POINTER(ctypes.c_double)
_c_u32_p = ctypes.POINTER(ctypes.c_uint32)
_c_u64_p = ctypes.POINTER(ctypes.c_uint64)
_c_i64_p = ctypes.POINTER(ctypes.c_int64)


class SdbDesc(ctypes.Structure):
    _fields_ = [
        ("model", ctypes.c_int32), ("nequat", ctypes.c_int32), ("nparams", ctypes.c_int32),
        ("nnoise", ctypes.c_int32), ("solver", ctypes.c_int32), ("stream", ctypes.c_int32),
        ("coupling", ctypes.c_int32), ("lanes", ctypes.c_int32), ("seed", ctypes.c_uint64),
        ("dt", ctypes.c_double), ("ksteps", ctypes.c_int64), ("chunks", ctypes.c_int64),
        ("orbits", ctypes.c_int64), ("orbit_offset", ctypes.c_int64),
    ]


# name -> (restype, argtypes); mirrors include/sdeb200.h one to one
ABI_VERSION = 2  # include/sdeb200.h SDB_ABI_VERSION

SIGNATURES = {
    "sdb_abi_version": (ctypes.c_int, []),
    "sdb_device_count": (ctypes.c_int, []),
    "sdb_open": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int), ctypes.c_int,
                                ctypes.POINTER(ctypes.c_void_p)]),
    "sdb_close": (None, [ctypes.c_void_p]),
    "sdb_last_error": (ctypes.c_char_p, [ctypes.c_void_p]),
    "sdb_run": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(SdbDesc), _c_double_p,
                               _c_double_p, _c_double_p, _c_i64_p]),
    "sdb_run_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(SdbDesc), ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.c_void_p]),
    "sdb_last_launch_count": (ctypes.c_int64, [ctypes.c_void_p]),
    "sdb_last_lanes": (ctypes.c_int32, [ctypes.c_void_p]),
    "sdb_last_lane_width": (ctypes.c_int32, [ctypes.c_void_p]),
    "sdb_last_tune_us": (ctypes.c_int64, [ctypes.c_void_p]),
    "sdb_host_alloc": (ctypes.c_int, [ctypes.c_int64, ctypes.POINTER(ctypes.c_void_p)]),
    "sdb_host_free": (None, [ctypes.c_void_p]),
    "sdb_last_layout": (None, [ctypes.c_void_p] + [ctypes.POINTER(ctypes.c_int32)] * 5),
    "sdb_philox_words": (ctypes.c_int, [ctypes.c_void_p, _c_u32_p, ctypes.c_int64, _c_u32_p]),
    "sdb_run_to_file": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(SdbDesc),
                                       _c_double_p, _c_double_p, ctypes.c_char_p, ctypes.c_int64,
                                       _c_i64_p]),
    "sdb_run_coherence": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(SdbDesc), _c_double_p,
                                         _c_double_p, _c_double_p, _c_i64_p]),
    "sdb_run_coherence_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(SdbDesc)]
                                 + [ctypes.c_void_p] * 5),
    "sdb_order_parameter": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                           _c_double_p, _c_double_p, _c_double_p]),
    "sdb_model_create": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                        ctypes.c_char_p, ctypes.c_char_p,
                                        ctypes.POINTER(ctypes.c_void_p)]),
    "sdb_model_free": (None, [ctypes.c_void_p]),
    "sdb_model_source": (ctypes.c_int64, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_char_p,
                                          ctypes.c_int64]),
    "sdb_model_build": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32]),
    "sdb_run_model": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(SdbDesc),
                                     _c_double_p, _c_double_p, _c_double_p, _c_i64_p]),
    "sdb_run_model_device": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.POINTER(SdbDesc)] + [ctypes.c_void_p] * 5),
    "sdb_model_eval": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                      ctypes.c_double, ctypes.c_int64, _c_double_p, _c_double_p,
                                      _c_double_p, _c_double_p]),
    "sdb_model_step": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32,
                                      ctypes.c_double, ctypes.c_double, ctypes.c_int64,
                                      _c_double_p, _c_double_p, _c_double_p, _c_double_p]),
    "sdb_normals": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64, _c_u32_p,
                                   ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint32,
                                   ctypes.c_int32, _c_double_p]),
    "sdb_stream_raw": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64,
                                      ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, _c_u64_p]),
    "sdb_sampling_uniforms": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, _c_u32_p,
                                             ctypes.c_int64, ctypes.c_int32, _c_double_p]),
    "sdb_sample_kuramoto": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint64,
                                           _c_u32_p, ctypes.c_int64, ctypes.c_double,
                                           ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                           ctypes.c_double, _c_double_p, _c_double_p]),
    "sdb_drift": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                 ctypes.c_int64, _c_double_p, _c_double_p, _c_double_p]),
    "sdb_fp64_peak": (ctypes.c_int, [ctypes.c_void_p, _c_double_p, _c_double_p]),
    "sdb_math_probe": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, _c_double_p,
                                      ctypes.c_int64, _c_double_p]),
    "sdb_step": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, ctypes.c_double,
                                _c_double_p, _c_double_p, _c_double_p, _c_double_p]),
}

_lib = None
_lib_lock = threading.RLock()
_contexts: dict = {}


class DeviceError(RuntimeError):
    """A CUDA / device-side failure reported by libsdeb200."""


def lib():
    """Load libsdeb200.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        with _lib_lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        "libsdeb200.so is not built (%s); run "
                        "`python -m paper_1908_03869_b200._build` -- there is no CPU fallback"
                        % LIB_PATH)
                handle = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in SIGNATURES.items():
                    fn = getattr(handle, name)
                    fn.restype = res
                    fn.argtypes = args
                if handle.sdb_abi_version() != ABI_VERSION:
                    raise RuntimeError("libsdeb200.so ABI mismatch")
                _lib = handle
    return _lib


def last_error(ctx=None) -> str:
    msg = lib().sdb_last_error(ctx)
    return msg.decode() if msg else ""


def check(status: int, ctx=None, what: str = "sdeb200"):
    """Map an sdb_status onto the reference's exception types."""
    if status == SDB_OK:
        return
    msg = "%s: %s" % (what, last_error(ctx))
    if status == SDB_ERR_CONFIG:
        from .engine import ConfigError
        raise ConfigError(msg)
    if status == SDB_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    if status == SDB_ERR_ARGUMENT:
        raise ValueError(msg)
    raise DeviceError(msg)


def device_count() -> int:
    return int(lib().sdb_device_count())


def context(devices=None):
    """Cached sdb_ctx for a device tuple (default: SDEB200_DEVICES or (0,)).

    Shared by every caller in the process.  The library serialises the public
    calls on one context (sdb_ctx::call_mu) and reports errors per calling
    thread, so concurrent run_batch calls from several Python threads are
    safe; device-buffer calls on different streams are ordered after each
    other's use of the context's scratch buffers."""
    if devices is None:
        env = os.environ.get("SDEB200_DEVICES")
        devices = tuple(int(d) for d in env.split(",")) if env else (0,)
    devices = tuple(int(d) for d in devices)
    ctx = _contexts.get(devices)
    if ctx is None:
        with _lib_lock:  # one context per device tuple, also under concurrent first calls
            ctx = _contexts.get(devices)
            if ctx is None:
                arr = (ctypes.c_int * len(devices))(*devices)
                out = ctypes.c_void_p()
                check(lib().sdb_open(arr, len(devices), ctypes.byref(out)), None, "sdb_open")
                ctx = out.value
                _contexts[devices] = ctx
    return ctx


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_c_double_p)


def u32ptr(a: np.ndarray):
    return a.ctypes.data_as(_c_u32_p)


def u64ptr(a: np.ndarray):
    return a.ctypes.data_as(_c_u64_p)


def i64ptr(a: np.ndarray):
    return a.ctypes.data_as(_c_i64_p)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


#: stores at least this large get transparent-huge-page backing (host_empty)
HUGE_STORE_BYTES = 64 << 20

_PROT_RW = 0x1 | 0x2                # PROT_READ | PROT_WRITE
_MAP_PRIVATE_ANON = 0x02 | 0x20     # MAP_PRIVATE | MAP_ANONYMOUS (Linux)
_MADV_HUGEPAGE = 14
_libc = None
_pool_lock = threading.Lock()
_pool: dict[int, list[int]] = {}    # mapping size -> addresses of free, populated mappings
_pool_bytes = 0


def _libc_fns():
    global _libc
    if _libc is None:
        c = ctypes.CDLL(None, use_errno=True)
        c.mmap.restype = ctypes.c_void_p
        c.mmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int,
                           ctypes.c_int, ctypes.c_long]
        c.munmap.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
        c.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
        _libc = c
    return _libc


def _pool_cap() -> int:
    """Bytes of released store mappings kept for reuse: SDEB200_HOST_POOL_MB,
    default min(16 GiB, 1/8 of physical memory); 0 disables the pool."""
    env = os.environ.get("SDEB200_HOST_POOL_MB")
    if env is not None:
        return int(env) << 20
    try:
        ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except (ValueError, OSError):
        ram = 8 << 30
    return min(16 << 30, ram // 8)


class _StoreMapping:
    """Owner of one anonymous mapping behind a large store.  It is the base of
    the ctypes buffer the ndarray views, so it dies only after the last view;
    its pages (already faulted in) then go back to the pool for the next run's
    store of the same size, else are unmapped."""

    __slots__ = ("addr", "nbytes")

    def __init__(self, addr: int, nbytes: int):
        self.addr, self.nbytes = addr, nbytes

    def __del__(self):
        global _pool_bytes
        try:
            with _pool_lock:
                if _pool_bytes + self.nbytes <= _pool_cap():
                    _pool.setdefault(self.nbytes, []).append(self.addr)
                    _pool_bytes += self.nbytes
                    return
            _libc_fns().munmap(self.addr, self.nbytes)
        except Exception:  # interpreter shutdown: the OS reclaims the mapping
            pass


def _take_mapping(nbytes: int) -> int:
    global _pool_bytes
    with _pool_lock:
        free = _pool.get(nbytes)
        if free:
            _pool_bytes -= nbytes
            return free.pop()
    c = _libc_fns()
    addr = c.mmap(None, nbytes, _PROT_RW, _MAP_PRIVATE_ANON, -1, 0)
    if addr is None or addr == ctypes.c_void_p(-1).value:
        raise MemoryError("mmap of a %d-byte store failed (errno %d)" % (nbytes, ctypes.get_errno()))
    c.madvise(addr, nbytes, _MADV_HUGEPAGE)  # best effort: THP may be disabled
    return addr


def host_empty(shape, dtype=np.float64) -> np.ndarray:
    """``np.empty`` for a large run output.  Below HUGE_STORE_BYTES a plain
    ``np.empty``; above, an anonymous mapping advised MADV_HUGEPAGE, recycled
    through a process-wide pool once the store is dropped.  The pipeline's
    drain threads write every byte of a store; into a fresh mapping that costs
    a page fault per page (pinned -> fresh copy 19-28 GB/s with 4 KiB pages,
    38 GB/s with 2 MiB pages, into resident pages 80 GB/s on the B200 host,
    tools/host_copy_bench.cpp), so repeated runs reuse populated mappings the
    way a caching allocator does.  The array is an ordinary writable ndarray
    (slicing, pickling, ctypes); its memory lives as long as any view of it."""
    dtype = np.dtype(dtype)
    nbytes = int(np.prod(shape, dtype=np.int64)) * dtype.itemsize
    if nbytes < HUGE_STORE_BYTES:
        return np.empty(shape, dtype)
    addr = _take_mapping(nbytes)
    buf = (ctypes.c_char * nbytes).from_address(addr)
    buf._owner = _StoreMapping(addr, nbytes)  # ctypes buffers take attributes
    return np.frombuffer(buf, dtype=dtype).reshape(shape)


class _PinnedBlock:
    """Owner of one sdb_host_alloc block (freed when the last view dies)."""

    __slots__ = ("addr",)

    def __init__(self, addr: int):
        self.addr = addr

    def __del__(self):
        try:
            if _lib is not None:
                _lib.sdb_host_free(self.addr)
        except Exception:  # interpreter shutdown
            pass


def host_pinned(shape, dtype=np.float64) -> np.ndarray:
    """An ndarray in page-locked host memory (cudaHostAlloc through
    sdb_host_alloc).  Run inputs in such arrays are DMA'd to the GPU without
    the host staging copy; pinning costs ~0.3 s per GB, so allocate once and
    refill, as for any pinned buffer."""
    dtype = np.dtype(dtype)
    nbytes = int(np.prod(shape, dtype=np.int64)) * dtype.itemsize
    out = ctypes.c_void_p()
    check(lib().sdb_host_alloc(nbytes, ctypes.byref(out)), None, "sdb_host_alloc")
    buf = (ctypes.c_char * max(nbytes, 1)).from_address(out.value)
    buf._owner = _PinnedBlock(out.value)
    return np.frombuffer(buf, dtype=dtype, count=int(np.prod(shape, dtype=np.int64))).reshape(shape)
