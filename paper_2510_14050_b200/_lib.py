"""ctypes binding of libnmx.so (include/nmx.h).

The product path has no CPU fallback: if the shared library is missing or no
CUDA device is visible, every compute entry point raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libnmx.so"

NMX_OK = 0
NMX_EINVAL = -1
NMX_ENOMEM = -2
NMX_ECUDA = -3
NMX_ENODEV = -4

GEN_UNIFORM = 0
GEN_POWERLAW = 1
REDUCE_SUM = 0
REDUCE_MAX = 1

# Every symbol include/nmx.h declares, with its ctypes signature.
_VP = C.c_void_p
_U64 = C.c_uint64
SIGNATURES = {
    "nmx_version": (C.c_int, []),
    "nmx_last_error": (C.c_char_p, []),
    "nmx_device_count": (C.c_int, [C.POINTER(C.c_int)]),
    "nmx_create": (C.c_int, [C.c_int, C.POINTER(_VP)]),
    "nmx_destroy": (None, [_VP]),
    "nmx_stream": (_VP, [_VP]),
    "nmx_synchronize": (C.c_int, [_VP]),
    "nmx_malloc": (C.c_int, [_VP, _U64, C.POINTER(_VP)]),
    "nmx_free": (C.c_int, [_VP, _VP]),
    "nmx_host_alloc": (C.c_int, [_U64, C.POINTER(_VP)]),
    "nmx_host_free": (C.c_int, [_VP]),
    "nmx_memcpy_h2d": (C.c_int, [_VP, _VP, _VP, _U64]),
    "nmx_memcpy_d2h": (C.c_int, [_VP, _VP, _VP, _U64]),
    "nmx_generate": (C.c_int, [_VP, C.c_int, _U64, _U64, _U64, _U64, _VP, _VP]),
    "nmx_stats9_device": (C.c_int, [_VP, _VP, _VP, _VP, _U64, _U64, _VP]),
    "nmx_stats9_host": (C.c_int, [_VP, _VP, _VP, _VP, _U64, _U64, _VP]),
    "nmx_stats9_host_i64": (C.c_int, [_VP, _VP, _VP, _VP, _U64, _U64, _VP]),
    "nmx_stats9_host_batches": (C.c_int, [_VP, _U64, _VP, _VP, _VP, _VP, _U64, _VP]),
    "nmx_stream_stats9": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _U64, _U64, _VP]),
    "nmx_stream_records": (C.c_int, [_VP, _VP, _VP, _U64, _U64, _VP]),
    "nmx_anonymize_begin": (C.c_int, [_VP, _VP, _VP, _U64, _VP]),
    "nmx_parse_matrix_text": (C.c_int, [_VP, _VP, _U64, _VP, _VP]),
    "nmx_format_matrix_text": (C.c_int, [_VP, _VP, _VP, _VP, _U64, _VP, _U64, _VP]),
    "nmx_anonymize_finish": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP]),
    "nmx_unpack_records": (C.c_int, [_VP, _VP, _U64, _VP, _VP, _VP, _U64]),
    "nmx_window_stats9_device": (C.c_int, [_VP, _VP, _VP, _VP, _U64, _U64, _U64, _VP]),
    "nmx_window_stats9_host": (C.c_int, [_VP, _VP, _VP, _VP, _U64, _U64, _U64, _VP]),
    "nmx_reduce_i64": (C.c_int, [_VP, _VP, _U64, C.c_int, _VP]),
    "nmx_coo_build": (C.c_int, [_VP, _VP, _VP, _VP, _U64, _U64, _U64, C.POINTER(_U64)]),
    "nmx_coo_fetch": (C.c_int, [_VP, _VP, _VP]),
    "nmx_coo_rowptr": (C.c_int, [_VP, _U64, _U64, _U64, _U64, _VP]),
    "nmx_flat_build": (C.c_int, [_VP, _VP, _U64, _VP, _VP, _U64, C.POINTER(_U64), C.POINTER(_U64)]),
    "nmx_flat_fetch": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP]),
    "nmx_coo_from_packets": (C.c_int, [_VP, _VP, _VP, _VP, _U64, C.POINTER(_VP)]),
    "nmx_coo_upload": (C.c_int, [_VP, _VP, _VP, _U64, C.POINTER(_VP)]),
    "nmx_coo_merge_add": (C.c_int, [_VP, _VP, _VP, C.POINTER(_VP)]),
    "nmx_coo_stats9": (C.c_int, [_VP, _VP, _VP]),
    "nmx_coo_nnz": (C.c_int, [_VP, C.POINTER(_U64)]),
    "nmx_coo_download": (C.c_int, [_VP, _VP, _VP, _VP]),
    "nmx_coo_free": (None, [_VP]),
    "nmx_coo_reserve": (C.c_int, [_VP, _U64]),
    "nmx_partition_packets": (C.c_int, [_VP, _VP, _VP, _VP, _U64, C.c_int, _VP, _VP, _VP]),
    "nmx_shard_rows": (C.c_int, [_VP, _VP, _VP, _U64, _U64, C.c_int, _VP, _VP, _VP, _VP]),
    "nmx_shard_cols": (C.c_int, [_VP, _VP, _VP, _U64, _U64, _VP]),
    "nmx_group_create": (C.c_int, [_VP, C.c_int, C.POINTER(_VP)]),
    "nmx_group_destroy": (None, [_VP]),
    "nmx_group_size": (C.c_int, [_VP, C.POINTER(C.c_int)]),
    "nmx_group_context": (C.c_int, [_VP, C.c_int, C.POINTER(_VP)]),
    "nmx_group_stats9_device": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _U64, _VP]),
    "nmx_group_stats9_host": (C.c_int, [_VP, _VP, _VP, _VP, _U64, _U64, _U64, _VP]),
    "nmx_group_last_exchange": (C.c_int, [_VP, C.POINTER(_U64), C.POINTER(_U64)]),
    "nmx_comm_unique_id": (C.c_int, [_VP]),
    "nmx_comm_init": (C.c_int, [_VP, _VP, C.c_int, C.c_int, C.POINTER(_VP)]),
    "nmx_comm_destroy": (None, [_VP]),
    "nmx_stats9_sharded": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _U64, _U64, _VP]),
    "nmx_stats9_sharded_host": (C.c_int, [_VP, _VP, _VP, _VP, _VP, _U64, _U64, _VP]),
    "nmx_comm_last_exchange": (C.c_int, [_VP, C.POINTER(_U64), C.POINTER(_U64)]),
    "nmx_last_kernel_class": (C.c_int, [_VP, C.POINTER(C.c_float), C.POINTER(C.c_int), C.POINTER(_U64), C.c_char_p,
                                         C.c_int]),
    "nmx_last_kernel_launches": (C.c_int, [_VP, C.c_int, C.POINTER(C.c_float), C.POINTER(_U64), C.POINTER(C.c_int)]),
    "nmx_last_stages": (C.c_int, [_VP, C.POINTER(C.c_float), C.c_int]),
    "nmx_last_timing": (C.c_int, [_VP, C.POINTER(C.c_float), C.POINTER(C.c_float), C.POINTER(C.c_int),
                                  C.POINTER(C.c_int)]),
}


class NativeUnavailable(RuntimeError):
    """libnmx.so is not built or no CUDA device is visible (there is no CPU fallback)."""


class NmxError(RuntimeError):
    """A CUDA or allocation failure inside libnmx.so."""


_lib = None
_lib_lock = threading.Lock()


def load(path: str | os.PathLike | None = None):
    """Load libnmx.so and bind every declared symbol (no device needed)."""
    global _lib
    with _lib_lock:
        if _lib is not None and path is None:
            return _lib
        p = Path(path) if path else LIB_PATH
        if not p.exists():
            raise NativeUnavailable(f"{p} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if path is None:
            _lib = lib
        return lib


def check(rc: int) -> None:
    if rc == NMX_OK:
        return
    msg = (load().nmx_last_error() or b"").decode(errors="replace")
    if rc == NMX_EINVAL:
        raise ValueError(msg)
    if rc == NMX_ENODEV:
        raise NativeUnavailable(msg)
    raise NmxError(f"libnmx error {rc}: {msg}")


class Context:
    """One device + one CUDA stream (include/nmx.h nmx_ctx)."""

    def __init__(self, device: int = 0, handle=None, owner=None):
        lib = load()
        if handle is None:
            h = C.c_void_p()
            check(lib.nmx_create(int(device), C.byref(h)))
        else:  # a group rank's context: owned (and destroyed) by the group
            h = handle
        self._h = h
        self._owner = owner
        self.device = int(device)
        self._lib = lib

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        if self._h and self._owner is None:
            self._lib.nmx_destroy(self._h)
        self._h = C.c_void_p()

    def __del__(self):  # pragma: no cover - interpreter shutdown ordering
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return self._lib.nmx_stream(self._h) or 0

    def last_timing(self):
        t, s = C.c_float(), C.c_float()
        sl, kl = C.c_int(), C.c_int()
        check(self._lib.nmx_last_timing(self._h, C.byref(t), C.byref(s), C.byref(sl), C.byref(kl)))
        st = (C.c_float * 8)()
        k = self._lib.nmx_last_stages(self._h, st, 8)
        dms, dl, db = C.c_float(), C.c_int(), C.c_uint64()
        name = C.create_string_buffer(64)
        check(self._lib.nmx_last_kernel_class(self._h, C.byref(dms), C.byref(dl), C.byref(db), name, 64))
        lms, lby, lc = (C.c_float * 32)(), (C.c_uint64 * 32)(), C.c_int()
        check(self._lib.nmx_last_kernel_launches(self._h, 32, lms, lby, C.byref(lc)))
        return dict(total_ms=t.value, sort_ms=s.value, sort_launches=sl.value, kernel_launches=kl.value,
                    stages_ms=[round(st[i], 4) for i in range(max(k, 0))],
                    dom_ms=dms.value, dom_launches=dl.value, dom_bytes=db.value, dom_name=name.value.decode(),
                    dom_per_launch=[(lms[i], lby[i]) for i in range(min(lc.value, 32))])


_contexts: dict[int, Context] = {}
_ctx_lock = threading.Lock()
_current = threading.local()


def context(device: int = 0) -> Context:
    """The calling thread's bound context (``using``), else the process-wide cached
    context of ``device``."""
    c = getattr(_current, "ctx", None)
    if c is not None:
        return c
    with _ctx_lock:
        c = _contexts.get(device)
        if c is None:
            c = Context(device)
            _contexts[device] = c
        return c


class using:
    """``with using(ctx):`` routes this thread's library calls to ``ctx`` (a group
    rank's own stream and workspace) whatever device argument they carry."""

    def __init__(self, ctx: Context):
        self.ctx = ctx

    def __enter__(self):
        self.prev = getattr(_current, "ctx", None)
        _current.ctx = self.ctx
        return self.ctx

    def __exit__(self, *exc):
        _current.ctx = self.prev


class Group:
    """G ranks (nmx_group), rank r on CUDA device ``devices[r]`` (several ranks may share
    a device). Owns one context per rank; the sharded statistics run in the library."""

    def __init__(self, devices):
        lib = load()
        devs = [int(d) for d in devices]
        arr = (C.c_int * len(devs))(*devs)
        h = C.c_void_p()
        check(lib.nmx_group_create(arr, len(devs), C.byref(h)))
        self._h = h
        self._lib = lib
        self.devices = devs
        self.contexts = []
        for r, d in enumerate(devs):
            ch = C.c_void_p()
            check(lib.nmx_group_context(h, r, C.byref(ch)))
            self.contexts.append(Context(d, handle=ch, owner=self))

    @property
    def size(self) -> int:
        return len(self.devices)

    def stats9_host(self, src, dst, valid=None, address_space: int = 1 << 32, batch_count: int = 1) -> tuple:
        s, d, v = _u32_host(src), _u32_host(dst), _valid_host(valid)
        if len(s) != len(d) or (v is not None and len(v) != len(s)):
            raise ValueError("src, dst and valid must have equal lengths")
        out = np.zeros(9, dtype=np.int64)
        check(self._lib.nmx_group_stats9_host(self._h, _ptr(s), _ptr(d), _ptr(v), len(s), int(address_space),
                                              int(batch_count), out.ctypes.data))
        return tuple(int(x) for x in out)

    def stats9_device(self, srcs, dsts, address_space: int = 1 << 32, valids=None) -> tuple:
        """Rank r's packets: device columns srcs[r] / dsts[r] on devices[r]."""
        g = self.size
        if len(srcs) != g or len(dsts) != g:
            raise ValueError(f"need one (src, dst) pair per rank ({g})")
        sp = (C.c_void_p * g)(*[_ptr(a) for a in srcs])
        dp = (C.c_void_p * g)(*[_ptr(a) for a in dsts])
        vp = (C.c_void_p * g)(*[_ptr(a) for a in valids]) if valids is not None else None
        ns = (C.c_uint64 * g)(*[int(a.numel()) for a in srcs])
        out = np.zeros(9, dtype=np.int64)
        check(self._lib.nmx_group_stats9_device(self._h, sp, dp, vp, ns, int(address_space), out.ctypes.data))
        return tuple(int(x) for x in out)

    def last_exchange(self) -> tuple[int, int]:
        a, b = C.c_uint64(), C.c_uint64()
        check(self._lib.nmx_group_last_exchange(self._h, C.byref(a), C.byref(b)))
        return int(a.value), int(b.value)

    def close(self) -> None:
        if self._h:
            for c in self.contexts:
                c._h = C.c_void_p()
            self._lib.nmx_group_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def device_count() -> int:
    lib = load()
    n = C.c_int(0)
    rc = lib.nmx_device_count(C.byref(n))
    return n.value if rc == NMX_OK else 0


def _ptr(a) -> int:
    if a is None:
        return 0
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return int(a.data_ptr())  # torch tensor (device or pinned host)


def _u32_host(a) -> np.ndarray:
    a = np.asarray(a)
    if a.dtype == np.uint32 and a.flags.c_contiguous:
        return a
    if a.size and (a.min() < 0 or a.max() > 0xFFFFFFFF):
        raise ValueError("addresses must lie in [0, 2^32)")
    return np.ascontiguousarray(a, dtype=np.uint32)


def _valid_host(v):
    if v is None:
        return None
    v = np.asarray(v)
    if v.dtype == np.bool_ or v.dtype == np.uint8:
        return np.ascontiguousarray(v).view(np.uint8)
    return np.ascontiguousarray(v != 0).view(np.uint8)


def _is_device(a) -> bool:
    return hasattr(a, "is_cuda") and bool(a.is_cuda)


def stats9(src, dst, valid=None, address_space: int = 1 << 32, device: int = 0) -> tuple:
    """Nine statistics of the summed traffic matrix (nmx_stats9_{host,device}).

    ``src``/``dst``: numpy arrays (host) or CUDA uint32/int32 tensors (device).
    """
    ctx = context(device)
    out = np.zeros(9, dtype=np.int64)
    if _is_device(src):
        n = int(src.numel())
        check(ctx._lib.nmx_stats9_device(ctx.handle, _ptr(src), _ptr(dst), _ptr(valid), n, int(address_space),
                                         out.ctypes.data))
    else:
        s, d, v = _u32_host(src), _u32_host(dst), _valid_host(valid)
        if len(s) != len(d) or (v is not None and len(v) != len(s)):
            raise ValueError("src, dst and valid must have equal lengths")
        check(ctx._lib.nmx_stats9_host(ctx.handle, _ptr(s), _ptr(d), _ptr(v), len(s), int(address_space),
                                       out.ctypes.data))
    return tuple(int(x) for x in out)


def _prefer_bundled_nccl() -> None:
    """libnmx opens NCCL at first use; point it at the nvidia-nccl wheel's library (the
    one torch loads) so one process never mixes two NCCL versions under one soname."""
    if os.environ.get("NMX_NCCL_LIB"):
        return
    import sys

    for p in sys.path:
        cand = Path(p) / "nvidia" / "nccl" / "lib" / "libnccl.so.2"
        if cand.exists():
            os.environ["NMX_NCCL_LIB"] = str(cand)
            return


def stats9_i64(src: np.ndarray, dst: np.ndarray, valid=None, address_space: int = 1 << 32, device: int = 0) -> tuple:
    """nmx_stats9_host_i64: the reference's int64 PacketStream columns (+ bool valid)
    straight from host memory (narrowed by library threads, pinned staging)."""
    ctx = context(device)
    s = np.ascontiguousarray(src, dtype=np.int64)
    d = np.ascontiguousarray(dst, dtype=np.int64)
    v = None if valid is None else np.ascontiguousarray(valid, dtype=bool).view(np.uint8)
    if len(s) != len(d) or (v is not None and len(v) != len(s)):
        raise ValueError("src, dst and valid must have equal lengths")
    out = np.zeros(9, dtype=np.int64)
    check(ctx._lib.nmx_stats9_host_i64(ctx.handle, s.ctypes.data, d.ctypes.data, _ptr(v), len(s), int(address_space),
                                       out.ctypes.data))
    return tuple(int(x) for x in out)


def comm_unique_id() -> bytes:
    """A fresh NCCL communicator id (nmx_comm_unique_id) for rank 0 to hand out."""
    _prefer_bundled_nccl()
    lib = load()
    buf = (C.c_uint8 * 128)()
    check(lib.nmx_comm_unique_id(buf))
    return bytes(buf)


class Communicator:
    """libnmx's own NCCL communicator for this process's rank (nmx_comm): the sharded
    nine statistics run inside the library (grouped ncclSend / ncclRecv exchanges,
    ncclAllGather of the part counts, ncclAllReduce SUM / MAX) on the context stream."""

    def __init__(self, uid: bytes, world: int, rank: int, device: int = 0):
        if len(uid) != 128:
            raise ValueError("an NCCL id is 128 bytes")
        _prefer_bundled_nccl()
        self.ctx = context(device)
        self.device, self.world, self.rank = device, world, rank
        self._h = C.c_void_p()
        idbuf = (C.c_uint8 * 128).from_buffer_copy(uid)
        check(self.ctx._lib.nmx_comm_init(self.ctx.handle, idbuf, int(world), int(rank), C.byref(self._h)))

    def stats9(self, src, dst, valid=None, address_space: int = 1 << 32) -> tuple:
        """This rank's packets (device tensors / DeviceArrays, or host arrays) -> the
        nine statistics of the matrix summed over every rank's packets."""
        out = np.zeros(9, dtype=np.int64)
        if _is_device(src):
            n = int(src.numel())
            check(self.ctx._lib.nmx_stats9_sharded(self.ctx.handle, self._h, _ptr(src), _ptr(dst), _ptr(valid), n,
                                                   int(address_space), out.ctypes.data))
        else:
            s, d, v = _u32_host(src), _u32_host(dst), _valid_host(valid)
            if len(s) != len(d) or (v is not None and len(v) != len(s)):
                raise ValueError("src, dst and valid must have equal lengths")
            check(self.ctx._lib.nmx_stats9_sharded_host(self.ctx.handle, self._h, _ptr(s), _ptr(d), _ptr(v), len(s),
                                                        int(address_space), out.ctypes.data))
        return tuple(int(x) for x in out)

    def last_exchange(self) -> tuple:
        a, b = C.c_uint64(), C.c_uint64()
        check(self.ctx._lib.nmx_comm_last_exchange(self._h, C.byref(a), C.byref(b)))
        return int(a.value), int(b.value)

    def close(self) -> None:
        if self._h:
            self.ctx._lib.nmx_comm_destroy(self._h)
            self._h = C.c_void_p()


def stats9_batches(batches, address_space: int = 1 << 32, device: int = 0) -> list:
    """Nine statistics of each of several independent host batches
    (nmx_stats9_host_batches): ``batches`` = [(src, dst) or (src, dst, valid), ...]
    host arrays; the result is one 9-tuple per batch, each equal to ``stats9`` of that
    batch. Batch k+1's H2D copy overlaps batch k's device work (pinned memory streams
    at full host-link bandwidth)."""
    ctx = context(device)
    cols = []
    for w in batches:
        s, d = _u32_host(w[0]), _u32_host(w[1])
        v = _valid_host(w[2]) if len(w) > 2 else None
        if len(s) != len(d) or (v is not None and len(v) != len(s)):
            raise ValueError("src, dst and valid must have equal lengths")
        cols.append((s, d, v))
    k = len(cols)
    srcp = (C.c_void_p * max(k, 1))(*[c[0].ctypes.data for c in cols])
    dstp = (C.c_void_p * max(k, 1))(*[c[1].ctypes.data for c in cols])
    anyv = any(c[2] is not None for c in cols)
    valp = (C.c_void_p * max(k, 1))(*[(c[2].ctypes.data if c[2] is not None else None) for c in cols])
    lens = (C.c_uint64 * max(k, 1))(*[len(c[0]) for c in cols])
    out = np.zeros(9 * max(k, 1), dtype=np.int64)
    check(ctx._lib.nmx_stats9_host_batches(ctx.handle, k, srcp, dstp, valp if anyv else None, lens,
                                           int(address_space), out.ctypes.data))
    del cols
    return [tuple(int(x) for x in out[9 * i:9 * i + 9]) for i in range(k)]


def stream_stats9(windows, address_space: int = 1 << 32, device: int = 0) -> tuple:
    """Nine statistics of the matrix summed over host packet windows
    (nmx_stream_stats9): ``windows`` = [(src, dst) or (src, dst, valid), ...] host
    arrays (uint32 columns; pinned memory streams at full host-link bandwidth).
    The H2D copy of window k+1 overlaps the device work of window k."""
    ctx = context(device)
    cols = []
    for w in windows:
        s, d = _u32_host(w[0]), _u32_host(w[1])
        v = _valid_host(w[2]) if len(w) > 2 else None
        if len(s) != len(d) or (v is not None and len(v) != len(s)):
            raise ValueError("src, dst and valid must have equal lengths")
        cols.append((s, d, v))
    k = len(cols)
    srcp = (C.c_void_p * max(k, 1))(*[c[0].ctypes.data for c in cols])
    dstp = (C.c_void_p * max(k, 1))(*[c[1].ctypes.data for c in cols])
    anyv = any(c[2] is not None for c in cols)
    valp = (C.c_void_p * max(k, 1))(*[(c[2].ctypes.data if c[2] is not None else None) for c in cols])
    lens = (C.c_uint64 * max(k, 1))(*[len(c[0]) for c in cols])
    out = np.zeros(9, dtype=np.int64)
    check(ctx._lib.nmx_stream_stats9(ctx.handle, srcp, dstp, valp if anyv else None, lens, k, int(address_space),
                                     out.ctypes.data))
    del cols
    return tuple(int(x) for x in out)


def _record_bytes(w) -> np.ndarray:
    a = np.asarray(w)
    if a.dtype.itemsize == 9 and a.dtype.names:  # structured packet records
        a = a.view(np.uint8).reshape(-1)
    if a.dtype != np.uint8 or a.ndim != 1 or len(a) % 9:
        raise ValueError("packet records must be whole 9-byte records (traffic.py:25)")
    return np.ascontiguousarray(a)


def stream_records(windows, address_space: int = 1 << 32, device: int = 0) -> tuple:
    """Nine statistics of the matrix summed over windows of raw packet-file records
    (9-byte {u32 src, u32 dst, u8 valid}, traffic.py:25) in host memory
    (nmx_stream_records; pinned memory streams at full host-link bandwidth)."""
    ctx = context(device)
    recs = [_record_bytes(w) for w in windows]
    k = len(recs)
    ptrs = (C.c_void_p * max(k, 1))(*[r.ctypes.data for r in recs])
    lens = (C.c_uint64 * max(k, 1))(*[len(r) // 9 for r in recs])
    out = np.zeros(9, dtype=np.int64)
    check(ctx._lib.nmx_stream_records(ctx.handle, ptrs, lens, k, int(address_space), out.ctypes.data))
    del recs
    return tuple(int(x) for x in out)


def unpack_records(d_rec, n: int, d_src, d_dst, d_valid, address_space: int = 1 << 32, device: int = 0) -> None:
    """Device records -> device u32 src / dst + u8 valid columns (nmx_unpack_records)."""
    ctx = context(device)
    check(ctx._lib.nmx_unpack_records(ctx.handle, _ptr(d_rec), int(n), _ptr(d_src), _ptr(d_dst), _ptr(d_valid),
                                      int(address_space)))


def anonymize_device(src, dst, key: int, device: int = 0, tables: bool = True):
    """Keyed first-seen dense relabel (traffic.py:107-137) on the GPU.

    ``src``/``dst``: host uint32-compatible arrays or DeviceArrays of n packets.
    Returns (src', dst' as DeviceArrays, k, distinct, code) -- ``distinct`` (ascending
    raw addresses) and ``code`` (their new labels) as uint32 numpy arrays when
    ``tables``, else None. perm = numpy default_rng(key).permutation(k), exactly
    the reference's draw, is generated here on the host between the two calls."""
    ctx = context(device)
    keep = []
    if not _is_device(src):
        s, d = _u32_host(src), _u32_host(dst)
        if len(s) != len(d):
            raise ValueError("src and dst must have equal lengths")
        ds, dd = DeviceArray(len(s), device=device), DeviceArray(len(s), device=device)
        if len(s):
            ds.upload(s)
            dd.upload(d)
        keep = [ds, dd]
        src, dst = ds, dd
    n = int(src.numel())
    k = C.c_uint64()
    check(ctx._lib.nmx_anonymize_begin(ctx.handle, _ptr(src), _ptr(dst), n, C.byref(k)))
    k = int(k.value)
    perm = np.ascontiguousarray(np.random.default_rng(key).permutation(k), dtype=np.uint32)
    so, do = DeviceArray(max(n, 1), device=device), DeviceArray(max(n, 1), device=device)
    distinct = np.empty(k, np.uint32) if tables else None
    code = np.empty(k, np.uint32) if tables else None
    check(ctx._lib.nmx_anonymize_finish(ctx.handle, perm.ctypes.data, _ptr(so), _ptr(do),
                                        distinct.ctypes.data if tables and k else None,
                                        code.ctypes.data if tables and k else None))
    del keep
    return so, do, k, distinct, code


# nmx_parse_matrix_text diagnoses (include/nmx.h NMX_TXT_*)
TXT_OK, TXT_HEADER, TXT_DIM, TXT_NNZ, TXT_FIELDS, TXT_INTEGERS, TXT_COUNT, TXT_BOUNDS, TXT_VALUE, TXT_ORDER, \
    TXT_WIDE, TXT_ENCODING = range(12)


def parse_matrix_text(text: bytes, device: int = 0):
    """Text matrix file bytes -> (info, COO handle or None), tokenised and validated on
    the GPU. info = (dim, nnz, entry lines, diagnosis, line): diagnosis TXT_OK with a
    handle, or the first rule the file breaks (the caller words the error)."""
    ctx = context(device)
    info = np.zeros(8, dtype=np.int64)
    h = C.c_void_p()
    buf = np.frombuffer(text, dtype=np.uint8) if len(text) else np.zeros(1, np.uint8)
    check(ctx._lib.nmx_parse_matrix_text(ctx.handle, buf.ctypes.data, len(text), info.ctypes.data, C.byref(h)))
    return tuple(int(x) for x in info[:5]), (h if h.value else None)


def format_matrix_text(rows, cols, values, device: int = 0) -> bytes:
    """The "row col value\n" lines of a matrix file, formatted on the GPU."""
    ctx = context(device)
    r = np.ascontiguousarray(rows, dtype=np.int64)
    c = np.ascontiguousarray(cols, dtype=np.int64)
    v = np.ascontiguousarray(values, dtype=np.int64)
    n = len(r)
    if n == 0:
        return b""
    size = C.c_uint64()
    check(ctx._lib.nmx_format_matrix_text(ctx.handle, r.ctypes.data, c.ctypes.data, v.ctypes.data, n, None, 0,
                                          C.byref(size)))
    out = np.empty(int(size.value), dtype=np.uint8)
    check(ctx._lib.nmx_format_matrix_text(ctx.handle, r.ctypes.data, c.ctypes.data, v.ctypes.data, n,
                                          out.ctypes.data, out.nbytes, C.byref(size)))
    return out.tobytes()


def window_stats9(src, dst, valid, address_space: int, window_size: int, device: int = 0) -> np.ndarray:
    """Per-window nine statistics, shape (ceil(n/W), 9) int64."""
    ctx = context(device)
    if _is_device(src):
        n = int(src.numel())
    else:
        src, dst, valid = _u32_host(src), _u32_host(dst), _valid_host(valid)
        n = len(src)
    nw = (n + window_size - 1) // window_size if window_size >= 1 else 0
    out = np.zeros((max(nw, 0), 9), dtype=np.int64)
    fn = ctx._lib.nmx_window_stats9_device if _is_device(src) else ctx._lib.nmx_window_stats9_host
    check(fn(ctx.handle, _ptr(src), _ptr(dst), _ptr(valid), n, int(address_space), int(window_size),
             out.ctypes.data if nw else 0))
    return out


def reduce_i64(data: np.ndarray, op: int, device: int = 0) -> int:
    ctx = context(device)
    a = np.ascontiguousarray(data, dtype=np.int64)
    out = np.zeros(1, dtype=np.int64)
    check(ctx._lib.nmx_reduce_i64(ctx.handle, _ptr(a), len(a), int(op), out.ctypes.data))
    return int(out[0])


def generate(kind: int, seed: int, offset: int, n: int, address_space: int, d_src, d_dst, device: int = 0) -> None:
    ctx = context(device)
    check(ctx._lib.nmx_generate(ctx.handle, int(kind), int(seed), int(offset), int(n), int(address_space),
                                _ptr(d_src), _ptr(d_dst)))


class DeviceArray:
    """Device memory from nmx_malloc, freed on close/GC. Quacks like a CUDA
    tensor for the entry points above (data_ptr / numel / is_cuda)."""

    is_cuda = True

    def __init__(self, n: int, itemsize: int = 4, device: int = 0):
        self.ctx = context(device)
        self.n = int(n)
        self.itemsize = itemsize
        p = C.c_void_p()
        check(self.ctx._lib.nmx_malloc(self.ctx.handle, max(self.n * itemsize, 1), C.byref(p)))
        self._p = p

    def data_ptr(self) -> int:
        return self._p.value or 0

    def numel(self) -> int:
        return self.n

    def upload(self, host: np.ndarray) -> "DeviceArray":
        host = np.ascontiguousarray(host)
        if host.nbytes > self.n * self.itemsize:
            raise ValueError("host array larger than device buffer")
        check(self.ctx._lib.nmx_memcpy_h2d(self.ctx.handle, self._p, host.ctypes.data, host.nbytes))
        return self

    def download(self, dtype=np.uint32) -> np.ndarray:
        out = np.empty(self.n * self.itemsize // np.dtype(dtype).itemsize, dtype=dtype)
        check(self.ctx._lib.nmx_memcpy_d2h(self.ctx.handle, out.ctypes.data, self._p, out.nbytes))
        return out

    def close(self) -> None:
        if self._p:
            self.ctx._lib.nmx_free(self.ctx.handle, self._p)
            self._p = C.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


class PinnedArray:
    """Page-locked host buffer (nmx_host_alloc) viewed as a numpy array."""

    def __init__(self, n: int, dtype=np.uint32):
        dt = np.dtype(dtype)
        self._lib = load()
        p = C.c_void_p()
        check(self._lib.nmx_host_alloc(max(n * dt.itemsize, 1), C.byref(p)))
        self._p = p
        buf = (C.c_char * max(n * dt.itemsize, 1)).from_address(p.value)
        self.array = np.frombuffer(buf, dtype=dt, count=n)

    def close(self) -> None:
        if self._p:
            self.array = None
            self._lib.nmx_host_free(self._p)
            self._p = C.c_void_p()

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass
