"""Packet streams and traffic matrices -- the reference's data layer on the B200.

Mirrors ``netmeter.traffic`` (/root/reference/pkg/src/netmeter/traffic.py)
name for name; every aggregation runs in libnmx.so:

* ``matrix_from_pairs`` / ``build_matrices`` (traffic.py:197-242): packed-key
  onesweep sort + reduce-by-key on the GPU (``nmx_coo_build``), dense CSR
  ``row_ptr`` per window by a GPU binary-search kernel (``nmx_coo_rowptr``);
* ``to_flat`` (traffic.py:263-292): row and column grouping on the GPU
  (``nmx_flat_build``).

The containers keep the reference layout (int64 CSR, dense in ``dim``) so the
reference's own tests and callers work unchanged. The hot path itself
(``analytics.stats9`` / ``analyze_summed``) never materialises them.
"""

from __future__ import annotations

import ctypes as C
from collections.abc import Mapping
from dataclasses import dataclass, field
from typing import Iterator

import numpy as np

from . import _lib

_PACKET_DTYPE = np.dtype([("src", "<u4"), ("dst", "<u4"), ("valid", "u1")])


class MatrixFormatError(ValueError):
    """A matrix violates the CSR invariants (traffic.py:28-29)."""


class MatrixFileError(ValueError):
    """A matrix file cannot be parsed; the message carries path and line (traffic.py:32-33)."""


@dataclass(frozen=True)
class PacketRecord:
    src: int
    dst: int
    valid: bool = True


@dataclass
class PacketStream:
    """Columnar packets (traffic.py:43-71): int64 src/dst, bool valid, address_space."""

    src: np.ndarray
    dst: np.ndarray
    valid: np.ndarray
    address_space: int

    def __post_init__(self):
        self.src = np.ascontiguousarray(self.src, dtype=np.int64)
        self.dst = np.ascontiguousarray(self.dst, dtype=np.int64)
        self.valid = np.ascontiguousarray(self.valid, dtype=bool)
        if not (len(self.src) == len(self.dst) == len(self.valid)):
            raise ValueError("src, dst and valid must have equal lengths")
        if self.address_space < 1:
            raise ValueError("address_space must be >= 1")
        if len(self.src):
            lo = min(self.src.min(), self.dst.min())
            hi = max(self.src.max(), self.dst.max())
            if lo < 0 or hi >= self.address_space:
                raise ValueError("addresses must lie in [0, address_space)")

    def __len__(self) -> int:
        return len(self.src)

    def records(self) -> Iterator[PacketRecord]:
        for s, d, v in zip(self.src.tolist(), self.dst.tolist(), self.valid.tolist()):
            yield PacketRecord(s, d, v)

    def wire(self):
        """The device wire format: u32 src / dst columns + u8 valid (8-9 B/packet)."""
        if self.address_space > 1 << 32:
            raise ValueError("address_space above 2^32 does not fit the 32-bit packet format")
        return (self.src.astype(np.uint32), self.dst.astype(np.uint32), self.valid.view(np.uint8))


@dataclass(frozen=True)
class AnonymizationMap:
    key: int
    mapping: dict = field(repr=False)


def generate_packets(n: int, address_space: int, seed: int, invalid_fraction: float = 0.0) -> PacketStream:
    """Uniform packets from PCG64, identical to traffic.py:82-104 for identical arguments
    (host input preparation; bulk synthetic inputs come from nmx_generate instead)."""
    if n < 0:
        raise ValueError("n must be >= 0")
    if address_space < 1:
        raise ValueError("address_space must be >= 1")
    if not 0.0 <= invalid_fraction <= 1.0:
        raise ValueError("invalid_fraction must be in [0, 1]")
    rng = np.random.default_rng(seed)
    src = rng.integers(0, address_space, size=n, dtype=np.int64)
    dst = rng.integers(0, address_space, size=n, dtype=np.int64)
    valid = rng.random(n) >= invalid_fraction if invalid_fraction > 0.0 else np.ones(n, dtype=bool)
    return PacketStream(src=src, dst=dst, valid=valid, address_space=address_space)


class AddressMap(Mapping):
    """Raw address -> anonymized index, the ``AnonymizationMap.mapping`` of
    traffic.py:74-79 as a read-only Mapping over two device-produced tables
    (ascending distinct addresses, their codes) instead of a k-entry Python dict."""

    def __init__(self, distinct: np.ndarray, code: np.ndarray):
        self._d = distinct
        self._c = code

    def __getitem__(self, address):
        try:
            a = int(address)
        except (TypeError, ValueError):
            raise KeyError(address) from None
        i = int(np.searchsorted(self._d, a)) if 0 <= a < 2**32 else len(self._d)
        if i < len(self._d) and int(self._d[i]) == a:
            return int(self._c[i])
        raise KeyError(address)

    def __iter__(self):
        return iter(self._d.tolist())

    def __len__(self) -> int:
        return len(self._d)

    def values(self):
        return self._c.astype(np.int64).tolist()


def anonymize(stream: PacketStream, key: int) -> tuple[PacketStream, AnonymizationMap]:
    """Relabel every observed address with a keyed pseudorandom dense index
    (traffic.py:107-137): first-seen order over src0, dst0, src1, dst1, ...,
    mapped through default_rng(key).permutation(k). The sort, run detection,
    first-seen ranking and relabel run on the GPU (nmx_anonymize_begin/finish,
    SURVEY.md 8(f) f3); addresses must fit the 32-bit packet format."""
    src, dst, _ = stream.wire()
    so, do, k, distinct, code = _lib.anonymize_device(src, dst, key)
    n = len(stream)
    s_out = so.download()[:n].astype(np.int64)
    d_out = do.download()[:n].astype(np.int64)
    so.close()
    do.close()
    anon = PacketStream(src=s_out, dst=d_out, valid=stream.valid.copy(), address_space=max(1, k))
    return anon, AnonymizationMap(key=key, mapping=AddressMap(distinct, code))


@dataclass(eq=False)
class TrafficMatrix:
    """One window's packet-count matrix in CSR form (traffic.py:140-194)."""

    window_id: int
    dim: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.row_ptr = np.ascontiguousarray(self.row_ptr, dtype=np.int64)
        self.col_idx = np.ascontiguousarray(self.col_idx, dtype=np.int64)
        self.values = np.ascontiguousarray(self.values, dtype=np.int64)

    @property
    def nnz(self) -> int:
        return len(self.col_idx)

    def __eq__(self, other) -> bool:
        if not isinstance(other, TrafficMatrix):
            return NotImplemented
        return (self.window_id == other.window_id and self.dim == other.dim
                and np.array_equal(self.row_ptr, other.row_ptr) and np.array_equal(self.col_idx, other.col_idx)
                and np.array_equal(self.values, other.values))

    def validate(self) -> None:
        """Raise MatrixFormatError unless the CSR invariants hold (traffic.py:170-188)."""
        if self.dim < 1:
            raise MatrixFormatError("dim must be >= 1")
        rp = self.row_ptr
        if len(rp) != self.dim + 1:
            raise MatrixFormatError("row_ptr must have dim + 1 entries")
        if rp[0] != 0 or np.any(rp[1:] < rp[:-1]):
            raise MatrixFormatError("row_ptr must start at 0 and be nondecreasing")
        if rp[-1] != len(self.col_idx) or len(self.col_idx) != len(self.values):
            raise MatrixFormatError("row_ptr[-1], col_idx and values must agree on nnz")
        if self.nnz:
            c = self.col_idx
            if c.min() < 0 or c.max() >= self.dim:
                raise MatrixFormatError("column indices must lie in [0, dim)")
            if self.values.min() < 1:
                raise MatrixFormatError("values must be positive packet counts")
            # strictly increasing within rows: a decrease is only legal at a row start
            starts = np.zeros(self.nnz, dtype=bool)
            starts[rp[:-1][rp[:-1] < rp[1:]]] = True
            bad = (c[1:] <= c[:-1]) & ~starts[1:]
            if np.any(bad):
                raise MatrixFormatError("column indices must be strictly increasing within rows")

    def to_dense(self) -> np.ndarray:
        dense = np.zeros((self.dim, self.dim), dtype=np.int64)
        rows = np.repeat(np.arange(self.dim, dtype=np.int64), np.diff(self.row_ptr))
        dense[rows, self.col_idx] = self.values
        return dense


def _bits(space: int) -> int:
    return max(1, (int(space) - 1).bit_length())


def _coo(src, dst, valid, space: int, window_size: int, device: int = 0):
    """Device build of the (windowed) unique-link COO; returns keys (u64) and counts."""
    ctx = _lib.context(device)
    s = np.ascontiguousarray(src, dtype=np.uint32)
    d = np.ascontiguousarray(dst, dtype=np.uint32)
    v = None if valid is None else np.ascontiguousarray(valid, dtype=bool).view(np.uint8)
    nnz = C.c_uint64(0)
    _lib.check(ctx._lib.nmx_coo_build(ctx.handle, s.ctypes.data, d.ctypes.data, v.ctypes.data if v is not None else None,
                                      len(s), int(space), int(window_size), C.byref(nnz)))
    keys = np.empty(nnz.value, dtype=np.uint64)
    counts = np.empty(nnz.value, dtype=np.int64)
    _lib.check(ctx._lib.nmx_coo_fetch(ctx.handle, keys.ctypes.data, counts.ctypes.data))
    return ctx, keys, counts


def _matrix_from_slice(ctx, keys, counts, lo, hi, window, b, dim, window_id) -> TrafficMatrix:
    row_ptr = np.empty(dim + 1, dtype=np.int64)
    _lib.check(ctx._lib.nmx_coo_rowptr(ctx.handle, int(lo), int(hi), int(window), int(dim), row_ptr.ctypes.data))
    cols = (keys[lo:hi] & np.uint64((1 << b) - 1)).astype(np.int64)
    return TrafficMatrix(window_id=window_id, dim=dim, row_ptr=row_ptr, col_idx=cols, values=counts[lo:hi])


def matrix_from_pairs(src, dst, dim: int, window_id: int = 0) -> TrafficMatrix:
    """Count-aggregate (src, dst) pairs into one CSR matrix (traffic.py:197-218)."""
    if dim < 1:
        raise ValueError("dim must be >= 1")
    if dim > 2**31:
        raise ValueError("dim too large for packed pair keys")
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    if len(src) != len(dst):
        raise ValueError("src and dst must have equal lengths")
    if len(src) and (min(src.min(), dst.min()) < 0 or max(src.max(), dst.max()) >= dim):
        raise ValueError("pairs must lie in [0, dim)")
    if len(src) == 0:
        return TrafficMatrix(window_id, dim, np.zeros(dim + 1, np.int64), np.empty(0, np.int64),
                             np.empty(0, np.int64))
    ctx, keys, counts = _coo(src, dst, None, dim, 0)
    return _matrix_from_slice(ctx, keys, counts, 0, len(keys), 0, _bits(dim), dim, window_id)


def build_matrices(stream: PacketStream, window_size: int, dim: int | None = None) -> list[TrafficMatrix]:
    """One matrix per window of ``window_size`` raw positions (traffic.py:221-242)."""
    if window_size < 1:
        raise ValueError("window_size must be >= 1")
    if dim is None:
        dim = stream.address_space
    if dim < 1:
        raise ValueError("dim must be >= 1")
    if dim > 2**31:
        raise ValueError("dim too large for packed pair keys")
    n = len(stream)
    nw = (n + window_size - 1) // window_size
    if nw == 0:
        return []
    if len(stream.src) and max(stream.src.max(), stream.dst.max()) >= dim:
        raise ValueError("addresses must lie in [0, dim)")
    b = _bits(dim)
    wb = max(0, (nw - 1).bit_length()) if nw > 1 else 0
    out = []
    if 2 * b + wb <= 64:
        ctx, keys, counts = _coo(stream.src, stream.dst, stream.valid, dim, window_size if nw > 1 else 0)
        win = keys >> np.uint64(2 * b) if 2 * b < 64 else np.zeros(len(keys), np.uint64)
        bounds = np.searchsorted(win, np.arange(nw + 1, dtype=np.uint64))
        for t in range(nw):
            out.append(_matrix_from_slice(ctx, keys, counts, bounds[t], bounds[t + 1], t, b, dim, t))
        return out
    for t in range(nw):  # keys too wide for a window field: one device build per window
        lo, hi = t * window_size, min((t + 1) * window_size, n)
        ctx, keys, counts = _coo(stream.src[lo:hi], stream.dst[lo:hi], stream.valid[lo:hi], dim, 0)
        out.append(_matrix_from_slice(ctx, keys, counts, 0, len(keys), 0, b, dim, t))
    return out


@dataclass
class FlatContainers:
    """Flat per-nonzero expansion of a CSR matrix (traffic.py:245-260)."""

    edges: np.ndarray
    weights: np.ndarray
    out_degrees: np.ndarray
    in_degrees: np.ndarray
    row_sums: np.ndarray
    col_sums: np.ndarray


def to_flat(matrix: TrafficMatrix, device: int = 0) -> FlatContainers:
    """Expand a valid CSR matrix into its flat containers (traffic.py:263-292), on the GPU."""
    matrix.validate()
    nnz = matrix.nnz
    if nnz == 0:
        e = np.empty(0, np.int64)
        return FlatContainers(np.empty((0, 2), np.int64), e.copy(), e.copy(), e.copy(),
                              np.empty((0, 2), np.int64), np.empty((0, 2), np.int64))
    ctx = _lib.context(device)
    r, c = C.c_uint64(0), C.c_uint64(0)
    _lib.check(ctx._lib.nmx_flat_build(ctx.handle, matrix.row_ptr.ctypes.data, matrix.dim, matrix.col_idx.ctypes.data,
                                       matrix.values.ctypes.data, nnz, C.byref(r), C.byref(c)))
    edge_src = np.empty(nnz, np.int64)
    rid, rnz, rsum = (np.empty(r.value, np.int64) for _ in range(3))
    cid, cnz, csum = (np.empty(c.value, np.int64) for _ in range(3))
    _lib.check(ctx._lib.nmx_flat_fetch(ctx.handle, edge_src.ctypes.data, rid.ctypes.data, rnz.ctypes.data,
                                       rsum.ctypes.data, cid.ctypes.data, cnz.ctypes.data, csum.ctypes.data))
    return FlatContainers(
        edges=np.column_stack([edge_src, matrix.col_idx]),
        weights=matrix.values.copy(),
        out_degrees=rnz,
        in_degrees=cnz,
        row_sums=np.column_stack([rid, rsum]),
        col_sums=np.column_stack([cid, csum]),
    )


# ---------------------------------------------------------------------------
# binary packet files (traffic.py:370-388): 9-byte little-endian records
# ---------------------------------------------------------------------------
def write_packets(stream: PacketStream, path) -> None:
    """Binary packet file: little-endian u32 src, u32 dst, u8 valid per record
    (traffic.py:370-378)."""
    if len(stream) and max(stream.src.max(), stream.dst.max()) >= 2**32:
        raise ValueError("addresses exceed the 32-bit record format")
    out = np.empty(len(stream), dtype=_PACKET_DTYPE)
    out["src"] = stream.src
    out["dst"] = stream.dst
    out["valid"] = stream.valid
    out.tofile(str(path))


def read_packets(path, address_space: int | None = None) -> PacketStream:
    """Read a binary packet file; address_space defaults to max address + 1
    (traffic.py:381-388)."""
    raw = np.fromfile(str(path), dtype=_PACKET_DTYPE)
    src = raw["src"].astype(np.int64)
    dst = raw["dst"].astype(np.int64)
    if address_space is None:
        address_space = int(max(src.max(), dst.max())) + 1 if len(raw) else 1
    return PacketStream(src=src, dst=dst, valid=raw["valid"] != 0, address_space=address_space)


# ---------------------------------------------------------------------------
# text matrix files (traffic.py:295-367)
# ---------------------------------------------------------------------------
def write_matrix(matrix: TrafficMatrix, path) -> None:
    """Coordinate text form: ``dim nnz`` header, then sorted ``row col value`` lines
    (traffic.py:295-304); the lines are formatted on the GPU."""
    matrix.validate()
    rows = np.repeat(np.arange(matrix.dim, dtype=np.int64), np.diff(matrix.row_ptr))
    body = _lib.format_matrix_text(rows, matrix.col_idx, matrix.values)
    with open(path, "wb") as f:
        f.write(f"{matrix.dim} {matrix.nnz}\n".encode())
        f.write(body)


_TXT_MESSAGES = {
    _lib.TXT_HEADER: "expected header 'dim nnz'",
    _lib.TXT_DIM: "dim must be >= 1",
    _lib.TXT_NNZ: "nnz must be >= 0",
    _lib.TXT_FIELDS: "expected 'row col value'",
    _lib.TXT_INTEGERS: "expected 'row col value' integers",
    _lib.TXT_VALUE: "value must be >= 1",
    _lib.TXT_ORDER: "entries must be sorted row-major with no duplicates",
}


def _ascii_form(data: bytes) -> bytes:
    """Text with non-ASCII whitespace, line breaks or digits, rewritten into the ASCII
    form the device tokenizer reads, line for line (so diagnosed line numbers stay the
    reference's): str.splitlines() / str.split() boundaries, int()-valid tokens in
    plain decimal. Everything else is left for the device to diagnose."""
    text = data.decode()  # UnicodeDecodeError (a ValueError), as Path.read_text raises

    def token(t: str) -> str:
        if t.isascii():
            return t
        try:
            return str(int(t))
        except ValueError:
            return "?"  # still not an integer: keeps the line's integer error

    return "\n".join(" ".join(token(t) for t in ln.split()) for ln in text.splitlines()).encode()


def _parse_text(path, data: bytes):
    """(dim, COO handle) of a matrix file parsed and validated on the GPU; malformed
    files raise MatrixFileError worded as the reference's read_matrix (traffic.py:307-367)."""
    (dim, nnz, entries, code, line), h = _lib.parse_matrix_text(data)
    if code == _lib.TXT_ENCODING:
        (dim, nnz, entries, code, line), h = _lib.parse_matrix_text(_ascii_form(data))
        if code == _lib.TXT_ENCODING:
            raise MatrixFileError(f"{path}: unreadable characters")
    if code == _lib.TXT_OK:
        return dim, h
    if code == _lib.TXT_COUNT:
        raise MatrixFileError(f"{path}: header claims {nnz} entries, file has {entries}")
    if code == _lib.TXT_BOUNDS:
        raise MatrixFileError(f"{path}: line {line}: row/col outside [0, {dim})")
    if code == _lib.TXT_WIDE:
        raise MatrixFileError(f"{path}: line {line}: dim beyond 2^32 (device matrix range)")
    raise MatrixFileError(f"{path}: line {line}: {_TXT_MESSAGES[code]}")


def read_matrix_device(path, window_id: int = 0):
    """Parse a matrix file on the GPU into a device COO (keys row << 32 | col, int64
    counts) without host containers: (dim, DeviceCOO)."""
    from .coo import DeviceCOO

    dim, h = _parse_text(path, open(path, "rb").read())
    return dim, DeviceCOO(h)


def read_matrix(path, window_id: int = 0) -> TrafficMatrix:
    """Parse a matrix file written by write_matrix (traffic.py:307-367): tokenised,
    converted and validated on the GPU; malformed files raise MatrixFileError naming
    the file and line, as the reference does."""
    from .coo import DeviceCOO

    dim, h = _parse_text(path, open(path, "rb").read())
    coo = DeviceCOO(h)
    keys, counts = coo.download()
    coo.close()
    rows = (keys >> np.uint64(32)).astype(np.int64)
    cols = (keys & np.uint64(0xFFFFFFFF)).astype(np.int64)
    row_ptr = np.zeros(dim + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=dim), out=row_ptr[1:])
    return TrafficMatrix(window_id=window_id, dim=dim, row_ptr=row_ptr, col_idx=cols, values=counts)


