"""CPU oracle for the netmeter traffic-matrix hot path -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it. The product package
(``paper_2510_14050_b200``) never imports anything under ``oracle/``.

It restates, in numpy, the reference algorithm of the path
packets -> traffic matrix -> statistics (all citations relative to
``/root/reference/pkg/src/netmeter``):

* ``ref_matrix_from_pairs``  restates ``traffic.py:197-218`` (packed key
  ``src*dim+dst``, ``np.unique(return_counts)``, dense ``row_ptr``);
* ``ref_build_matrices``     restates ``traffic.py:221-242`` (windows by raw
  position, invalid packets dropped, positions kept);
* ``ref_to_flat``            restates ``traffic.py:263-292`` (edges, weights,
  degrees, row/col sums via repeat / reduceat / add.at);
* ``ref_analyze_flat``       restates ``analytics.py:95-106`` plus the three
  extra Graph Challenge maxima composed from ``max_scan``
  (``analytics.py:89-92``) over ``weights``, ``row_sums[:,1]``,
  ``col_sums[:,1]``;
* ``ref_analyze_dataset``    restates ``analytics.py:109-130`` totals;
* ``oracle_analyze_pairs``   restates the brute-force set/dict oracle
  ``analytics.py:133-157`` (extended to nine statistics);
* ``stats9_packed``          hypersparse packed-u64 restatement of the same
  semantics for sizes whose dense ``dim`` the reference cannot hold
  (SURVEY.md 8(c) "Large sizes");
* ``generate_packets`` / ``anonymize`` restate ``traffic.py:82-104`` and
  ``traffic.py:107-137`` (input preparation for configs 1-2);
* ``gen_uniform`` / ``gen_powerlaw`` are the counter-based splitmix64
  generators of SURVEY.md 8(d) (cfg3/cfg4); ``paper_2510_14050_b200``'s
  CUDA generator implements the identical integer function.

Parity pinning: ``tests/golden/make_golden.py`` imports the real reference
from ``/root/reference`` in the build container and records its outputs in
``tests/golden/golden.json``; ``tests/test_oracle.py`` checks this module
against every one of those vectors.
"""

from __future__ import annotations

import numpy as np

# Canonical order of the nine statistics everywhere in this repo.
STATS9_FIELDS = (
    "valid_packets",
    "unique_links",
    "max_link_packets",
    "unique_sources",
    "max_source_packets",
    "max_fanout",
    "unique_destinations",
    "max_destination_packets",
    "max_fanin",
)
# Order of the six reference measures (analytics.py:31-40, AggregateReport).
REPORT6_FIELDS = (
    "valid_packets",
    "unique_links",
    "unique_sources",
    "max_fanout",
    "unique_destinations",
    "max_fanin",
)

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


# ----------------------------------------------------------------------------
# generators
# ----------------------------------------------------------------------------
def splitmix64(x: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser of (x + golden gamma); uint64 in, uint64 out."""
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _scale(v32: np.ndarray, address_space: int) -> np.ndarray:
    """Map a uniform u32 onto [0, address_space) by multiply-shift (exact ints)."""
    if address_space == 1 << 32:
        return v32.astype(np.uint32)
    return ((v32.astype(np.uint64) * np.uint64(address_space)) >> np.uint64(32)).astype(np.uint32)


def gen_uniform(seed: int, offset: int, n: int, address_space: int = 1 << 32):
    """cfg3 generator: src = lo32(sm64(seed*2^40 + 2i)), dst = hi32(sm64(seed*2^40 + 2i + 1)).

    ``i`` runs over [offset, offset+n) so the stream is chunk-addressable.
    Returns (src, dst) as uint32 arrays in [0, address_space).
    """
    base = np.uint64((seed << 40) & 0xFFFFFFFFFFFFFFFF)
    i = np.arange(offset, offset + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        c = base + np.uint64(2) * i
        s = splitmix64(c) & np.uint64(0xFFFFFFFF)
        d = splitmix64(c + np.uint64(1)) >> np.uint64(32)
    return _scale(s, address_space), _scale(d, address_space)


def _octave(bits: np.ndarray) -> np.ndarray:
    e = bits >> np.uint64(59)
    low = bits & ((np.uint64(1) << e) - np.uint64(1))
    rank = (np.uint64(1) << e) | low
    with np.errstate(over="ignore"):
        return (rank * np.uint64(0x9E3779B1)) & np.uint64(0xFFFFFFFF)


def gen_powerlaw(seed: int, offset: int, n: int, address_space: int = 1 << 32):
    """cfg4 "octave" generator: e = bits>>59, rank = 2^e | (bits & (2^e-1)),
    address = rank * 0x9E3779B1 mod 2^32 (a bijection that scatters heavy hitters)."""
    base = np.uint64((seed << 40) & 0xFFFFFFFFFFFFFFFF)
    i = np.arange(offset, offset + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        c = base + np.uint64(2) * i
        s = _octave(splitmix64(c))
        d = _octave(splitmix64(c + np.uint64(1)))
    return _scale(s, address_space), _scale(d, address_space)


def generate_packets(n: int, address_space: int, seed: int, invalid_fraction: float = 0.0):
    """Restates traffic.py:82-104 (PCG64 via default_rng; same call sequence).

    Returns (src int64, dst int64, valid bool)."""
    rng = np.random.default_rng(seed)
    src = rng.integers(0, address_space, size=n, dtype=np.int64)
    dst = rng.integers(0, address_space, size=n, dtype=np.int64)
    if invalid_fraction > 0.0:
        valid = rng.random(n) >= invalid_fraction
    else:
        valid = np.ones(n, dtype=bool)
    return src, dst, valid


def anonymize(src: np.ndarray, dst: np.ndarray, key: int):
    """Restates traffic.py:107-137 without the Python dict: first-seen rank
    (src before dst) mapped through default_rng(key).permutation(k).

    Returns (src', dst', address_space')."""
    n = len(src)
    inter = np.empty(2 * n, dtype=np.int64)
    inter[0::2] = src
    inter[1::2] = dst
    distinct, first_pos, inverse = np.unique(inter, return_index=True, return_inverse=True)
    order = np.argsort(first_pos, kind="stable")
    rank = np.empty(len(distinct), dtype=np.int64)
    rank[order] = np.arange(len(distinct), dtype=np.int64)
    perm = np.random.default_rng(key).permutation(len(distinct)).astype(np.int64)
    relabeled = perm[rank][inverse]
    return relabeled[0::2].copy(), relabeled[1::2].copy(), max(1, len(distinct))


def compact_ids(src: np.ndarray, dst: np.ndarray):
    """Relabel-invariant compaction (np.unique return_inverse) so the dense
    reference restatement can hold raw 2^32 address spaces."""
    n = len(src)
    both = np.concatenate([np.asarray(src, np.int64), np.asarray(dst, np.int64)])
    distinct, inverse = np.unique(both, return_inverse=True)
    return inverse[:n].astype(np.int64), inverse[n:].astype(np.int64), max(1, len(distinct))


# ----------------------------------------------------------------------------
# faithful restatement of the reference path (dense in dim, like the reference)
# ----------------------------------------------------------------------------
def ref_matrix_from_pairs(src, dst, dim: int):
    """traffic.py:197-218 -> (row_ptr, col_idx, values), all int64."""
    if dim < 1:
        raise ValueError("dim must be >= 1")
    if dim > 2**31:
        raise ValueError("dim too large for packed pair keys")
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    keys, counts = np.unique(src * dim + dst, return_counts=True)
    rows = keys // dim
    cols = keys % dim
    row_ptr = np.zeros(dim + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=dim), out=row_ptr[1:])
    return row_ptr, cols, counts.astype(np.int64)


def ref_build_matrices(src, dst, valid, window_size: int, dim: int):
    """traffic.py:221-242 -> list of (row_ptr, col_idx, values)."""
    if window_size < 1:
        raise ValueError("window_size must be >= 1")
    n = len(src)
    out = []
    for t in range(0, (n + window_size - 1) // window_size):
        lo, hi = t * window_size, min((t + 1) * window_size, n)
        keep = valid[lo:hi]
        out.append(ref_matrix_from_pairs(src[lo:hi][keep], dst[lo:hi][keep], dim))
    return out


def ref_to_flat(row_ptr, col_idx, values, dim: int) -> dict:
    """traffic.py:263-292 (validation omitted: inputs come from ref_matrix_from_pairs)."""
    row_nnz = np.diff(row_ptr)
    edge_src = np.repeat(np.arange(dim, dtype=np.int64), row_nnz)
    nnz = len(col_idx)
    edges = np.column_stack([edge_src, col_idx]) if nnz else np.empty((0, 2), np.int64)
    occupied_rows = np.flatnonzero(row_nnz > 0)
    if len(occupied_rows):
        row_totals = np.add.reduceat(values, row_ptr[:-1][occupied_rows])
    else:
        row_totals = np.empty(0, dtype=np.int64)
    row_sums = np.column_stack([occupied_rows, row_totals]).astype(np.int64)
    col_nnz = np.bincount(col_idx, minlength=dim)
    col_totals = np.zeros(dim, dtype=np.int64)
    np.add.at(col_totals, col_idx, values)
    occupied_cols = np.flatnonzero(col_nnz > 0)
    col_sums = np.column_stack([occupied_cols, col_totals[occupied_cols]]).astype(np.int64)
    return dict(
        edges=edges,
        weights=values.copy(),
        out_degrees=row_nnz[occupied_rows].astype(np.int64),
        in_degrees=col_nnz[occupied_cols].astype(np.int64),
        row_sums=row_sums,
        col_sums=col_sums,
    )


def ref_read_matrix(path):
    """traffic.py:307-367 restated for well-formed files, with the reference's own
    per-line Python tokenising (the cost the CLI end-to-end clock is dominated
    by): -> (dim, row_ptr, col_idx, values)."""
    from pathlib import Path

    lines = [parts for parts in (ln.split() for ln in Path(path).read_text().splitlines()) if parts]
    dim, nnz = (int(t) for t in lines[0])
    entries = np.empty((len(lines) - 1, 3), dtype=np.int64)
    for k, parts in enumerate(lines[1:]):
        entries[k] = [int(t) for t in parts]
    assert len(entries) == nnz
    rows, cols, values = entries[:, 0], entries[:, 1], entries[:, 2]
    row_ptr = np.zeros(dim + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=dim), out=row_ptr[1:])
    return dim, row_ptr, cols, values


def _max0(a) -> int:
    """max_scan semantics (analytics.py:89-92): empty -> 0, INT64_MIN -> 0."""
    a = np.asarray(a, dtype=np.int64)
    if a.size == 0:
        return 0
    m = int(a.max())
    return 0 if m == np.iinfo(np.int64).min else m


def ref_analyze_flat(flat: dict) -> tuple:
    """analytics.py:95-106 plus the three max_scan compositions -> 9-tuple."""
    return (
        int(np.add.reduce(flat["weights"])) if len(flat["weights"]) else 0,
        len(flat["edges"]),
        _max0(flat["weights"]),
        len(flat["row_sums"]),
        _max0(flat["row_sums"][:, 1]) if len(flat["row_sums"]) else 0,
        _max0(flat["out_degrees"]),
        len(flat["col_sums"]),
        _max0(flat["col_sums"][:, 1]) if len(flat["col_sums"]) else 0,
        _max0(flat["in_degrees"]),
    )


def ref_stats9(src, dst, valid, dim: int) -> tuple:
    """Nine statistics of the summed matrix by the reference's own route:
    build_matrices(stream, window_size=len(stream)) -> to_flat -> analyze
    (SURVEY.md 0.10). Empty stream -> all zeros."""
    n = len(src)
    if n == 0:
        return (0,) * 9
    (m,) = ref_build_matrices(src, dst, valid, n, dim)
    return ref_analyze_flat(ref_to_flat(*m, dim))


def ref_analyze_dataset(src, dst, valid, window_size: int, dim: int):
    """analytics.py:109-130 on build_matrices windows, nine statistics per window.

    Totals: sums of the counting measures, max of the maxima."""
    reports = [ref_analyze_flat(ref_to_flat(*m, dim))
               for m in ref_build_matrices(src, dst, valid, window_size, dim)]
    return reports, totals9(reports)


def totals9(reports) -> tuple:
    """Dataset totals (analytics.py:122-129) extended to nine statistics."""
    sums = {0, 1, 3, 6}
    out = []
    for k in range(9):
        vals = [r[k] for r in reports]
        out.append(sum(vals) if k in sums else max(vals, default=0))
    return tuple(out)


def to6(s9) -> tuple:
    """Project nine statistics onto the reference AggregateReport order."""
    return (s9[0], s9[1], s9[3], s9[5], s9[6], s9[8])


# ----------------------------------------------------------------------------
# brute-force oracle (analytics.py:133-157), nine statistics
# ----------------------------------------------------------------------------
def oracle_analyze_pairs(pairs) -> tuple:
    pairs = [(int(s), int(d)) for s, d in pairs]
    links: dict = {}
    for p in pairs:
        links[p] = links.get(p, 0) + 1
    dsts_of: dict = {}
    srcs_of: dict = {}
    src_pk: dict = {}
    dst_pk: dict = {}
    for (s, d), c in links.items():
        dsts_of.setdefault(s, set()).add(d)
        srcs_of.setdefault(d, set()).add(s)
        src_pk[s] = src_pk.get(s, 0) + c
        dst_pk[d] = dst_pk.get(d, 0) + c
    return (
        len(pairs),
        len(links),
        max(links.values(), default=0),
        len(dsts_of),
        max(src_pk.values(), default=0),
        max((len(v) for v in dsts_of.values()), default=0),
        len(srcs_of),
        max(dst_pk.values(), default=0),
        max((len(v) for v in srcs_of.values()), default=0),
    )


# ----------------------------------------------------------------------------
# hypersparse packed-key restatement (same semantics, never O(dim))
# ----------------------------------------------------------------------------
def _runs(sorted_vals: np.ndarray):
    """Run starts and lengths of a sorted array."""
    if len(sorted_vals) == 0:
        return np.empty(0, np.int64), np.empty(0, np.int64)
    head = np.empty(len(sorted_vals), dtype=bool)
    head[0] = True
    np.not_equal(sorted_vals[1:], sorted_vals[:-1], out=head[1:])
    starts = np.flatnonzero(head)
    lens = np.diff(np.append(starts, len(sorted_vals)))
    return starts, lens


def stats9_packed(src, dst, valid=None) -> tuple:
    """Nine statistics via key = (src<<32)|dst (order-equal to src*dim+dst for
    any dim <= 2^32). Counts are int64."""
    src = np.asarray(src).astype(np.uint64)
    dst = np.asarray(dst).astype(np.uint64)
    if valid is not None:
        valid = np.asarray(valid, dtype=bool)
        src, dst = src[valid], dst[valid]
    n = len(src)
    if n == 0:
        return (0,) * 9
    keys = np.sort((src << np.uint64(32)) | dst)
    starts, counts = _runs(keys)
    ukeys = keys[starts]
    del keys
    usrc = ukeys >> np.uint64(32)
    rs, rl = _runs(usrc)  # rl = fan-out per source
    row_pk = np.add.reduceat(counts, rs)
    udst = (ukeys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    order = np.argsort(udst, kind="stable")
    sdst = udst[order]
    cs, cl = _runs(sdst)  # cl = fan-in per destination
    col_pk = np.add.reduceat(counts[order], cs)
    return (
        int(n),
        int(len(ukeys)),
        int(counts.max()),
        int(len(rs)),
        int(row_pk.max()),
        int(rl.max()),
        int(len(cs)),
        int(col_pk.max()),
        int(cl.max()),
    )


def stats9_windows_packed(src, dst, valid, window_size: int):
    """Per-window nine statistics (analyze_dataset semantics) via the packed restatement."""
    n = len(src)
    reports = []
    for t in range(0, (n + window_size - 1) // window_size):
        lo, hi = t * window_size, min((t + 1) * window_size, n)
        v = None if valid is None else valid[lo:hi]
        reports.append(stats9_packed(src[lo:hi], dst[lo:hi], v))
    return reports, totals9(reports)


def coo_packed(src, dst, valid=None):
    """Sorted unique keys ((src<<32)|dst, uint64) and int64 counts."""
    src = np.asarray(src).astype(np.uint64)
    dst = np.asarray(dst).astype(np.uint64)
    if valid is not None:
        valid = np.asarray(valid, dtype=bool)
        src, dst = src[valid], dst[valid]
    keys = np.sort((src << np.uint64(32)) | dst)
    starts, counts = _runs(keys)
    return keys[starts], counts.astype(np.int64)


def stats9_from_coo(ukeys: np.ndarray, counts: np.ndarray) -> tuple:
    """Nine statistics of a sorted unique COO (keys (src<<32)|dst, counts)."""
    if len(ukeys) == 0:
        return (0,) * 9
    usrc = ukeys >> np.uint64(32)
    rs, rl = _runs(usrc)
    row_pk = np.add.reduceat(counts, rs)
    udst = (ukeys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    order = np.argsort(udst, kind="stable")
    cs, cl = _runs(udst[order])
    col_pk = np.add.reduceat(counts[order], cs)
    return (int(counts.sum()), int(len(ukeys)), int(counts.max()), int(len(rs)), int(row_pk.max()),
            int(rl.max()), int(len(cs)), int(col_pk.max()), int(cl.max()))


def merge_add_coo(ka, ca, kb, cb):
    """Element-wise sum of two sorted unique COO matrices (K10 semantics)."""
    k = np.concatenate([ka, kb])
    c = np.concatenate([ca, cb]).astype(np.int64)
    order = np.argsort(k, kind="stable")
    k, c = k[order], c[order]
    starts, _ = _runs(k)
    return k[starts], np.add.reduceat(c, starts) if len(k) else c


def checksum_u32(a: np.ndarray) -> str:
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.uint32).tobytes()).hexdigest()[:16]
