"""Multi-GPU nine statistics: one process per GPU, NCCL all-to-all exchange.

Production (NCCL process group): the whole pipeline below runs inside libnmx.so
through its own NCCL communicator (``nmx_stats9_sharded``, ``_lib.Communicator``);
torch.distributed only hands the 128-byte communicator id from rank 0 to the others.
The Python orchestration in ``sharded_stats9`` is the same pipeline with the
exchanges in torch.distributed, kept for gloo (CPU tests, several ranks on one GPU).

SURVEY.md 8(e). Each rank holds a contiguous shard of the packet stream
(partition_even rule, partitioning.py:62-70). The summed matrix's statistics
need one exchange per axis:

1. route every valid packet to owner(src) = (fmix32(src) * G) >> 32 (all-to-all,
   8 B per packet); the owner then holds every packet of its sources, so one
   local sort finalises its links and rows (fields 0-5 exact, disjoint by src);
2. route each unique link's (dst, count) to owner(dst) (all-to-all, 8 B per
   link); the owner groups its destinations (fields 6-8 exact);
3. one int64 all-reduce SUM over {valid, links, sources, destinations} and one
   MAX over {max link, max source packets, max fan-out, max destination
   packets, max fan-in}.

Every operation is integer and order-independent, so the result is
bit-identical for every G. The device work behind ``ops`` is libnmx.so
(``CudaShardOps``); tests drive the same orchestration over ``gloo`` with a
CPU stand-in for the device ops (tests/test_distributed.py).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

SUM_FIELDS = (0, 1, 3, 6)
MAX_FIELDS = (2, 4, 5, 7, 8)
ROW_FIELDS = (0, 1, 2, 3, 4, 5)
COL_FIELDS = (6, 7, 8)


def fmix32(x: np.ndarray) -> np.ndarray:
    """murmur3 32-bit finaliser (same integer function as nmx_kernels.cuh fmix32)."""
    h = np.asarray(x, dtype=np.uint32).astype(np.uint64)
    m = np.uint64(0xFFFFFFFF)
    h ^= h >> np.uint64(16)
    h = (h * np.uint64(0x85EBCA6B)) & m
    h ^= h >> np.uint64(13)
    h = (h * np.uint64(0xC2B2AE35)) & m
    h ^= h >> np.uint64(16)
    return h


def owner(x: np.ndarray, parts: int) -> np.ndarray:
    """owner(x) = (fmix32(x) * parts) >> 32."""
    return ((fmix32(x) * np.uint64(parts)) >> np.uint64(32)).astype(np.int64)


class CudaShardOps:
    """Device stages from libnmx.so over torch CUDA int32 tensors (raw u32 bits)."""

    def __init__(self, device: int = 0):
        import torch

        from . import _lib

        self.torch = torch
        self._lib = _lib
        self.device = device
        self.ctx = _lib.context(device)

    def empty(self, n: int):
        return self.torch.empty(max(int(n), 1), dtype=self.torch.int32, device=f"cuda:{self.device}")[: int(n)]

    def sync(self):
        self.torch.cuda.current_stream(self.device).synchronize()

    def partition_packets(self, src, dst, valid, parts: int):
        n = int(src.numel())
        out_s, out_d = self.empty(n), self.empty(n)
        counts = (C.c_uint64 * parts)()
        self.sync()
        self._lib.check(self.ctx._lib.nmx_partition_packets(
            self.ctx.handle, src.data_ptr(), dst.data_ptr(), valid.data_ptr() if valid is not None else None, n,
            parts, out_s.data_ptr(), out_d.data_ptr(), counts))
        c = [int(x) for x in counts]
        tot = sum(c)
        return out_s[:tot], out_d[:tot], c

    def rows(self, src, dst, space: int, parts: int):
        n = int(src.numel())
        out_d, out_c = self.empty(n), self.empty(n)
        counts = (C.c_uint64 * parts)()
        stats = np.zeros(9, dtype=np.int64)
        self.sync()
        self._lib.check(self.ctx._lib.nmx_shard_rows(
            self.ctx.handle, src.data_ptr() if n else None, dst.data_ptr() if n else None, n, int(space), parts,
            out_d.data_ptr() if n else None, out_c.data_ptr() if n else None, counts, stats.ctypes.data))
        c = [int(x) for x in counts]
        tot = sum(c)
        return stats, out_d[:tot], out_c[:tot], c

    def cols(self, dst, cnt, space: int):
        u = int(dst.numel())
        stats = np.zeros(9, dtype=np.int64)
        self.sync()
        self._lib.check(self.ctx._lib.nmx_shard_cols(
            self.ctx.handle, dst.data_ptr() if u else None, cnt.data_ptr() if u else None, u, int(space),
            stats.ctypes.data))
        return stats

    def int64_tensor(self, values):
        return self.torch.tensor(list(values), dtype=self.torch.int64, device=f"cuda:{self.device}")


def _host_staged(dist, group) -> bool:
    """gloo exchanges host tensors only: device tensors are staged through the host
    (used to run the multi-rank flow with several ranks on one GPU; NCCL in production)."""
    return dist.get_backend(group) == "gloo"


def _alltoall_counts(torch, dist, counts, ops, group):
    send = ops.int64_tensor(counts)
    recv = ops.int64_tensor([0] * len(counts))
    if _host_staged(dist, group):
        r = torch.zeros(len(counts), dtype=torch.int64)
        dist.all_to_all_single(r, send.cpu(), group=group)
        return [int(x) for x in r.tolist()]
    dist.all_to_all_single(recv, send, group=group)
    return [int(x) for x in recv.tolist()]


def _alltoall(dist, ops, send, send_counts, recv_counts, group):
    recv = ops.empty(sum(recv_counts))
    if _host_staged(dist, group) and recv.is_cuda:
        r = recv.new_empty(recv.shape, device="cpu")
        dist.all_to_all_single(r, send.cpu(), output_split_sizes=recv_counts, input_split_sizes=send_counts,
                               group=group)
        recv.copy_(r)
        return recv
    dist.all_to_all_single(recv, send, output_split_sizes=recv_counts, input_split_sizes=send_counts, group=group)
    return recv


def _all_reduce(dist, t, op, group):
    if _host_staged(dist, group) and t.is_cuda:
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)


def sharded_stats9(src, dst, valid, address_space: int, ops, group=None) -> tuple:
    """Nine statistics of the matrix summed over every rank's packets.

    ``src``/``dst`` (int32 tensors holding u32 bits) are this rank's shard;
    ``ops`` provides the device stages (CudaShardOps in production)."""
    import torch
    import torch.distributed as dist

    G = dist.get_world_size(group)
    # exchange 1: packets by owner(src)
    ps, pd, c1 = ops.partition_packets(src, dst, valid, G)
    r1 = _alltoall_counts(torch, dist, c1, ops, group)
    rs = _alltoall(dist, ops, ps, c1, r1, group)
    rd = _alltoall(dist, ops, pd, c1, r1, group)
    ops.sync()
    # local links + rows, then exchange 2: column entries by owner(dst)
    row9, cd, cc, c2 = ops.rows(rs, rd, address_space, G)
    r2 = _alltoall_counts(torch, dist, c2, ops, group)
    rcd = _alltoall(dist, ops, cd, c2, r2, group)
    rcc = _alltoall(dist, ops, cc, c2, r2, group)
    ops.sync()
    col9 = ops.cols(rcd, rcc, address_space)
    mine = [int(row9[i]) for i in ROW_FIELDS] + [int(col9[i]) for i in COL_FIELDS]
    s = ops.int64_tensor([mine[i] for i in SUM_FIELDS])
    m = ops.int64_tensor([mine[i] for i in MAX_FIELDS])
    _all_reduce(dist, s, dist.ReduceOp.SUM, group)
    _all_reduce(dist, m, dist.ReduceOp.MAX, group)
    out = [0] * 9
    for i, v in zip(SUM_FIELDS, s.tolist()):
        out[i] = int(v)
    for i, v in zip(MAX_FIELDS, m.tolist()):
        out[i] = int(v)
    return tuple(out)


_OPS: dict = {}


def _cuda_ops(device: int) -> CudaShardOps:
    ops = _OPS.get(device)
    if ops is None:
        ops = _OPS[device] = CudaShardOps(device)
    return ops


def as_i32_tensor(buf, device: int):
    """View a DeviceArray (nmx_malloc) as a torch int32 CUDA tensor (no copy)."""
    import torch

    if isinstance(buf, torch.Tensor):
        return buf
    n = buf.numel()
    holder = _DeviceView(buf.data_ptr(), n, device)
    return torch.as_tensor(holder, device=f"cuda:{device}")


class _DeviceView:
    """__cuda_array_interface__ wrapper so torch can alias nmx_malloc memory."""

    def __init__(self, ptr: int, n: int, device: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i4", "data": (ptr, False), "version": 3,
                                         "strides": None}


_COMMS: dict = {}


def native_communicator(device: int, group=None):
    """libnmx's NCCL communicator for this rank of ``group`` (made once: rank 0 draws the
    id, torch.distributed broadcasts its 128 bytes -- the only use of the process group);
    None when the group's backend is not NCCL (gloo: CPU tests, several ranks on one GPU)."""
    import torch.distributed as dist

    if dist.get_backend(group) != "nccl":
        return None
    key = (device, id(group))
    comm = _COMMS.get(key)
    if comm is None:
        from . import _lib

        box = [_lib.comm_unique_id() if dist.get_rank(group) == 0 else None]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        comm = _COMMS[key] = _lib.Communicator(box[0], dist.get_world_size(group), dist.get_rank(group), device)
    return comm


def sharded_stats9_device(src, dst, address_space: int, device: int = 0, valid=None, group=None) -> tuple:
    """This rank's device shard -> the summed matrix's nine statistics. On NCCL the whole
    pipeline runs in libnmx (nmx_stats9_sharded); gloo runs the same stages with the
    exchanges in torch.distributed (host-staged)."""
    comm = native_communicator(device, group)
    if comm is not None:
        return comm.stats9(src, dst, valid, address_space)
    ops = _cuda_ops(device)
    return sharded_stats9(as_i32_tensor(src, device), as_i32_tensor(dst, device), valid, address_space, ops, group)


def sharded_stats9_host(src: np.ndarray, dst: np.ndarray, address_space: int, device: int = 0, group=None) -> tuple:
    """Host shard -> H2D -> sharded statistics (the multi-GPU e2e entry)."""
    import torch

    from ._lib import _u32_host

    comm = native_communicator(device, group)
    if comm is not None:
        return comm.stats9(src, dst, None, address_space)
    # range-checked u32 first (an int64 column reinterpreted as int32 would be two words per address)
    s = torch.from_numpy(_u32_host(src).view(np.int32)).to(f"cuda:{device}", non_blocking=True)
    d = torch.from_numpy(_u32_host(dst).view(np.int32)).to(f"cuda:{device}", non_blocking=True)
    return sharded_stats9(s, d, None, address_space, _cuda_ops(device), group)
