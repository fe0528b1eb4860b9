"""Multi-rank orchestration of paper_2510_14050_b200.distributed over gloo (CPU).

The NCCL path on GPUs runs the same `sharded_stats9` with libnmx.so device
stages; here the device stages are replaced by a numpy stand-in built on the
oracle, so the exchange logic (owner routing, count exchange, split sizes,
SUM/MAX all-reduce) is checked bit-exactly against the single-process oracle.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import netmeter_oracle as orc
from paper_2510_14050_b200 import distributed as nd
from paper_2510_14050_b200.partitioning import partition_even


class NumpyShardOps:
    """CPU stand-in for CudaShardOps (test infrastructure only)."""

    def empty(self, n):
        return torch.empty(int(n), dtype=torch.int32)

    def sync(self):
        pass

    def int64_tensor(self, values):
        return torch.tensor(list(values), dtype=torch.int64)

    @staticmethod
    def _u32(t):
        return t.numpy().view(np.uint32)

    def _route(self, key, cols, parts):
        o = nd.owner(key, parts)
        order = np.argsort(o, kind="stable")
        counts = np.bincount(o, minlength=parts).tolist()
        return [torch.from_numpy(np.ascontiguousarray(c[order]).view(np.int32)) for c in cols], counts

    def partition_packets(self, src, dst, valid, parts):
        s, d = self._u32(src), self._u32(dst)
        if valid is not None:
            keep = valid.numpy().astype(bool)
            s, d = s[keep], d[keep]
        (rs, rd), counts = self._route(s, (s, d), parts)
        return rs, rd, counts

    def rows(self, src, dst, space, parts):
        s, d = self._u32(src), self._u32(dst)
        st = np.array(orc.stats9_packed(s, d), dtype=np.int64)
        keys, counts = orc.coo_packed(s, d)
        ld = (keys & np.uint64(0xFFFFFFFF)).astype(np.uint32)
        (od, oc), c = self._route(ld, (ld, counts.astype(np.uint32)), parts)
        return st, od, oc, c

    def cols(self, dst, cnt, space):
        d, c = self._u32(dst), self._u32(cnt).astype(np.int64)
        out = np.zeros(9, dtype=np.int64)
        if len(d):
            order = np.argsort(d, kind="stable")
            sd, sc = d[order], c[order]
            starts, lens = orc._runs(sd)
            sums = np.add.reduceat(sc, starts)
            out[6], out[7], out[8] = len(starts), sums.max(), lens.max()
        return out


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cases, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        for (gen, lg, space, frac) in cases:
            g = orc.gen_uniform if gen == "uniform" else orc.gen_powerlaw
            s, d = g(3, 0, 1 << lg, space)
            valid = None
            if frac:
                valid = np.random.default_rng(9).random(len(s)) >= frac
            off, ln = partition_even(len(s), world).spans[rank]
            st = torch.from_numpy(s[off:off + ln].view(np.int32).copy())
            dt = torch.from_numpy(d[off:off + ln].view(np.int32).copy())
            vt = None if valid is None else torch.from_numpy(valid[off:off + ln].astype(np.uint8))
            out.append(nd.sharded_stats9(st, dt, vt, space, NumpyShardOps()))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


CASES = [("uniform", 14, 1 << 32, 0.0), ("powerlaw", 15, 1 << 32, 0.0), ("uniform", 13, 300, 0.3),
         ("powerlaw", 12, 1 << 10, 0.1)]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_stats_match_single_process_oracle(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, CASES, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for k, (gen, lg, space, frac) in enumerate(CASES):
        g = orc.gen_uniform if gen == "uniform" else orc.gen_powerlaw
        s, d = g(3, 0, 1 << lg, space)
        valid = None if not frac else np.random.default_rng(9).random(len(s)) >= frac
        want = orc.stats9_packed(s, d, valid)
        for r in range(world):
            assert tuple(results[r][k]) == want, (world, r, k)


def test_owner_is_balanced_and_deterministic():
    x = np.arange(1 << 16, dtype=np.uint32)
    for parts in (1, 2, 4, 8):
        o = nd.owner(x, parts)
        assert o.min() >= 0 and o.max() < parts
        c = np.bincount(o, minlength=parts)
        assert c.max() - c.min() < 0.05 * c.mean() + 2
    assert np.array_equal(nd.owner(x, 8), nd.owner(x.copy(), 8))
