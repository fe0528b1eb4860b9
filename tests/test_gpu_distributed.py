"""Device stages of the multi-GPU path on one B200.

G ranks are simulated in one process (each 'rank' runs nmx_partition_packets /
nmx_shard_rows / nmx_shard_cols; the all-to-all is done by slicing), and the
real NCCL orchestration runs as a world-size-1 process group."""

import os
import socket

import numpy as np
import pytest

from oracle import netmeter_oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    from paper_2510_14050_b200.distributed import CudaShardOps

    return CudaShardOps(0)


def _t(ops, a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).to("cuda:0")


def _simulate(ops, s, d, valid, space, G):
    from paper_2510_14050_b200 import distributed as nd
    from paper_2510_14050_b200.partitioning import partition_even

    import torch

    spans = partition_even(len(s), G).spans
    # exchange 1
    inbox = [[[], []] for _ in range(G)]
    for off, ln in spans:
        v = None if valid is None else torch.from_numpy(valid[off:off + ln].astype(np.uint8)).to("cuda:0")
        ps, pd, c = ops.partition_packets(_t(ops, s[off:off + ln]), _t(ops, d[off:off + ln]), v, G)
        at = 0
        for o in range(G):
            inbox[o][0].append(ps[at:at + c[o]])
            inbox[o][1].append(pd[at:at + c[o]])
            at += c[o]
    # rows + exchange 2
    rows, inbox2 = [], [[[], []] for _ in range(G)]
    for o in range(G):
        rs, rd = torch.cat(inbox[o][0]), torch.cat(inbox[o][1])
        st, cd, cc, c = ops.rows(rs, rd, space, G)
        rows.append(st)
        at = 0
        for q in range(G):
            inbox2[q][0].append(cd[at:at + c[q]])
            inbox2[q][1].append(cc[at:at + c[q]])
            at += c[q]
    cols = [ops.cols(torch.cat(inbox2[q][0]), torch.cat(inbox2[q][1]), space) for q in range(G)]
    out = [0] * 9
    for i in nd.SUM_FIELDS:
        out[i] = int(sum((rows[r] if i < 6 else cols[r])[i] for r in range(G)))
    for i in nd.MAX_FIELDS:
        out[i] = int(max((rows[r] if i < 6 else cols[r])[i] for r in range(G)))
    return tuple(out)


@pytest.mark.parametrize("G", [1, 2, 3, 8])
@pytest.mark.parametrize("kind", ["uniform", "powerlaw"])
def test_simulated_ranks_match_oracle(ops, G, kind):
    gen = orc.gen_uniform if kind == "uniform" else orc.gen_powerlaw
    for lg, space, frac in ((18, 1 << 32, 0.0), (16, 5000, 0.25)):
        s, d = gen(21, 0, 1 << lg, space)
        valid = None if not frac else np.random.default_rng(2).random(len(s)) >= frac
        assert _simulate(ops, s, d, valid, space, G) == orc.stats9_packed(s, d, valid), (G, kind, lg)


@pytest.mark.parametrize("G", [1, 2, 3])
@pytest.mark.parametrize("kind", ["uniform", "powerlaw"])
def test_simulated_ranks_msd_sizes(ops, G, kind):
    # >= 2^20 packets per rank: the shard stages take the MSD path (rows with
    # heavy buckets, column slots with holes partitioned by owner(dst))
    gen = orc.gen_uniform if kind == "uniform" else orc.gen_powerlaw
    s, d = gen(23, 0, (1 << 22) + 7, 1 << 32)
    valid = np.random.default_rng(3).random(len(s)) >= 0.1
    assert _simulate(ops, s, d, valid, 1 << 32, G) == orc.stats9_packed(s, d, valid), (G, kind)


def test_nccl_world_of_one():
    import torch
    import torch.distributed as dist

    from paper_2510_14050_b200 import _lib
    from paper_2510_14050_b200 import distributed as nd

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n = 1 << 20
        ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
        _lib.generate(_lib.GEN_POWERLAW, 4, 0, n, 1 << 32, ds, dd)
        got = nd.sharded_stats9_device(ds, dd, 1 << 32)
        assert got == orc.stats9_packed(ds.download(), dd.download())
        hs, hd = ds.download(), dd.download()
        assert nd.sharded_stats9_host(hs, hd, 1 << 32) == got
        # the NCCL group ran libnmx's own communicator, not the torch exchanges
        comm = nd.native_communicator(0)
        assert comm is not None and comm.last_exchange() == (8 * n, 8 * got[1])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("lg,space,kind", [(0, 1 << 32, "uniform"), (12, 7, "uniform"), (18, 5000, "powerlaw"),
                                           (21, 1 << 32, "powerlaw"), (22, 1 << 32, "uniform")])
def test_native_communicator_world_of_one(lg, space, kind):
    """nmx_comm without torch.distributed: id -> nmx_comm_init -> nmx_stats9_sharded[_host]
    (grouped ncclSend / ncclRecv to itself, ncclAllGather, ncclAllReduce) equals the oracle,
    invalid packets included."""
    from paper_2510_14050_b200 import _lib

    comm = _lib.Communicator(_lib.comm_unique_id(), 1, 0, device=0)
    try:
        n = (1 << lg) if lg else 0
        g = orc.gen_uniform if kind == "uniform" else orc.gen_powerlaw
        s, d = g(21, 0, n, space)
        v = np.random.default_rng(lg).random(n) >= 0.2
        want = orc.stats9_packed(s, d, v)
        assert comm.stats9(s, d, v, space) == want
        if n:
            ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
            ds.upload(s)
            dd.upload(d)
            assert comm.stats9(ds, dd, None, space) == orc.stats9_packed(s, d)
        if n and space < (1 << 32):  # addresses beyond the address space are rejected, not packed
            with pytest.raises(Exception, match="address"):
                comm.stats9(s, d + np.uint32(space), None, space)
    finally:
        comm.close()


def _gpu_worker(rank, world, port, cases, q):
    import torch
    import torch.distributed as dist

    from paper_2510_14050_b200 import distributed as nd
    from paper_2510_14050_b200.partitioning import partition_even

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = []
        for (gen, lg, space) in cases:
            g = orc.gen_uniform if gen == "uniform" else orc.gen_powerlaw
            s, d = g(5, 0, 1 << lg, space)
            off, ln = partition_even(len(s), world).spans[rank]
            st = torch.from_numpy(s[off:off + ln].view(np.int32).copy()).to("cuda:0")
            dt = torch.from_numpy(d[off:off + ln].view(np.int32).copy()).to("cuda:0")
            out.append(nd.sharded_stats9_device(st, dt, space, device=0))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_multi_process_device_stages(world):
    # every rank a real process running the libnmx shard stages on the one GPU; the
    # exchanges go through gloo staged on the host (NCCL in production): the same
    # orchestration bench.py runs under torchrun, MSD-sized shards included
    import multiprocessing as mp

    cases = [("uniform", 21, 1 << 32), ("powerlaw", 22, 1 << 32), ("powerlaw", 20, 1 << 16)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, cases, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for k, (gen, lg, space) in enumerate(cases):
        g = orc.gen_uniform if gen == "uniform" else orc.gen_powerlaw
        s, d = g(5, 0, 1 << lg, space)
        want = orc.stats9_packed(s, d)
        for r in range(world):
            assert tuple(results[r][k]) == want, (world, r, k)


def test_bench_spawns_ranks():
    """`bench.py --gpus 2` launches its own two ranks (torch.distributed.run) without an
    external torchrun; with both ranks pinned to the one GPU and gloo staging the
    exchanges, the printed line has n_gpus == 2 and the one-GPU statistics."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    from paper_2510_14050_b200 import _lib

    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, NMX_BENCH_DEVICE="0", NMX_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--steps", "1", "--warmup", "3",
                        "--log2n", "22", "--no-cpu", "--no-e2e"], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    n = 1 << 22
    ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
    try:
        _lib.generate(_lib.GEN_UNIFORM, 7, 0, n, 1 << 32, ds, dd)
        assert line["stats9"] == list(_lib.stats9(ds, dd, None, 1 << 32))
    finally:
        ds.close()
        dd.close()


def test_bench_cfg5_sharded_ranks():
    """`bench.py --config cfg5 --gpus 2`: each rank's partition_even share in pinned host
    memory through the sharded host entry; the statistics equal one device's."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    from paper_2510_14050_b200 import _lib

    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, NMX_BENCH_DEVICE="0", NMX_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--config", "cfg5", "--gpus", "2", "--steps", "1",
                        "--warmup", "3", "--log2n", "23"], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    n = 1 << 23
    ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
    try:
        _lib.generate(_lib.GEN_UNIFORM, 7, 0, n, 1 << 32, ds, dd)
        assert line["stats9"] == list(_lib.stats9(ds, dd, None, 1 << 32))
    finally:
        ds.close()
        dd.close()
