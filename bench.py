"""Benchmark: packets/s for traffic-matrix build + 9 statistics (BASELINE.json metric).

Workload (N=1): BASELINE config 3 -- 2^30 packets uniform over the 2^32 address
space (splitmix64 generator), summed into one hypersparse
traffic matrix, nine Graph Challenge statistics. One step = one full pass of
the hot path (ingest -> onesweep sort -> unique links/rows -> column sort ->
columns -> 9 int64 to host) over the whole batch.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl nmx|reference]
                  [--config cfg3|cfg4|cfg2|cfg1] [--log2n L]

N > 1 runs one rank per GPU: under torchrun (the driver's launch) it uses the
ranks torchrun made; `python bench.py --gpus N` without torchrun re-launches
itself under `torch.distributed.run --nproc-per-node N`. The 2^30 packets are
sharded across ranks and exchanged by owner(src) / owner(dst) over NCCL
(paper_2510_14050_b200/distributed.py), total work fixed -> "scaling": "strong".

`--impl reference` times the reference's own CPU path -- the unmodified
`netmeter` package installed in baseline/_ref (build_matrices -> to_flat ->
analyze_matrix + 3 x max_scan with make_group_scheduler(1, os.cpu_count())) --
on the host cores, rank 0 only, on a bounded sample of the same workload per
step (ids compacted outside the timed region: the reference rejects dim > 2^31).
Without baseline/_ref it falls back to the numpy port in oracle/ (kind "port").
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "packets/sec for traffic-matrix build + 9 stats at 1/2/4/8 B200; % HBM roofline"
CONFIGS = {
    # name: (log2 n, address space, generator)
    "cfg3": (30, 1 << 32, "uniform"),
    "cfg4": (30, 1 << 32, "powerlaw"),
    "cfg2": (23, 1 << 24, "uniform"),
    "cfg1": (17, 1 << 18, "uniform"),
    # config 5: 2^32 packets streamed from pinned host buffers in 2^28-packet windows;
    # one B200 takes them through the out-of-core source/destination part split
    # (nmx_stream_stats9 above 2^31 packets), N ranks take 2^32 / N each
    "cfg5": (32, 1 << 32, "uniform"),
    # 9-byte packet-file records (traffic.py:25) in pinned host
    # memory, streamed raw and unpacked on the GPU (nmx_stream_records)
    "file": (29, 1 << 32, "uniform"),
    # anonymize (traffic.py:107-137) of a cfg2-sized stream
    "anon": (23, 1 << 32, "uniform"),
    # `netmeter analyze` of a generated text dataset (CLI defaults:
    # address space 2^16, 2^17-packet windows -> 8 files at 2^20 packets)
    "cli": (20, 1 << 16, "uniform"),
}


def _traffic(kernel: str, items_per_launch: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the kernel class, from
    the committed ncu capture (profiles/traffic_latest.json, tools/ncu_traffic.py), scaled
    from the captured call's items per launch to this one's; None if absent."""
    try:
        t = json.loads((ROOT / "profiles" / "traffic_latest.json").read_text())
    except Exception:
        return None
    ks = [v for k, v in t["kernels"].items() if kernel and kernel in k]
    if not ks:
        return None
    per_item = sum(v["dram_bytes"] for v in ks) / sum(v["launches"] for v in ks) / t["items_per_launch"]
    return round(per_item * items_per_launch)


def _per_launch(totals, peak_gbs):
    """The dominant class launch by launch, averaged over the timed steps: CUDA-event
    ms, algorithmic bytes, GB/s and fraction of the HBM peak (nmx_last_kernel_launches)."""
    runs = [t.get("dom_per_launch") or [] for t in totals]
    if not runs or any(len(r) != len(runs[0]) for r in runs):
        return None
    out = []
    for i in range(len(runs[0])):
        ms = sum(r[i][0] for r in runs) / len(runs)
        by = runs[0][i][1]
        gbs = by / (ms / 1e3) / 1e9 if ms else 0.0
        out.append({"ms": round(ms, 4), "bytes": by, "gbs": round(gbs, 1), "frac": round(gbs / peak_gbs, 4)})
    return out


def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            # the timed region can be shorter than nvidia-smi's start-up: wait for its first sample
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5 and self.proc.poll() is None:
                time.sleep(0.01)
            self.lines.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self.post = False
        if self.proc and not self.lines:
            # a region shorter than the 20 ms sampling period: report the sample taken
            # right after it (flagged) rather than none
            t0 = time.time()
            while not self.lines and time.time() - t0 < 1 and self.proc.poll() is None:
                time.sleep(0.005)
            self.post = bool(self.lines)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower() in ("active", "1", "yes"):
                    reasons.add(nm)
        out = {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
               "reasons": sorted(reasons), "samples": len(sm)}
        if getattr(self, "post", False):
            out["sampled"] = "right after the timed region (shorter than the 20 ms sampling period)"
        return out


def host_info() -> dict:
    """Host cores and RAM of the box the CPU legs run on."""
    ram = None
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemTotal:"):
                ram = round(int(ln.split()[1]) / 2**20, 1)
    except OSError:
        pass
    return {"os_cpu_count": os.cpu_count(), "ram_gib": ram}


def _sample_packets(config: str, log2n: int, space: int, gen: str):
    """The CPU legs' input sample (prepared outside the timed region): cfg1 / cfg2 are
    generate_packets + anonymize (BASELINE configs 1-2; anonymized ids are already
    dense), the splitmix64 configs are compacted with np.unique(return_inverse)
    because the reference rejects dim > 2^31 (traffic.py:203-204)."""
    import numpy as np

    from oracle import netmeter_oracle as orc

    if config in ("cfg1", "cfg2"):
        seed = 1 if config == "cfg1" else 2
        s, d, _ = orc.generate_packets(1 << log2n, 1 << 32, seed)
        return orc.anonymize(s, d, seed)
    g = orc.gen_uniform if gen == "uniform" else orc.gen_powerlaw
    s, d = g(7, 0, 1 << log2n, space)
    return orc.compact_ids(s, d)


def _reference_pkg():
    """The unmodified reference package from baseline/_ref (None if not installed)."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "netmeter").is_dir():
        return None
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import netmeter
    from netmeter import analytics, resources, traffic

    return netmeter, traffic, analytics, resources


def cpu_reference_rate(config: str, log2n: int, space: int, gen: str, reps: int = 1):
    """The reference's own path on a bounded sample: PacketStream -> build_matrices(stream,
    len) -> to_flat -> analyze_matrix + max_scan over weights / row_sums[:,1] /
    col_sums[:,1] (traffic.py:221-292, analytics.py:89-106) with
    make_group_scheduler(1, os.cpu_count()) (resources.py:139-159).
    Returns (packets/s, best seconds, stats9, kind, cores)."""
    import numpy as np

    s, d, dim = _sample_packets(config, log2n, space, gen)
    pkg = _reference_pkg()
    n = len(s)
    if pkg is None:  # numpy port fallback
        from oracle import netmeter_oracle as orc

        valid = np.ones(n, dtype=bool)
        best, st = None, None
        for _ in range(reps):
            t0 = time.perf_counter()
            st = orc.ref_stats9(s, d, valid, dim)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        return n / best, best, st, "port", 1
    _, traffic, analytics, resources = pkg
    cores = os.cpu_count() or 1
    stream = traffic.PacketStream(s, d, np.ones(n, dtype=bool), dim)
    best, st = None, None
    with resources.make_group_scheduler(1, cores) as sched:
        for _ in range(reps):
            t0 = time.perf_counter()
            (m,) = traffic.build_matrices(stream, window_size=n)
            flat = traffic.to_flat(m)
            r = analytics.analyze_matrix(flat, sched)
            mx_link = analytics.max_scan(flat.weights, sched)
            mx_src = analytics.max_scan(flat.row_sums[:, 1] if len(flat.row_sums) else [], sched)
            mx_dst = analytics.max_scan(flat.col_sums[:, 1] if len(flat.col_sums) else [], sched)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
            st = (r.valid_packets, r.unique_links, mx_link, r.unique_sources, mx_src, r.max_fanout,
                  r.unique_destinations, mx_dst, r.max_fanin)
    return n / best, best, st, "reference", cores


def _cpu_sample_desc(config, sample, kind, cores, secs=None, reps=None):
    what = ("baseline/_ref netmeter (the unmodified reference): build_matrices -> to_flat -> analyze_matrix "
            f"+ 3 x max_scan, make_group_scheduler(1, {cores}); numpy's unique/sort/bincount run on one core, "
            "the reductions on the pool" if kind == "reference" else
            "oracle/netmeter_oracle.py ref_stats9 (numpy port of traffic.py:197-292 + analytics.py:95-106)")
    inp = ("generate_packets + anonymize (BASELINE input)" if config in ("cfg1", "cfg2") else
           "the same generator, ids compacted outside the timed region")
    t = f", best of {reps} ({secs:.2f} s each)" if secs is not None else ""
    return f"2^{sample} packets per step, {inp}{t}; {what}"


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    log2n, space, gen = CONFIGS[args.config]
    if args.log2n:
        log2n = args.log2n
    sample = min(log2n, args.ref_log2n)
    for _ in range(args.warmup):
        cpu_reference_rate(args.config, sample, space, gen)
    rates = []
    t0 = time.perf_counter()
    kind, cores = "port", 1
    for _ in range(args.steps):
        r, _, _, kind, cores = cpu_reference_rate(args.config, sample, space, gen)
        rates.append(r)
    wall = time.perf_counter() - t0
    value = statistics.median(rates)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "packets/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": f"{args.config}: 2^{log2n} packets {gen} over {space} addresses, summed matrix, 9 stats",
                   "sample": f"2^{sample} packets of the same workload per step"},
        "cpu_baseline": {"value": value, "unit": "packets/s", "cores": cores, "kind": kind,
                         "sample": _cpu_sample_desc(args.config, sample, kind, cores), "host": host_info()},
        "e2e": {"value": value, "unit": "packets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_cfg5(args) -> None:
    """Streamed windows (pinned host -> device, overlapped) + merge-add; rank 0 only."""
    import numpy as np

    from paper_2510_14050_b200 import _lib
    from paper_2510_14050_b200 import coo as nc

    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        return run_cfg5_sharded(args)
    log2n, space, gen = CONFIGS["cfg5"]
    if args.log2n:
        log2n = args.log2n
    w = 1 << min(28, log2n)
    nwin = (1 << log2n) // w
    kind = _lib.GEN_UNIFORM if gen == "uniform" else _lib.GEN_POWERLAW
    ds, dd = _lib.DeviceArray(w), _lib.DeviceArray(w)
    wins = []
    for k in range(nwin):  # inputs prepared outside the timed region
        _lib.generate(kind, 7, k * w, w, space, ds, dd)
        ps, pd = _lib.PinnedArray(w), _lib.PinnedArray(w)
        ps.array[:] = ds.download()
        pd.array[:] = dd.download()
        wins.append((ps, pd))
    ds.close()
    dd.close()
    views = [(a.array, b.array) for a, b in wins]
    for _ in range(max(1, min(args.warmup, 1))):
        stats = nc.stream_stats9_pinned(views)
    times = []
    with ClockSampler(0) as clk:
        for _ in range(args.steps):
            t0 = time.perf_counter()
            stats = nc.stream_stats9_pinned(views)
            times.append(time.perf_counter() - t0)
    best = min(times)
    n_total = nwin * w
    parity = golden_parity("cfg5", log2n, gen, stats)
    print(json.dumps({
        "metric": METRIC, "value": n_total / best, "unit": "packets/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": best * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"cfg5: {nwin} windows x 2^{int(np.log2(w))} packets {gen} streamed from pinned host "
                               "memory (nmx_stream_stats9: the H2D of window t+1 on a copy stream overlaps the "
                               "device work of window t; up to 2^31 packets the windows' level-1 partitions form "
                               "one device-resident running sum, above it every window is split on arrival into "
                               "owner(src) part arenas, each part's rows and each owner(dst) column part run in "
                               "turn)", "packets": n_total,
                   "timing": "wall clock of the host call (it is host-synchronous), best of steps"},
        "stats9": list(stats),
        "parity": parity,
        "e2e": {"value": n_total / best, "unit": "packets/s", "h2d_bytes_per_step": 8 * n_total,
                "d2h_bytes_per_step": 72},
        "clocks": clk.summary(),
    }), flush=True)
    for a, b in wins:
        a.close()
        b.close()


def run_cfg5_sharded(args) -> None:
    """cfg5 on N ranks: each rank holds its partition_even share of the 2^32 packets in
    pinned host memory and calls the sharded host entry (nmx_stats9_sharded_host: H2D,
    owner(src) / owner(dst) exchanges over libnmx's NCCL communicator, SUM / MAX);
    timed on the host around the call between barriers, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2510_14050_b200 import _lib
    from paper_2510_14050_b200 import distributed as nd

    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    local = int(os.environ.get("NMX_BENCH_DEVICE", os.environ.get("LOCAL_RANK", "0")))
    backend = os.environ.get("NMX_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local)
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    log2n, space, gen = CONFIGS["cfg5"]
    if args.log2n:
        log2n = args.log2n
    n_total = 1 << log2n
    q, r = divmod(n_total, world)
    n = q + (1 if rank < r else 0)
    off = rank * q + min(rank, r)
    kind = _lib.GEN_UNIFORM if gen == "uniform" else _lib.GEN_POWERLAW
    hs, hd = _lib.PinnedArray(n), _lib.PinnedArray(n)
    chunk = 1 << 26
    ds, dd = _lib.DeviceArray(min(n, chunk), device=local), _lib.DeviceArray(min(n, chunk), device=local)
    for lo in range(0, n, chunk):  # inputs prepared outside the timed region
        ln = min(chunk, n - lo)
        _lib.generate(kind, 7, off + lo, ln, space, ds, dd, device=local)
        hs.array[lo:lo + ln] = ds.download()[:ln]
        hd.array[lo:lo + ln] = dd.download()[:ln]
    ds.close()
    dd.close()

    def step():
        return nd.sharded_stats9_host(hs.array, hd.array, space, device=local)

    for _ in range(max(1, min(args.warmup, 1))):
        stats = step()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            dist.barrier()
            t0 = time.perf_counter()
            stats = step()
            times.append(time.perf_counter() - t0)
    mt = torch.tensor([min(times)], dtype=torch.float64, device=f"cuda:{local}" if backend == "nccl" else "cpu")
    dist.all_reduce(mt, op=dist.ReduceOp.MAX)
    best = float(mt.item())
    parity = golden_parity("cfg5", log2n, gen, stats)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": n_total / best, "unit": "packets/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": best * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": {"workload": f"cfg5: 2^{log2n} packets {gen} over {space} addresses in pinned host memory, "
                                   f"partition_even shares of {world} ranks, each through nmx_stats9_sharded_host "
                                   "(H2D, NCCL owner(src) / owner(dst) exchanges, SUM / MAX)",
                       "packets": n_total, "parallelism": f"shards{world}",
                       "timing": "host wall clock of the call between barriers, best of steps, max over ranks"},
            "stats9": list(stats), "parity": parity,
            "e2e": {"value": n_total / best, "unit": "packets/s", "h2d_bytes_per_step": 8 * n_total,
                    "d2h_bytes_per_step": 72 * world},
            "clocks": clk.summary(),
        }), flush=True)
    dist.barrier()
    dist.destroy_process_group()
    hs.close()
    hd.close()


def run_file(args) -> None:
    """Packet-file records (9 B/packet) in pinned host memory -> nine statistics; rank 0 only."""
    import numpy as np

    from paper_2510_14050_b200 import _lib

    if int(os.environ.get("RANK", "0")) != 0:
        return
    log2n, space, gen = CONFIGS["file"]
    if args.log2n:
        log2n = args.log2n
    n = 1 << log2n
    w = 1 << min(25, log2n)
    kind = _lib.GEN_UNIFORM if gen == "uniform" else _lib.GEN_POWERLAW
    rec = _lib.PinnedArray(9 * n, dtype=np.uint8)  # the file image, prepared outside the timed region
    view = rec.array.view(np.dtype([("src", "<u4"), ("dst", "<u4"), ("valid", "u1")]))
    ds, dd = _lib.DeviceArray(w), _lib.DeviceArray(w)
    for k in range(n // w):
        _lib.generate(kind, 7, k * w, w, space, ds, dd)
        view["src"][k * w:(k + 1) * w] = ds.download()
        view["dst"][k * w:(k + 1) * w] = dd.download()
    view["valid"][:] = 1
    ds.close()
    dd.close()
    windows = [rec.array[i:i + 9 * w] for i in range(0, 9 * n, 9 * w)]
    stats = _lib.stream_records(windows, space)
    times = []
    with ClockSampler(0) as clk:
        for _ in range(args.steps):
            t0 = time.perf_counter()
            stats = _lib.stream_records(windows, space)
            times.append(time.perf_counter() - t0)
    best = min(times)
    print(json.dumps({
        "metric": METRIC, "value": n / best, "unit": "packets/s", "n_gpus": 1, "steps": args.steps,
        "warmup": 1, "ms_per_step": best * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"file: 2^{log2n} packets as 9-byte packet-file records (traffic.py:25) in pinned host "
                               f"memory, {n // w} windows of 2^{int(np.log2(w))} streamed raw (9 B/packet H2D on a "
                               "copy stream), unpacked on the GPU, summed matrix, 9 statistics (nmx_stream_records)",
                   "packets": n, "timing": "wall clock of the host call (host-synchronous), best of steps"},
        "stats9": list(stats),
        "e2e": {"value": n / best, "unit": "packets/s", "h2d_bytes_per_step": 9 * n, "d2h_bytes_per_step": 72},
        "clocks": clk.summary(),
    }), flush=True)
    rec.close()


def run_anon(args) -> None:
    """anonymize (traffic.py:107-137) on the GPU vs the numpy restatement; rank 0 only."""
    import numpy as np

    from oracle import netmeter_oracle as orc
    from paper_2510_14050_b200 import _lib

    if int(os.environ.get("RANK", "0")) != 0:
        return
    log2n, space, gen = CONFIGS["anon"]
    if args.log2n:
        log2n = args.log2n
    n = 1 << log2n
    src, dst = (orc.gen_uniform if gen == "uniform" else orc.gen_powerlaw)(3, 0, n, space)
    ds, dd = _lib.DeviceArray(n), _lib.DeviceArray(n)
    ds.upload(src)
    dd.upload(dst)
    dev_t, host_t = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        so, do, k, _, _ = _lib.anonymize_device(ds, dd, 17, tables=False)  # device in, device out
        t1 = time.perf_counter()
        so.close(); do.close()
        so, do, k, dist, code = _lib.anonymize_device(src, dst, 17)  # host in, host out (+ tables)
        s_out, d_out = so.download(), do.download()
        t2 = time.perf_counter()
        so.close(); do.close()
        if i >= args.warmup:
            dev_t.append(t1 - t0)
            host_t.append(t2 - t1)
    t0 = time.perf_counter()
    rs, rd, rk = orc.anonymize(src.astype(np.int64), dst.astype(np.int64), 17)
    cpu = time.perf_counter() - t0
    assert k == rk and np.array_equal(s_out, rs) and np.array_equal(d_out, rd)
    print(json.dumps({
        "metric": "packets/sec for anonymize (traffic.py:107-137)", "value": n / min(dev_t), "unit": "packets/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": min(dev_t) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": f"anon: anonymize 2^{log2n} {gen} packets over {space} addresses, key 17; value = "
                               "device columns in/out incl. the host permutation draw (numpy default_rng(key)."
                               "permutation(k), the reference's own RNG); e2e = host arrays in, host arrays + "
                               "distinct/code tables out", "packets": n, "distinct": k,
                   "timing": "wall clock of the host calls, best of steps"},
        "e2e": {"value": n / min(host_t), "unit": "packets/s", "h2d_bytes_per_step": 8 * n + 4 * k,
                "d2h_bytes_per_step": 8 * n + 8 * k},
        "cpu_baseline": {"value": n / cpu, "unit": "packets/s", "cores": 1, "kind": "port",
                         "sample": f"the same 2^{log2n} packets through oracle/netmeter_oracle.py anonymize "
                                   "(numpy restatement of traffic.py:107-137 without its Python dict)"},
    }), flush=True)


def run_cli(args) -> None:
    """CLI analyze end to end (text files -> reports) vs the reference's per-line parse; rank 0 only."""
    import tempfile

    from oracle import netmeter_oracle as orc
    from paper_2510_14050_b200 import cli

    if int(os.environ.get("RANK", "0")) != 0:
        return
    log2n, space, _ = CONFIGS["cli"]
    if args.log2n:
        log2n = args.log2n
    n = 1 << log2n
    with tempfile.TemporaryDirectory() as d:
        manifest = cli.cmd_generate(n=n, address_space=space, seed=1, window_size=cli.DEFAULT_WINDOW, out_dir=d)
        for _ in range(args.warmup):
            cli.run_cell(d, 1, None, 1)
        runs = [cli.run_cell(d, 1, None, 1) for _ in range(args.steps)]
        best_e2e = min(r[2].end_to_end_time for r in runs)
        best_an = min(r[2].analysis_time for r in runs)
        totals = runs[0][1]
        t0 = time.perf_counter()
        ref = []
        for name in manifest["files"]:
            dim, rp, ci, va = orc.ref_read_matrix(os.path.join(d, name))
            ref.append(orc.ref_analyze_flat(orc.ref_to_flat(rp, ci, va, dim)))
        cpu = time.perf_counter() - t0
        assert sum(r[0] for r in ref) == totals.valid_packets
        nbytes = sum(os.path.getsize(os.path.join(d, f)) for f in manifest["files"])
    print(json.dumps({
        "metric": "packets/sec end to end of `netmeter analyze` (cli.py:105-136)", "value": n / best_e2e,
        "unit": "packets/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": best_e2e * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": f"cli: analyze {manifest['window_count']} text matrix files ({nbytes} bytes) of "
                               f"2^{log2n} packets generated by `generate` (address space {space}, window 2^17): "
                               "files tokenised and validated on the GPU into device COO matrices, per-window "
                               "statistics on the device", "packets": n, "analysis_ms": best_an * 1e3,
                   "timing": "wall clock: load + containers + analysis (the reference's end-to-end clock)"},
        "e2e": {"value": n / best_e2e, "unit": "packets/s", "h2d_bytes_per_step": nbytes,
                "d2h_bytes_per_step": 72 * manifest["window_count"]},
        "cpu_baseline": {"value": n / cpu, "unit": "packets/s", "cores": 1, "kind": "port",
                         "sample": "the same files through oracle ref_read_matrix (the reference's per-line parse) "
                                   "+ ref_to_flat + ref_analyze_flat"},
    }), flush=True)


def golden_parity(config: str, log2n: int, gen: str, stats) -> dict:
    """The printed stats9 against the committed goldens: tests/golden/full_size.json
    (bounded-RAM chunked CPU oracle, oracle/make_full_size.py) for the splitmix64
    configs, tests/golden/golden.json (made by the reference package itself) for the
    generate_packets + anonymize configs 1-2."""
    try:
        if gen in ("uniform", "powerlaw"):
            g = json.loads((ROOT / "tests" / "golden" / "full_size.json").read_text())["cases"]
            name = {(30, "uniform"): "cfg3_seed7", (30, "powerlaw"): "cfg4_seed7", (31, "uniform"): "cfg5_2^31_seed7",
                    (32, "uniform"): "cfg5_2^32_seed7", (32, "powerlaw"): "cfg5pl_2^32_seed7"}.get((log2n, gen))
            src = "tests/golden/full_size.json (oracle/nmx_oracle.c chunked CPU oracle)"
        else:
            g = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())["cases"]
            name = config
            src = "tests/golden/golden.json (the reference netmeter package's own output)"
        if name is None or name not in g:
            return {"golden": None}
        want = list(g[name]["stats9"])
        return {"golden": f"{src}: {name}", "equal": list(stats) == want, "want": want}
    except (OSError, KeyError, ValueError):
        return {"golden": None}


def _step_traffic(config: str, n_total: int, world: int):
    """Measured DRAM bytes of one hot-path call from profiles/traffic_<config>.json."""
    if world != 1:
        return None
    try:
        t = json.loads((ROOT / "profiles" / f"traffic_{config}.json").read_text())
    except Exception:
        return None
    if t.get("items_per_launch") != n_total or not t.get("calls"):
        return None
    return {"bytes": round(sum(v["dram_bytes"] for v in t["kernels"].values()) / t["calls"]),
            "source": f"profiles/traffic_{config}.json ({t.get('report', '')}, {t['calls']} call(s))"}


def run_nmx(args) -> None:
    import torch

    from paper_2510_14050_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # validation of the multi-rank flow on a one-GPU box: NMX_BENCH_DEVICE pins every
    # rank to one device and NMX_DIST_BACKEND=gloo stages the exchanges through the host
    # (numbers from such a run are not scaling measurements)
    backend = os.environ.get("NMX_DIST_BACKEND", "nccl")
    if "NMX_BENCH_DEVICE" in os.environ:
        local = int(os.environ["NMX_BENCH_DEVICE"])
    log2n, space, gen = CONFIGS[args.config]
    if args.log2n:
        log2n = args.log2n
    n_total = 1 << log2n
    kind = _lib.GEN_UNIFORM if gen == "uniform" else _lib.GEN_POWERLAW
    if local >= torch.cuda.device_count():
        sys.exit(f"bench: rank {rank} wants cuda:{local} but only {torch.cuda.device_count()} GPU(s) are visible "
                 "(NMX_BENCH_DEVICE=0 NMX_DIST_BACKEND=gloo pins every rank to one GPU for a functional run)")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines: every rank's device on record
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    ctx = _lib.context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))

    # this rank's contiguous shard of the packet stream (partition_even rule)
    base, rem = divmod(n_total, world)
    n = base + (1 if rank < rem else 0)
    off = rank * base + min(rank, rem)
    ds, dd = _lib.DeviceArray(n, device=local), _lib.DeviceArray(n, device=local)
    if args.config in ("cfg1", "cfg2") and not args.log2n:
        # BASELINE configs 1-2: generate_packets(n, 2^32, seed) -> anonymize(key=seed) through
        # the package's own API (the anonymize runs on the GPU), outside the timed region
        from paper_2510_14050_b200 import traffic as nt

        seed = 1 if args.config == "cfg1" else 2
        st, _ = nt.anonymize(nt.generate_packets(n_total, 1 << 32, seed), key=seed)
        space = st.address_space
        ws, wd, _ = st.wire()
        ds.upload(ws[off:off + n])
        dd.upload(wd[off:off + n])
        gen = "generate_packets + anonymize"
    else:
        _lib.generate(kind, 7, off, n, space, ds, dd, device=local)  # this rank's shard, chunk-addressable

    if world > 1:
        from paper_2510_14050_b200 import distributed as nd

        def step():
            return nd.sharded_stats9_device(ds, dd, space, device=local)
    else:
        def step():
            return _lib.stats9(ds, dd, None, space, device=local)

    for _ in range(args.warmup):
        stats = step()
    timing_last = ctx.last_timing()

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(local)

    # ---- device-resident timed region (value) ----
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dom_ms, dom_launch, dom_bytes, launches, totals = 0.0, 0, 0, 0, []
    barrier()
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            stats = step()
            t = ctx.last_timing()
            dom_ms += t["dom_ms"]
            dom_launch += t["dom_launches"]
            dom_bytes += t["dom_bytes"]
            launches += t["kernel_launches"]
            totals.append(t)
        e1.record(stream)
        barrier()
    ms = e0.elapsed_time(e1)
    if dist is not None:
        mt = torch.tensor([ms], device=f"cuda:{local}" if backend == "nccl" else "cpu")
        dist.all_reduce(mt, op=dist.ReduceOp.MAX)
        ms = float(mt.item())
    ms_per_step = ms / args.steps
    value = n_total / (ms_per_step / 1e3)

    # ---- end-to-end through the public C-ABI host entry (pinned host buffers) ----
    e2e = None
    if not args.no_e2e:
        hs, hd = _lib.PinnedArray(n), _lib.PinnedArray(n)
        hs.array[:] = ds.download()
        hd.array[:] = dd.download()
        if world > 1:
            from paper_2510_14050_b200 import distributed as nd

            def hstep():
                return nd.sharded_stats9_host(hs.array, hd.array, space, device=local)
        else:
            def hstep():
                return _lib.stats9(hs.array, hd.array, None, space, device=local)
        hstats = hstep()
        assert hstats == stats, (hstats, stats)
        barrier()
        t0 = time.perf_counter()
        e0.record(stream)
        for _ in range(args.e2e_steps):
            hstep()
        e1.record(stream)
        barrier()
        ems = e0.elapsed_time(e1) / args.e2e_steps
        if dist is not None:
            mt = torch.tensor([ems], device=f"cuda:{local}" if backend == "nccl" else "cpu")
            dist.all_reduce(mt, op=dist.ReduceOp.MAX)
            ems = float(mt.item())
        single = {"value": n_total / (ems / 1e3), "unit": "packets/s", "h2d_bytes_per_step": 8 * n_total,
                  "d2h_bytes_per_step": 72 * world, "ms_per_step": ems, "steps": args.e2e_steps,
                  "api": ("nmx_stats9_sharded_host (include/nmx.h, libnmx's NCCL communicator) via "
                          "paper_2510_14050_b200.distributed.sharded_stats9_host" if world > 1 and backend == "nccl"
                          else "nmx_stats9_host (include/nmx.h) via paper_2510_14050_b200._lib.stats9") +
                         ", pinned host buffers, one call per step (copy, then device work)"}
        e2e = single
        nbatch = max(2, args.steps)
        if world == 1:
            # a run of K batches through nmx_stats9_host_batches: every step's H2D copy (8 B /
            # packet from pinned memory) and its 72-byte result read-back stay inside the
            # timed region; batch k+1's copy overlaps batch k's device work
            batches = [(hs.array, hd.array)] * nbatch
            got = _lib.stats9_batches(batches[:1], space, device=local)
            assert got == [tuple(stats)], (got, stats)
            barrier()
            e0.record(stream)
            res = _lib.stats9_batches(batches, space, device=local)
            e1.record(stream)
            barrier()
            assert all(r == tuple(stats) for r in res), res
            bms = e0.elapsed_time(e1) / nbatch
            e2e = {"value": n_total / (bms / 1e3), "unit": "packets/s", "h2d_bytes_per_step": 8 * n_total,
                   "d2h_bytes_per_step": 72, "ms_per_step": bms, "steps": nbatch,
                   "api": "nmx_stats9_host_batches (include/nmx.h) via paper_2510_14050_b200._lib.stats9_batches: "
                          f"{nbatch} independent 2^{log2n}-packet batches (one per timed step) from pinned host buffers in one "
                          "call; batch k+1's H2D copy overlaps batch k's device work",
                   "single_call": single}
        hs.close()
        hd.close()

    # ---- the drop-in API end to end: analytics.stats9(PacketStream) on the reference's
    # own int64 columns (host memory, not pinned), the call a netmeter user makes ----
    dropin = None
    if not args.no_e2e and world == 1 and args.config in ("cfg3", "cfg4"):
        import numpy as np

        from paper_2510_14050_b200 import analytics as na
        from paper_2510_14050_b200.traffic import PacketStream

        stream = PacketStream(src=ds.download().astype(np.int64), dst=dd.download().astype(np.int64),
                              valid=np.ones(n, dtype=bool), address_space=space)  # outside the timed region
        got = na.stats9(stream).astuple()
        assert got == tuple(stats), (got, stats)
        times = []
        for _ in range(2):
            t0 = time.perf_counter()
            na.stats9(stream)
            times.append(time.perf_counter() - t0)
        best = min(times)
        dropin = {"value": n_total / best, "unit": "packets/s", "ms_per_step": best * 1e3, "steps": 2,
                  "h2d_bytes_per_step": 9 * n_total, "d2h_bytes_per_step": 72,
                  "api": "paper_2510_14050_b200.analytics.stats9(PacketStream) (int64 src / dst + bool valid in "
                         "pageable host memory, as traffic.py:43-71 holds them) -> nmx_stats9_host_i64: library "
                         "threads narrow each 2^24-packet window into pinned slots while the previous window is "
                         "copied and partitioned",
                  "timing": "wall clock of the host-synchronous call, best of 2"}
        del stream

    parity = golden_parity(args.config, log2n, gen, stats)
    windows = None
    if world == 1 and args.config == "cfg2" and not args.log2n:
        windows = cfg2_windows(ds, dd, space, args, local)
    side = None
    if world == 1 and args.config == "cfg3" and not args.log2n and not args.no_side:
        ds.close()
        dd.close()
        side = {"cfg4": side_config("cfg4", args, local)}
    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    peaks, peak_kind = _peaks()
    # dominant kernel class (MSD partition scatter; onesweep pass on the LSD path): item
    # bytes in + out per launch (u64 levels 16 B, the narrowing column level 12 B, the u32
    # column levels 8 B), timed by CUDA events around every launch
    pass_ms = dom_ms / max(dom_launch, 1)
    bytes_per_launch = dom_bytes // max(dom_launch, 1)
    achieved = bytes_per_launch / (pass_ms / 1e3) / 1e9 if pass_ms else 0.0
    roof = {"bound": "hbm", "kernel": timing_last.get("dom_name", ""), "achieved": round(achieved, 1),
            "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4),
            "peak_kind": peak_kind, "traffic": _traffic(timing_last.get("dom_name", ""), n_total // max(world, 1)),
            "launches_per_step": dom_launch // max(args.steps, 1),
            "bytes_per_launch": bytes_per_launch, "avg_launch_ms": round(pass_ms, 4),
            "share_of_step": round(dom_ms / ms, 4) if ms else None,
            "per_launch": _per_launch(totals, peaks["hbm_gbs"]),
            "note": "algorithmic bytes = item bytes read + written per launch, averaged over the class "
                    "(16 B per item on the u64 levels, 12 B on the column level that narrows items to u32, "
                    "8 B on the u32 column levels); traffic per launch from ncu dram__bytes in profiles/"}
    # whole step: DRAM bytes the step actually moves (sum over its kernels of ncu
    # dram__bytes_read + write, profiles/traffic_<config>.json, one captured call of the
    # same configuration) / step time. SURVEY.md 8(d)'s canonical LSD byte count
    # (n(16+16P) + u(36+16Pc)) is reported beside it for reference only: this design moves
    # fewer bytes than that pipeline, so dividing it by the step time is not a bandwidth.
    b = 32 if space == 1 << 32 else max(1, (space - 1).bit_length())
    P, Pc = 2 * ((b + 7) // 8), (b + 7) // 8
    b_lsd = n_total * (16 + 16 * P) + stats[1] * (36 + 16 * Pc)
    measured = _step_traffic(args.config, n_total, world)
    whole = {"survey_lsd_bytes": b_lsd}
    if measured:
        gbs = measured["bytes"] / (ms_per_step / 1e3) / 1e9
        whole.update({"dram_bytes_per_step": measured["bytes"], "bytes_per_packet": round(measured["bytes"] / n_total, 2),
                      "achieved_gbs": round(gbs, 1), "frac": round(gbs / peaks["hbm_gbs"], 4),
                      "source": measured["source"]})

    cpu = None
    if not args.no_cpu:
        sample = min(log2n, args.cpu_log2n)
        rate, secs, _, ckind, cores = cpu_reference_rate(args.config, sample, space if args.config not in
                                                         ("cfg1", "cfg2") else 1 << 32, gen, reps=2)
        cpu = {"value": rate, "unit": "packets/s", "cores": cores, "kind": ckind,
               "sample": _cpu_sample_desc(args.config, sample, ckind, cores, secs, 2), "host": host_info()}
    stage_ms = timing_last.get("stages_ms", [])
    line = {
        "metric": METRIC, "value": value, "unit": "packets/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"{args.config}: 2^{log2n} packets {gen} over {space} addresses "
                               f"({'splitmix64, SURVEY.md 8(d)' if gen in ('uniform', 'powerlaw') else 'BASELINE.md'}) "
                               "summed into one traffic matrix, 9 statistics",
                   "packets": n_total, "address_space": space, "parallelism": f"shards{world}",
                   "l2": "inputs (8 GiB) and sort buffers larger than L2; no flush needed"},
        "stats9": list(stats),
        "parity": parity,
        "roofline": roof,
        "whole_step": {**whole, "stages_ms": stage_ms,
                       "stages": (["setup", "row partition", "row groups (smem)", "heavy rows", "column partition",
                                   "column groups (smem)", "heavy columns + d2h"]
                                  if timing_last.get("dom_name") == "msd_scatter" and len(stage_ms) == 7 else
                                  ["hist+plan", "row sort", "link/row", "col sort", "col+d2h"]
                                  if len(stage_ms) == 5 else "stages of the rank's last library call")},
        "e2e": e2e,
        "e2e_dropin": dropin,
        "windows": windows,
        "other_configs": side,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "gpu_launches": launches,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    if parity.get("equal") is False:
        sys.exit(f"bench: stats9 {list(stats)} differ from the golden {parity['want']}")


def cfg2_windows(ds, dd, space: int, args, local: int) -> dict:
    """BASELINE config 2's second output: the per-window analyze_dataset reports of the
    64 windows of 2^17 packets (nmx_window_stats9_device on the same device columns),
    K calls between CUDA events, checked against the reference-made golden."""
    import torch

    from paper_2510_14050_b200 import _lib

    window = 1 << 17
    ctx = _lib.context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    for _ in range(args.warmup):
        per = _lib.window_stats9(ds, dd, None, space, window, device=local)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(local)
    e0.record(stream)
    for _ in range(args.steps):
        per = _lib.window_stats9(ds, dd, None, space, window, device=local)
    e1.record(stream)
    torch.cuda.synchronize(local)
    ms = e0.elapsed_time(e1) / args.steps
    try:
        want = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())["cases"]["cfg2"]["windows9"]
        equal = per.tolist() == want
    except (OSError, KeyError, ValueError):
        equal = None
    n = int(ds.n)
    return {"workload": f"cfg2 per-window reports: {per.shape[0]} windows of 2^17 packets (build_matrices(s, 2^17) -> "
                        "analyze_dataset, analytics.py:109-130), device-resident",
            "value": n / (ms / 1e3), "unit": "packets/s", "ms_per_step": ms, "steps": args.steps,
            "parity": {"golden": "tests/golden/golden.json cfg2 windows9 (the reference netmeter package's own output)",
                       "equal": equal}}


def side_config(name: str, args, local: int) -> dict:
    """A second BASELINE config timed device-resident in the same run (one GPU): its own
    input, W warm-up + K timed calls between CUDA events on the library stream, and its
    statistics against the committed golden."""
    import torch

    from paper_2510_14050_b200 import _lib

    log2n, space, gen = CONFIGS[name]
    n = 1 << log2n
    kind = _lib.GEN_UNIFORM if gen == "uniform" else _lib.GEN_POWERLAW
    ds, dd = _lib.DeviceArray(n, device=local), _lib.DeviceArray(n, device=local)
    _lib.generate(kind, 7, 0, n, space, ds, dd, device=local)
    for _ in range(args.warmup):
        stats = _lib.stats9(ds, dd, None, space, device=local)
    ctx = _lib.context(local)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    torch.cuda.synchronize(local)
    e0.record(stream)
    for _ in range(args.steps):
        stats = _lib.stats9(ds, dd, None, space, device=local)
        launches += ctx.last_timing()["kernel_launches"]
    e1.record(stream)
    torch.cuda.synchronize(local)
    ms = e0.elapsed_time(e1) / args.steps
    t = ctx.last_timing()
    ds.close()
    dd.close()
    return {"workload": f"{name}: 2^{log2n} packets {gen} over {space} addresses, device-resident",
            "value": n / (ms / 1e3), "unit": "packets/s", "ms_per_step": ms, "steps": args.steps,
            "warmup": args.warmup, "stats9": list(stats), "parity": golden_parity(name, log2n, gen, stats),
            "stages_ms": t.get("stages_ms"), "gpu_launches": launches}


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: re-launch under torch.distributed.run with one
    rank per GPU (127.0.0.1 rendezvous, a free port); rank 0 prints the JSON line.
    NCCL's communicator set-up lines (NCCL_DEBUG=INFO, INIT) go to the log so every
    rank's device is on record."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="nmx", choices=["nmx", "reference"])
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--log2n", type=int, default=0)
    ap.add_argument("--ref-log2n", type=int, default=24, help="reference-arm sample per step")
    ap.add_argument("--cpu-log2n", type=int, default=24, help="cpu_baseline sample (about 10-30 s of CPU work)")
    ap.add_argument("--e2e-steps", type=int, default=4)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-side", action="store_true", help="skip the cfg4 side measurement of the default run")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        sys.exit(f"bench: --gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE')}")
    if args.impl == "reference":
        run_reference(args)
    elif args.config == "cfg5":
        run_cfg5(args)
    elif args.config == "file":
        run_file(args)
    elif args.config == "anon":
        run_anon(args)
    elif args.config == "cli":
        run_cli(args)
    else:
        run_nmx(args)


if __name__ == "__main__":
    main()
