"""Benchmark: packets/s for traffic-matrix build + 9 statistics (BASELINE.json metric).

Workload (N=1): BASELINE config 3 -- 2^30 packets uniform over the 2^32 address
space (splitmix64 generator), summed into one hypersparse
traffic matrix, nine Graph Challenge statistics. One step = one full pass of
the hot path (ingest -> onesweep sort -> unique links/rows -> column sort ->
columns -> 9 int64 to host) over the whole batch.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl nmx|reference]
                  [--config cfg3|cfg4|cfg2|cfg1] [--log2n L]

N > 1 is launched by torchrun (one rank per GPU): the 2^30 packets are sharded
across ranks and exchanged by owner(src) / owner(dst) over NCCL
(paper_2510_14050_b200/distributed.py), total work fixed -> "scaling": "strong".

`--impl reference` times the reference's CPU path (the numpy port in
oracle/netmeter_oracle.py of build_matrices -> to_flat -> analyze_matrix, the
reference is pure Python and cannot travel to the GPU box) on the host cores,
rank 0 only, on a bounded sample of the same workload per step.
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
    # config 5 streamed from pinned host buffers in 2^28-packet windows into one
    # device-resident running sum; 2^31 of the 2^32 packets fit one B200 (positions
    # are u32 with a flag bit), 8 B200 take 2^29 each
    "cfg5": (31, 1 << 32, "uniform"),
    # 9-byte packet-file records (traffic.py:25) in pinned host
    # memory, streamed raw and unpacked on the GPU (nmx_stream_records)
    "file": (29, 1 << 32, "uniform"),
    # anonymize (traffic.py:107-137) of a cfg2-sized stream
    "anon": (23, 1 << 32, "uniform"),
    # `netmeter analyze` of a generated text dataset (CLI defaults:
    # address space 2^16, 2^17-packet windows -> 8 files at 2^20 packets)
    "cli": (20, 1 << 16, "uniform"),
}


def _traffic(kernel: str, bytes_per_launch: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch, from the committed ncu
    capture (profiles/traffic_latest.json, tools/ncu_traffic.py), scaled from the
    captured size to this launch's size by the per-item ratio; None if absent."""
    try:
        t = json.loads((ROOT / "profiles" / "traffic_latest.json").read_text())
    except Exception:
        return None
    ks = [v for k, v in t["kernels"].items() if kernel and kernel in k]
    if not ks:
        return None
    per_item = sum(v["dram_bytes"] for v in ks) / sum(v["launches"] for v in ks) / t["items_per_launch"]
    return round(per_item * bytes_per_launch / 16)


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


def cpu_port_rate(log2n: int, space: int, gen: str, reps: int = 1):
    """The reference's CPU path (numpy port) on a bounded sample: packets/s."""
    import numpy as np

    from oracle import netmeter_oracle as orc

    g = orc.gen_uniform if gen == "uniform" else orc.gen_powerlaw
    s, d = g(7, 0, 1 << log2n, space)
    cs, cd, dim = orc.compact_ids(s, d)  # excluded from timing
    valid = np.ones(len(cs), dtype=bool)
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        orc.ref_stats9(cs, cd, valid, dim)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return (1 << log2n) / best, best


def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    log2n, space, gen = CONFIGS[args.config]
    sample = min(log2n, args.ref_log2n)
    for _ in range(args.warmup):
        cpu_port_rate(sample, space, gen)
    rates = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r, _ = cpu_port_rate(sample, space, gen)
        rates.append(r)
    wall = time.perf_counter() - t0
    value = statistics.median(rates)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "packets/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": f"{args.config}: 2^{log2n} packets {gen} over {space} addresses, summed matrix, 9 stats",
                   "sample": f"2^{sample} packets of the same generator per step (ids compacted outside the timed region)"},
        "cpu_baseline": {"value": value, "unit": "packets/s", "cores": 1, "kind": "port",
                         "sample": f"2^{sample} packets/step; oracle/netmeter_oracle.py ref_stats9 = numpy port of "
                                   "traffic.py:197-292 + analytics.py:95-106 (numpy build is single-threaded)"},
        "e2e": {"value": value, "unit": "packets/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def run_cfg5(args) -> None:
    """Streamed windows (pinned host -> device, overlapped) + merge-add; rank 0 only."""
    import numpy as np

    from paper_2510_14050_b200 import _lib
    from paper_2510_14050_b200 import coo as nc

    if int(os.environ.get("RANK", "0")) != 0:
        return
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
    print(json.dumps({
        "metric": METRIC, "value": n_total / best, "unit": "packets/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": best * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"cfg5: {nwin} windows x 2^{int(np.log2(w))} packets {gen} streamed from pinned host "
                               "memory (nmx_stream_stats9: the H2D of window t+1 on a copy stream overlaps the "
                               "level-1 partition of window t into the device-resident running sum; the remaining "
                               "levels and the 9 statistics of the summed matrix run once)", "packets": n_total,
                   "timing": "wall clock of the host call (it is host-synchronous), best of steps"},
        "stats9": list(stats),
        "e2e": {"value": n_total / best, "unit": "packets/s", "h2d_bytes_per_step": 8 * n_total,
                "d2h_bytes_per_step": 72},
        "clocks": clk.summary(),
    }), flush=True)
    for a, b in wins:
        a.close()
        b.close()


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
            cli._timed_run(d, 1, None, 1)
        runs = [cli._timed_run(d, 1, None, 1) for _ in range(args.steps)]
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
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

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
        e2e = {"value": n_total / (ems / 1e3), "unit": "packets/s", "h2d_bytes_per_step": 8 * n_total,
               "d2h_bytes_per_step": 72 * world, "ms_per_step": ems, "steps": args.e2e_steps,
               "api": "nmx_stats9_host (include/nmx.h) via paper_2510_14050_b200._lib.stats9, pinned host buffers"}
        hs.close()
        hd.close()

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    peaks, peak_kind = _peaks()
    # dominant kernel class (MSD partition scatter; onesweep pass on the LSD path):
    # 8 B in + 8 B out per item per launch, timed by CUDA events around every launch
    pass_ms = dom_ms / max(dom_launch, 1)
    bytes_per_launch = dom_bytes // max(dom_launch, 1)
    achieved = bytes_per_launch / (pass_ms / 1e3) / 1e9 if pass_ms else 0.0
    roof = {"bound": "hbm", "kernel": timing_last.get("dom_name", ""), "achieved": round(achieved, 1),
            "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4),
            "peak_kind": peak_kind, "traffic": _traffic(timing_last.get("dom_name", ""), bytes_per_launch),
            "launches_per_step": dom_launch // max(args.steps, 1),
            "bytes_per_launch": bytes_per_launch, "avg_launch_ms": round(pass_ms, 4),
            "share_of_step": round(dom_ms / ms, 4) if ms else None,
            "note": "algorithmic bytes = 8 B read + 8 B write per item per launch; traffic per launch from ncu "
                    "dram__bytes in profiles/"}
    # whole-step algorithmic bytes: n(16+16P) + u(36+16Pc), P = 2*ceil(b/8), Pc = ceil(b/8)
    b = 32 if space == 1 << 32 else max(1, (space - 1).bit_length())
    P, Pc = 2 * ((b + 7) // 8), (b + 7) // 8
    u = stats[1]
    b_alg = n_total * (16 + 16 * P) + u * (36 + 16 * Pc)
    whole = b_alg / (ms_per_step / 1e3) / 1e9

    cpu = None
    if not args.no_cpu and world == 1:
        sample = min(log2n, args.cpu_log2n)
        rate, secs = cpu_port_rate(sample, space, gen, reps=2)
        cpu = {"value": rate, "unit": "packets/s", "cores": 1, "kind": "port",
               "sample": f"2^{sample} packets of the {args.config} generator, best of 2 ({secs:.2f} s each); "
                         "oracle/netmeter_oracle.py ref_stats9 (numpy port of traffic.py:197-292 + "
                         "analytics.py:95-106; ids compacted outside the timed region)"}
    stage_ms = timing_last.get("stages_ms", [])
    line = {
        "metric": METRIC, "value": value, "unit": "packets/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic",
        "config": {"workload": f"{args.config}: 2^{log2n} packets {gen} over {space} addresses (splitmix64, "
                               "SURVEY.md 8(d)) summed into one traffic matrix, 9 statistics",
                   "packets": n_total, "address_space": space, "parallelism": f"shards{world}",
                   "l2": "inputs (8 GiB) and sort buffers larger than L2; no flush needed"},
        "stats9": list(stats),
        "roofline": roof,
        "whole_step": {"b_alg_bytes": b_alg, "achieved_gbs": round(whole, 1),
                       "frac": round(whole / peaks["hbm_gbs"], 4), "stages_ms": stage_ms,
                       "stages": (["setup", "row partition", "row groups (smem)", "heavy rows", "column partition",
                                   "column groups (smem)", "heavy columns + d2h"]
                                  if timing_last.get("dom_name") == "msd_scatter" and len(stage_ms) == 7 else
                                  ["hist+plan", "row sort", "link/row", "col sort", "col+d2h"]
                                  if len(stage_ms) == 5 else "stages of the rank's last library call")},
        "e2e": e2e,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "gpu_launches": launches,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="nmx", choices=["nmx", "reference"])
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    ap.add_argument("--log2n", type=int, default=0)
    ap.add_argument("--ref-log2n", type=int, default=22, help="reference-arm sample per step")
    ap.add_argument("--cpu-log2n", type=int, default=24, help="cpu_baseline sample (about 10-30 s of CPU work)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
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
