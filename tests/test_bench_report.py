"""bench.py's report helpers on CPU: the per-launch roofline table and the ncu traffic
scaling (no GPU; the driver reads these keys from the JSON line)."""

import json

import pytest

import bench


def test_per_launch_averages_steps_and_fractions():
    totals = [{"dom_per_launch": [(2.0, 16 << 30), (1.0, 8 << 30)]},
              {"dom_per_launch": [(4.0, 16 << 30), (1.0, 8 << 30)]}]
    got = bench._per_launch(totals, 6000.0)
    assert [g["ms"] for g in got] == [3.0, 1.0]
    assert [g["bytes"] for g in got] == [16 << 30, 8 << 30]
    gbs0 = (16 << 30) / 3e-3 / 1e9
    assert got[0]["gbs"] == pytest.approx(gbs0, abs=0.1)
    assert got[0]["frac"] == pytest.approx(gbs0 / 6000.0, abs=1e-4)


def test_per_launch_needs_matching_launch_lists():
    assert bench._per_launch([], 6000.0) is None
    assert bench._per_launch([{"dom_per_launch": [(1.0, 1)]}, {"dom_per_launch": []}], 6000.0) is None


def test_traffic_scales_by_items_per_launch():
    t = json.loads((bench.ROOT / "profiles" / "traffic_latest.json").read_text())
    ks = [v for k, v in t["kernels"].items() if "msd_scatter" in k]
    per_launch = sum(v["dram_bytes"] for v in ks) / sum(v["launches"] for v in ks)
    assert bench._traffic("msd_scatter", t["items_per_launch"]) == round(per_launch)
    assert bench._traffic("msd_scatter", t["items_per_launch"] // 4) == pytest.approx(per_launch / 4, rel=1e-6)
    assert bench._traffic("no_such_kernel", 1 << 20) is None
