"""Generate tests/golden/golden.json by running the REAL reference package.

Run in the build container only (it reads /root/reference, which does not
exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every expected value below comes from ``netmeter`` itself
(``/root/reference/pkg/src/netmeter``): the six reference measures from
``analyze_matrix`` / ``analyze_dataset`` (analytics.py:95-130) and the three
extra Graph Challenge maxima from the reference's own ``max_scan``
(analytics.py:89-92) over ``to_flat``'s ``weights``, ``row_sums[:,1]`` and
``col_sums[:,1]`` (traffic.py:245-292). Inputs are regenerated on the GPU box
by the oracle's restatement of ``generate_packets`` / ``anonymize``; their
sha256 prefixes are stored so generator drift is caught.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import netmeter  # noqa: E402  (the reference)
from netmeter.analytics import analyze_dataset, analyze_matrix, max_scan  # noqa: E402
from netmeter.resources import make_inline_scheduler  # noqa: E402
from netmeter.traffic import (  # noqa: E402
    PacketStream,
    TrafficMatrix,
    anonymize,
    build_matrices,
    generate_packets,
    to_flat,
)

from oracle import netmeter_oracle as orc  # noqa: E402

SCHED = make_inline_scheduler()


def ref9_flat(flat) -> list[int]:
    r = analyze_matrix(flat, SCHED)
    mx_link = max_scan(flat.weights, SCHED)
    mx_src = max_scan(flat.row_sums[:, 1] if len(flat.row_sums) else [], SCHED)
    mx_dst = max_scan(flat.col_sums[:, 1] if len(flat.col_sums) else [], SCHED)
    return [r.valid_packets, r.unique_links, mx_link, r.unique_sources, mx_src,
            r.max_fanout, r.unique_destinations, mx_dst, r.max_fanin]


def ref9_stream(stream: PacketStream) -> list[int]:
    """Nine statistics of the summed matrix: one window spanning all packets."""
    if len(stream) == 0:
        return [0] * 9
    (m,) = build_matrices(stream, window_size=len(stream))
    return ref9_flat(to_flat(m))


def ref9_windows(stream: PacketStream, window: int):
    flats = [to_flat(m) for m in build_matrices(stream, window)]
    per = [ref9_flat(f) for f in flats]
    reports, totals = analyze_dataset(flats, SCHED)
    # the reference's own totals for the six measures pin orc.totals9
    return per, [totals.valid_packets, totals.unique_links, totals.unique_sources,
                 totals.max_fanout, totals.unique_destinations, totals.max_fanin]


def main() -> None:
    out: dict = {"generated_by": "tests/golden/make_golden.py", "reference": "netmeter " + netmeter.__version__,
                 "stats9_fields": list(orc.STATS9_FIELDS), "cases": {}}
    cases = out["cases"]
    t0 = time.time()

    # hand fixtures: tests/test_acceptance.py:91-102, tests/test_analytics.py:98-106,128-130
    hand = TrafficMatrix(0, 2, [0, 2, 3], [0, 1, 1], [2, 1, 3])
    other = TrafficMatrix(1, 2, [0, 2, 3], [0, 1, 0], [4, 1, 1])
    f = to_flat(hand)
    cases["hand"] = {
        "pairs": [[0, 0], [0, 0], [0, 1], [1, 1], [1, 1], [1, 1]],
        "stats9": ref9_flat(f),
        "flat": {k: getattr(f, k).tolist() for k in
                 ("edges", "weights", "out_degrees", "in_degrees", "row_sums", "col_sums")},
    }
    cases["hand_other"] = {"pairs": [[0, 0]] * 4 + [[0, 1], [1, 0]], "stats9": ref9_flat(to_flat(other))}
    pairs = [(0, 1), (0, 1), (1, 0)]
    s = PacketStream(np.array([p[0] for p in pairs]), np.array([p[1] for p in pairs]), np.ones(3, bool), 2)
    cases["oracle_hand"] = {"pairs": [list(p) for p in pairs], "stats9": ref9_stream(s)}
    s = PacketStream(np.array([0, 0]), np.array([0, 0]), np.ones(2, bool), 1)
    cases["self_loops"] = {"pairs": [[0, 0], [0, 0]], "stats9": ref9_stream(s)}
    s = PacketStream(np.array([0, 0, 1]), np.array([1, 1, 0]), np.array([True, False, True]), 2)
    cases["invalid_hand"] = {"pairs": [[0, 1], [0, 1], [1, 0]], "valid": [1, 0, 1], "stats9": ref9_stream(s)}

    # known-answer corpus modelled on tests/test_acceptance.py:54-73 (seed 20260810),
    # 200 windows (n <= 10^4, space <= 256), plus invalid packets on every 5th.
    rng = np.random.default_rng(20260810)
    corpus = []
    for k in range(200):
        n = int(rng.integers(0, 10_001))
        space = int(rng.integers(1, 257))
        seed = int(rng.integers(0, 2**63))
        frac = 0.2 if k % 5 == 4 else 0.0
        st = generate_packets(n, space, seed, invalid_fraction=frac)
        corpus.append({"n": n, "space": space, "seed": seed, "invalid_fraction": frac,
                       "stats9": ref9_stream(st)})
    cases["corpus"] = corpus

    # generate_packets-based configs (cfg1; small windowed datasets)
    def gp_case(n, space, seed, key=None, frac=0.0, window=None):
        st = generate_packets(n, space, seed, invalid_fraction=frac)
        if key is not None:
            st, _ = anonymize(st, key=key)
        c = {"n": n, "space": space, "seed": seed, "anon_key": key, "invalid_fraction": frac,
             "address_space": st.address_space,
             "src_sha": orc.checksum_u32(st.src), "dst_sha": orc.checksum_u32(st.dst),
             "stats9": ref9_stream(st)}
        if window is not None:
            per, tot6 = ref9_windows(st, window)
            c["window"] = window
            c["windows9"] = per
            c["totals6"] = tot6
        return c

    cases["cfg1"] = gp_case(2**17, 2**32, seed=1, key=1)
    print("cfg1 done", time.time() - t0, flush=True)
    # tests/test_acceptance.py:76-88 configuration-invariance dataset
    cases["invariance"] = gp_case(10**6, 4096, seed=31415, key=31415, window=2**17)
    cases["windows_small"] = gp_case(10_000, 64, seed=77, window=512)
    cases["windows_invalid"] = gp_case(50_000, 300, seed=5, frac=0.25, window=4096)
    cases["cfg2"] = gp_case(2**23, 2**32, seed=2, key=2, window=2**17)
    print("cfg2 done", time.time() - t0, flush=True)

    # splitmix64 generators (cfg3/cfg4 shapes), compacted for the reference's dim limit
    def sm_case(kind, n, seed, space):
        gen = orc.gen_uniform if kind == "uniform" else orc.gen_powerlaw
        src, dst = gen(seed, 0, n, space)
        cs, cd, dim = orc.compact_ids(src, dst)
        st = PacketStream(cs, cd, np.ones(n, bool), dim)
        return {"kind": kind, "n": n, "seed": seed, "space": space,
                "src_sha": orc.checksum_u32(src), "dst_sha": orc.checksum_u32(dst),
                "stats9": ref9_stream(st)}

    sm = {}
    for kind in ("uniform", "powerlaw"):
        for lg, space in ((16, 2**32), (20, 2**32), (20, 2**16), (22, 2**32), (24, 2**32)):
            sm[f"{kind}_2^{lg}_space{space}"] = sm_case(kind, 2**lg, seed=7, space=space)
            print(kind, lg, space, "done", time.time() - t0, flush=True)
    cases["splitmix"] = sm

    path = ROOT / "tests" / "golden" / "golden.json"
    path.write_text(json.dumps(out, indent=1) + "\n")
    print("wrote", path, "in", round(time.time() - t0, 1), "s")


if __name__ == "__main__":
    main()
