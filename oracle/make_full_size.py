"""Write tests/golden/full_size.json: nine statistics at the BASELINE sizes from the
bounded-RAM chunked oracle (oracle/nmx_oracle.c) -- TEST INFRASTRUCTURE ONLY.

    python oracle/make_full_size.py            # ~10 min on 8 cores, < 3 GiB RAM

The oracle is pinned before use: it must reproduce every reference-generated
splitmix64 golden in tests/golden/golden.json (made by the real netmeter package,
2^16 .. 2^24) and the in-memory numpy restatement ``stats9_packed`` at 2^26;
the script refuses to write otherwise. The cases are the bench's (seed 7) and
the GPU tests' (seed 11) cfg3 / cfg4 streams at 2^30 packets over 2^32, and the
cfg5 streams (seed 7) at 2^31 and 2^32.
"""

from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import big  # noqa: E402
from oracle import netmeter_oracle as orc  # noqa: E402

CASES = [
    # (name, kind, seed, log2 n)
    ("cfg3_seed7", "uniform", 7, 30),
    ("cfg3_seed11", "uniform", 11, 30),
    ("cfg4_seed7", "powerlaw", 7, 30),
    ("cfg4_seed11", "powerlaw", 11, 30),
    ("cfg5_2^31_seed7", "uniform", 7, 31),
    ("cfg5_2^32_seed7", "uniform", 7, 32),
    ("cfg5pl_2^32_seed7", "powerlaw", 7, 32),
]


def pin() -> dict:
    g = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())["cases"]["splitmix"]
    checked = []
    for name, c in g.items():
        got = big.stats9_gen(big.UNIFORM if c["kind"] == "uniform" else big.POWERLAW, c["seed"], 0, c["n"],
                             c["space"], bucket_bits=4)
        assert got == tuple(c["stats9"]), (name, got, c["stats9"])
        checked.append(name)
    for kind, gen in (("uniform", orc.gen_uniform), ("powerlaw", orc.gen_powerlaw)):
        s, d = gen(5, 0, 1 << 26)
        want = orc.stats9_packed(s, d)
        got = big.stats9_gen(big.UNIFORM if kind == "uniform" else big.POWERLAW, 5, 0, 1 << 26)
        assert got == want, (kind, got, want)
        checked.append(f"{kind}_2^26_seed5 == stats9_packed")
    return {"reference_goldens": checked}


def main() -> None:
    out_path = ROOT / "tests" / "golden" / "full_size.json"
    old = json.loads(out_path.read_text()) if out_path.exists() else {"cases": {}}
    t0 = time.time()
    pinned = pin()
    print("oracle pinned", round(time.time() - t0, 1), "s", flush=True)
    out = {"generated_by": "oracle/make_full_size.py (oracle/nmx_oracle.c, bounded-RAM chunked packed-key oracle)",
           "pinned_against": pinned, "stats9_fields": list(orc.STATS9_FIELDS),
           "generator": "SURVEY.md 8(d) splitmix64 counter generators (oracle gen_uniform / gen_powerlaw)",
           "cases": old.get("cases", {})}
    only = set(sys.argv[1:])
    for name, kind, seed, lg in CASES:
        if only and name not in only:
            continue
        t = time.time()
        st = big.stats9_gen(big.UNIFORM if kind == "uniform" else big.POWERLAW, seed, 0, 1 << lg)
        out["cases"][name] = {"kind": kind, "seed": seed, "n": 1 << lg, "space": 1 << 32, "offset": 0,
                              "stats9": list(st), "oracle_seconds": round(time.time() - t, 1),
                              "threads": big.load().nmx_oracle_threads()}
        print(name, st, round(time.time() - t, 1), "s", flush=True)
        out_path.write_text(json.dumps(out, indent=1) + "\n")
    print("wrote", out_path, round(time.time() - t0, 1), "s", "cores", os.cpu_count())


if __name__ == "__main__":
    main()
