"""Generate tests/golden/cli_golden.json by running the REAL reference CLI.

Build container only (reads /root/reference, absent on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_cli_golden.py

Records, for a few `netmeter generate` datasets, the manifest, the sha256 of every
matrix file the reference writes (traffic.py:295-304 write_matrix, cli.py:43-73),
and the per-window / total reports of `netmeter analyze` (cli.py:144-173).
"""

from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from netmeter.cli import cmd_analyze, cmd_generate  # noqa: E402

CASES = [
    {"n": 10, "space": 8, "seed": 3, "window": 4, "invalid": 0.0},
    {"n": 500, "space": 32, "seed": 9, "window": 64, "invalid": 0.0},
    {"n": 2000, "space": 64, "seed": 5, "window": 256, "invalid": 0.1},
    {"n": 100_000, "space": 2**20, "seed": 7, "window": 2**15, "invalid": 0.05},
]


def main() -> None:
    out = []
    for c in CASES:
        with tempfile.TemporaryDirectory() as d:
            manifest = cmd_generate(n=c["n"], address_space=c["space"], seed=c["seed"], window_size=c["window"],
                                    out_dir=d, invalid_fraction=c["invalid"])
            files = {p.name: hashlib.sha256(p.read_bytes()).hexdigest() for p in sorted(Path(d).iterdir())}
            reports, totals, _ = cmd_analyze(d)
        out.append({"case": c, "manifest": manifest, "sha256": files,
                    "reports": [r.to_dict() for r in reports], "totals": totals.to_dict()})
    path = Path(__file__).with_name("cli_golden.json")
    path.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print(f"wrote {path}")


if __name__ == "__main__":
    main()
