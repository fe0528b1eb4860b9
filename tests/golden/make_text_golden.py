"""Generate tests/golden/text_golden.json by running the REAL reference read_matrix
(traffic.py:307-367) on a corpus of well-formed and malformed matrix texts.

Run in the build container only (it reads /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_text_golden.py

Each case records the raw bytes (base64) and either the parsed matrix (dim, row_ptr,
col_idx, values) or the exception type and message (the file path replaced by
``{path}``). tests/test_gpu_cli.py checks the device tokenizer / validator against it.
"""

from __future__ import annotations

import base64
import json
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True
ROOT = Path(__file__).resolve().parents[2]

from netmeter.traffic import read_matrix  # noqa: E402  (the reference)

TEXTS = [
    "2 1\n0 1 4\n",
    "\n2 1\n\n0 1 4\n\n",
    "2 2\r\n0 1 4\r\n1 1 +7\r\n",
    "2 2\r0 1 4\r1 1 7\r",
    "2\t1\n 0   1\t4",
    "3 3\n0 0 1_000\n0 2 007\n2 1 1\n",
    "3 2\n0 0 1\x0b2 1 1\n",
    "3 2\n0 0 1\x0c2 1 1\x1c",
    "3 2\n0\x1f0 1\n2 1 1\n",
    "3 2\n0 0 1\n\x1d\x1e2 1 1\n",
    "2 1\n0 1 4\n",
    "2 1 0 1 4\n",
    "2 1\n0 1 ٤\n",
    "2 1\n0 1 4",
    "",
    "\n\n \t\n",
    "2\n0 1 4\n",
    "2 1 5\n0 1 4\n",
    "x 1\n0 1 4\n",
    "0 1\n0 0 4\n",
    "-3 0\n",
    "2 -1\n",
    "2 0\n",
    "2 1\n0 1\n",
    "2 1\n0 1 4 5\n",
    "2 1\n0 1 four\n",
    "2 1\n0 1 4.0\n",
    "2 1\n0 1 1__0\n",
    "2 1\n0 1 _1\n",
    "2 1\n0 1 1_\n",
    "2 1\n0 1 +-4\n",
    "2 1\n0 1 -\n",
    "2 1\n0 1 9223372036854775808\n",
    "2 1\n0 1 9223372036854775807\n",
    "2 2\n0 1 4\n1 x 1\n1 1\n",
    "2 2\n0 1 4\n1 1\n1 x 1\n",
    "2 2\n0 1 4\n",
    "2 1\n0 1 4\n1 1 1\n",
    "2 2\n0 1 4\n2 1 1\n",
    "2 2\n0 1 4\n1 -1 1\n",
    "2 2\n0 1 0\n1 1 1\n",
    "2 2\n0 1 -3\n1 1 1\n",
    "2 2\n1 1 3\n0 1 1\n",
    "2 2\n0 1 3\n0 1 1\n",
    "3 3\n0 1 3\n5 1 1\n0 0 0\n",
    "3 3\n0 1 0\n1 0 1\n0 0 1\n",
    "4 3\n0 0 1\n\n1 3 2\n3 3 9\n",
    "5 1\n  +4   -0   +1  \n",
    "2 1\r\n\r\n0 1 4\r\n",
    "2 1\n0 1 4\n\x00\n",
]


def main() -> None:
    cases = []
    with tempfile.TemporaryDirectory() as d:
        path = Path(d) / "m.txt"
        for text in TEXTS:
            data = text.encode()
            path.write_bytes(data)
            case = {"bytes": base64.b64encode(data).decode()}
            try:
                m = read_matrix(path)
                case.update(ok=True, dim=int(m.dim), row_ptr=m.row_ptr.tolist(), col_idx=m.col_idx.tolist(),
                            values=m.values.tolist())
            except Exception as e:  # noqa: BLE001 - the reference's own outcome is the record
                case.update(ok=False, error=type(e).__name__, message=str(e).replace(str(path), "{path}"))
            cases.append(case)
    out = ROOT / "tests" / "golden" / "text_golden.json"
    out.write_text(json.dumps({"generated_by": "tests/golden/make_text_golden.py", "cases": cases}, indent=1) + "\n")
    print("wrote", out, len(cases), "cases")


if __name__ == "__main__":
    main()
