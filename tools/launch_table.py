"""Per-kernel totals from an ncu --metrics gpu__time_duration.sum --csv launch list (developer tool).

    python tools/launch_table.py gpurun_out/launches.csv [skip_first_n_launches]
"""
import csv, sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
skip = int(sys.argv[2]) if len(sys.argv) > 2 else 0
agg = OrderedDict()
seq = []
for r in rows[1 + skip:]:
    name = r[ki].split("(")[0].replace("void ", "")[:90]
    v = float(r[vi].replace(",", ""))
    v *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(r[ui], 1.0)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += v
    seq.append((name, v))
tot = sum(v for _, v in seq)
print(f"total {tot:.3f} ms over {len(seq)} launches")
for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{ms:9.3f} ms {n:4d}x {100*ms/tot:5.1f}%  {k}")
if "-v" in sys.argv:
    for n, v in seq:
        print(f"{v:9.3f} {n}")
