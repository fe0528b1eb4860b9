"""Summarise an ncu report into per-kernel DRAM traffic (developer tool).

    python tools/ncu_traffic.py gpurun_out/prof.ncu-rep profiles/rNN_traffic.json ITEMS [CALLS]

ITEMS = items per launch of the profiled call (e.g. 2^28); the JSON records
dram bytes read + written per launch and per item for every kernel captured.
bench.py scales the dominant kernel's per-item traffic by its items per launch.
"""
import csv, io, json, subprocess, sys

rep, out, items = sys.argv[1], sys.argv[2], int(sys.argv[3])
calls = int(sys.argv[4]) if len(sys.argv) > 4 else 0  # hot-path calls captured (0: unknown)
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
units = rows[1]
res = {}
for r in rows[2:]:
    name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
    if "generate" in name or name.startswith("gen_kernel"):  # the input generator is not part of the call
        continue
    rd = float(r[h.index("dram__bytes_read.sum")].replace(",", ""))
    wr = float(r[h.index("dram__bytes_write.sum")].replace(",", ""))
    unit = units[h.index("dram__bytes_read.sum")]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    ms = float(r[h.index("gpu__time_duration.sum")].replace(",", ""))
    tunit = units[h.index("gpu__time_duration.sum")]
    ms *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1, "second": 1e3}.get(tunit, 1)
    e = res.setdefault(name, {"launches": 0, "dram_bytes": 0.0, "ms": 0.0})
    e["launches"] += 1
    e["dram_bytes"] += (rd + wr) * scale
    e["ms"] += ms
for k, e in res.items():
    e["dram_bytes_per_launch"] = e["dram_bytes"] / e["launches"]
    e["dram_bytes_per_item"] = e["dram_bytes_per_launch"] / items
    e["ms_per_launch"] = e["ms"] / e["launches"]
json.dump({"report": rep, "items_per_launch": items, "calls": calls, "kernels": res}, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
