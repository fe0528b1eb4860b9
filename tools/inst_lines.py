"""Per-CUDA-line executed instructions of one kernel from an ncu report (developer
tool): python tools/inst_lines.py rep.ncu-rep kernel_regex [top]"""
import collections, csv, io, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "--kernel-name", f"regex:{kre}"], capture_output=True, text=True).stdout
agg = collections.Counter(); src = {}; h = None; fn = None
for r in csv.reader(io.StringIO(txt)):
    if r and r[0] == "File Path": fn = r[1].split("/")[-1]
    if r and r[0] == "Line No":
        h = r; ie = h.index("Instructions Executed"); continue
    if h is None or len(r) <= ie or not r[0].strip().isdigit(): continue
    try: n = float(r[ie] or 0)
    except ValueError: continue
    k = (fn, int(r[0])); agg[k] += n; src[k] = r[1].strip()[:90]
tot = sum(agg.values()) or 1
print(f"warp instructions executed {tot:.4g}")
for k, v in agg.most_common(top):
    print(f"{k[0]}:{k[1]:<5d} {100 * v / tot:5.1f}% {v / 1e6:8.1f}M | {src.get(k, '')}")
