"""Per-CUDA-line instruction / stall shares of one kernel from an ncu report (developer tool).

    python tools/src_lines.py gpurun_out/prof.ncu-rep kernel_regex [top]
"""
import collections, csv, io, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass",
                      "--kernel-name", f"regex:{kre}"], capture_output=True, text=True).stdout
agg = collections.OrderedDict(); src = {}
h = None; fn = None
for r in csv.reader(io.StringIO(txt)):
    if r and r[0] == "File Path": fn = r[1].split("/")[-1]
    if r and r[0] == "Line No":
        h = r; ie = h.index("Instructions Executed"); ws = h.index("Warp Stall Sampling (All Samples)"); continue
    if h is None or len(r) < ie + 1 or not r[0].strip().isdigit(): continue
    key = (fn, int(r[0])); src[key] = r[1].strip()[:90]
    try: n = float(r[ie] or 0); s = float(r[ws] or 0)
    except ValueError: continue
    a = agg.setdefault(key, [0, 0]); a[0] += n; a[1] += s
tot = sum(v[0] for v in agg.values()) or 1; tws = sum(v[1] for v in agg.values()) or 1
print(f"warp instructions {tot:.4g}, stall samples {tws:.4g}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]}:{k[1]:<5d} {100*v[0]/tot:5.1f}% inst {100*v[1]/tws:5.1f}% stall | {src.get(k, '')}")
