"""Top CUDA source lines by warp-stall samples from an ncu report (cuda,sass view):
python tools/ncu_source.py rep.ncu-rep kernel_regex [launch_skip] [top]"""
import csv, io, subprocess, sys
rep, rx = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name",
                      "regex:" + rx, "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout
rows, fname, h = [], None, None
for row in csv.reader(io.StringIO(out)):
    if len(row) >= 2 and row[0] == "File Path":
        fname = row[1].split("/")[-1]
    elif row and row[0] == "Line No":
        h = row
    elif h and len(row) == len(h) and row[0] not in ("", "Line No"):
        rows.append((fname, row))
si = h.index("Warp Stall Sampling (All Samples)")
ii = h.index("Instructions Executed")
num = lambda v: float(v) if v not in ("", "-") else 0.0
tot = sum(num(x[si]) for _, x in rows) or 1
itot = sum(num(x[ii]) for _, x in rows) or 1
print(f"total samples {tot:.0f}, warp instructions {itot:.4g}")
for f, x in sorted(rows, key=lambda t: -num(t[1][si]))[:top]:
    print(f"{num(x[si]) / tot * 100:5.1f}% st {num(x[ii]) / itot * 100:5.1f}% in {f}:{x[0]:>5} | {x[1].strip()[:96]}")
