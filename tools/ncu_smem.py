"""Shared-memory wavefronts (total, excessive = bank conflicts) by CUDA source
line from an ncu report: python tools/ncu_smem.py rep.ncu-rep kernel_regex [top]"""
import csv, io, subprocess, sys
rep, rx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--kernel-name",
                      "regex:" + rx, "--launch-count", "1"], capture_output=True, text=True).stdout
rows, fname, h = [], None, None
for row in csv.reader(io.StringIO(out)):
    if len(row) >= 2 and row[0] == "File Path":
        fname = row[1].split("/")[-1]
    elif row and row[0] == "Line No":
        h = row
    elif h and len(row) == len(h) and row[0] not in ("", "Line No"):
        rows.append((fname, row))
num = lambda v: float(v) if v not in ("", "-") else 0.0
iw, ie = h.index("L1 Wavefronts Shared"), h.index("L1 Wavefronts Shared Excessive")
tw = sum(num(x[iw]) for _, x in rows) or 1
te = sum(num(x[ie]) for _, x in rows)
print(f"shared wavefronts {tw:.4g}, excessive {te:.4g}")
for f, x in sorted(rows, key=lambda t: -num(t[1][iw]))[:top]:
    print(f"{num(x[iw]) / tw * 100:5.1f}% wf {num(x[ie]) / tw * 100:5.1f}% excess {f}:{x[0]:>5} | {x[1].strip()[:96]}")
