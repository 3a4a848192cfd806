"""Writes profiles/<round>/ summaries from gpurun_out/ ncu captures:
   python tools/write_profiles.py r01
- ncu_<target>_<kernel>.txt : key metrics + top stall reasons + top source lines
- traffic_<app>.json (profiles/): dram bytes per launch of the dominant kernel
  (read by bench.py for roofline.traffic)
- launches_cf4.csv summary (kernel share of the headline step)"""
import csv
import glob
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
out = os.path.join(ROOT, "profiles", rnd)
os.makedirs(out, exist_ok=True)
# dominant timeline record per bench workload -> the kernels it is made of
# (3-MC's "extend_fused_L1" is the warp kernel + the tiled block kernel)
DOMINANT = {"cf4": ["local_warp_kernel"], "tc": ["edge_lane_kernel", "edge_chunk"], "mc3": ["mc3_warp", "mc3_block"],
            "mc4": ["mc4_roots"], "fsm": ["efan_kernel"]}
traffic = {}


def raw(rep):
    r = list(csv.reader(io.StringIO(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                                                   capture_output=True, text=True).stdout)))
    return r[0], r[1], r[2:]


def val(h, u, row, name):
    if name not in h:
        return None
    i = h.index(name)
    try:
        v = float(row[i].replace(",", ""))
    except ValueError:
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9, "ns": 1e-9,
             "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1, "s": 1}
    return v * scale.get(u[i], 1)


for rep in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "full_*.ncu-rep"))):
    tag = os.path.basename(rep)[len("full_"):-len(".ncu-rep")]
    h, u, rows = raw(rep)
    if not rows:
        continue
    lines = [f"# ncu --set full: {tag}  (report {os.path.basename(rep)})"]
    for row in rows:
        kname = row[h.index("Kernel Name")].split("(")[0]
        t = val(h, u, row, "gpu__time_duration.sum")
        rd = val(h, u, row, "dram__bytes_read.sum") or 0
        wr = val(h, u, row, "dram__bytes_write.sum") or 0
        l2 = val(h, u, row, "lts__t_bytes.sum")
        if not l2:
            sec = val(h, u, row, "lts__t_sectors.sum")
            l2 = 32.0 * sec if sec else None
        lines.append(f"kernel {kname}")
        lines.append(f"  duration_ms {t * 1e3:.4f}" if t else "  duration_ms ?")
        lines.append(f"  dram_read_GB {rd / 1e9:.3f}  dram_write_GB {wr / 1e9:.3f}  dram_GBps {((rd + wr) / t / 1e9) if t else 0:.1f}")
        if l2:
            lines.append(f"  l2_bytes_GB {l2 / 1e9:.3f}  l2_GBps {l2 / t / 1e9 if t else 0:.1f}")
        for m, lab in [("lts__t_sector_hit_rate.pct", "l2_hit_pct"),
                       ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_pct"),
                       ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
                       ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_pct"),
                       ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads_per_inst (warp efficiency x32)"),
                       ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_throughput_pct"),
                       ("launch__registers_per_thread", "registers"),
                       ("smsp__inst_executed.sum", "warp_instructions")]:
            v = val(h, u, row, m)
            if v is not None:
                lines.append(f"  {lab} {v:.2f}")
        st = [(h[i], row[i]) for i in range(len(h)) if h[i].startswith("smsp__pcsamp_warps_issue_stalled")
              and not h[i].endswith("not_issued")]
        tot = sum(float(x or 0) for _, x in st) or 1
        top = sorted(st, key=lambda x: -float(x[1] or 0))[:6]
        lines.append("  stalls " + ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * float(v) / tot:.1f}%"
                                           for k, v in top))
        app = tag.split("_")[0]
        if app in DOMINANT and any(k in kname for k in DOMINANT[app]) and t:
            e = traffic.setdefault(app, {"kernels": [], "dram_bytes_per_launch": 0.0, "l2_bytes_per_launch": 0.0,
                                         "duration_ms_ncu": 0.0, "sources": []})
            e["kernels"].append(kname)
            e["dram_bytes_per_launch"] += rd + wr
            e["l2_bytes_per_launch"] += l2 or 0.0
            e["duration_ms_ncu"] += t * 1e3
            e["sources"].append(f"profiles/{rnd}/ncu_{tag}.txt")
    src = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_source.py"), rep, ".", "0", "15"],
                         capture_output=True, text=True).stdout
    lines.append("top source lines (stall share, instruction share):")
    lines += ["  " + x for x in src.splitlines()]
    with open(os.path.join(out, f"ncu_{tag}.txt"), "w") as f:
        f.write("\n".join(lines) + "\n")
    print("wrote", f"ncu_{tag}.txt")

for app, e in traffic.items():
    with open(os.path.join(ROOT, "profiles", f"traffic_{app}.json"), "w") as f:
        json.dump(e, f, indent=1)

lc = os.path.join(ROOT, "gpurun_out", "launches_cf4.csv")
if os.path.exists(lc):
    rows = [r for r in csv.reader(open(lc)) if len(r) > 10 and r[0] != "ID"]
    agg = {}
    for r in rows:
        n = r[4].split("(")[0]
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += float(r[-1])
    tot = sum(v[1] for v in agg.values()) or 1
    with open(os.path.join(out, "launches_cf4_summary.txt"), "w") as f:
        f.write("# ncu --metrics gpu__time_duration.sum (cold, serialised) of `bench.py --app cf4 --steps 2 --warmup 3`\n")
        f.write("# includes warm-up, timed, clock-padding and e2e (upload + orientation) steps\n")
        for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"{t / 1e3:10.1f} us {100 * t / tot:5.1f}%  x{c:<4d} {n}\n")
    os.replace(lc, os.path.join(out, "launches_cf4.csv"))
    print("wrote launches summary")
