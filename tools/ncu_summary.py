"""Summarise ncu --set full reports: python tools/ncu_summary.py rep1.ncu-rep ..."""
import csv, io, subprocess, sys
WANT = [
    ("gpu__time_duration.sum", "time_ms", "time"),
    ("dram__bytes_read.sum", "dram_rd_MB", None),
    ("dram__bytes_write.sum", "dram_wr_MB", None),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct", 1),
    ("lts__t_bytes.sum", "l2_MB", None),
    ("lts__t_sector_hit_rate.pct", "l2_hit_pct", 1),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct", 1),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ_pct", 1),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "thr_per_inst", 1),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_pct", 1),
    ("launch__registers_per_thread", "regs", 1),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem_conflicts", 1),
]
UNITS = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3, "Tbyte": 1e6}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    if len(r) < 3:
        return
    h, units = r[0], r[1]
    for row in r[2:]:
        d = {"kernel": row[h.index("Kernel Name")].split("(")[0][-40:]}
        for m, name, scale in WANT:
            if m not in h:
                continue
            i = h.index(m)
            try:
                v = float(row[i].replace(",", ""))
            except ValueError:
                d[name] = None
                continue
            if scale is None:
                v *= UNITS.get(units[i], 1)
            elif scale == "time":
                v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1, "ms": 1}.get(units[i], 1)
            d[name] = round(v, 2)
        yield d


for rep in sys.argv[1:]:
    print("#", rep)
    for d in rows(rep):
        print("  " + ", ".join(f"{k}={v}" for k, v in d.items()))
