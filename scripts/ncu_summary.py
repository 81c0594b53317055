"""Summarises an `ncu --set full` report (.ncu-rep) into a per-launch CSV of
the metrics the roofline needs (duration, DRAM bytes, DRAM %, tensor-pipe %,
occupancy, registers).  Usage: python scripts/ncu_summary.py rep.ncu-rep out.csv"""
import csv
import io
import subprocess
import sys

WANT = [
    ("kernel", "Kernel Name"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("regs", "launch__registers_per_thread"),
    ("duration_us", "gpu__time_duration.sum"),
    ("dram_read_bytes", "dram__bytes_read.sum"),
    ("dram_write_bytes", "dram__bytes_write.sum"),
    ("dram_pct_peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
    ("sm_active_cycles", "sm__cycles_active.avg"),
    ("elapsed_cycles", "gpc__cycles_elapsed.max"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("tensor_pipe_pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
    ("l2_hit_pct", "lts__t_sector_hit_rate.pct"),
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "us": 1, "msecond": 1e3}

raw = subprocess.check_output(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], text=True)
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
out = csv.writer(open(sys.argv[2], "w", newline=""))
out.writerow([k for k, _ in WANT])
for r in rows[2:]:
    vals = []
    for key, m in WANT:
        if m not in hdr:
            vals.append("")
            continue
        i = hdr.index(m)
        v = r[i]
        if key.endswith("_bytes") or key == "duration_us":
            try:
                v = f"{float(v.replace(',', '')) * SCALE.get(units[i], 1):.6g}"
            except ValueError:
                pass
        if key == "kernel":
            v = v.split("(")[0].replace("void ", "").replace("cascade::", "")
        vals.append(v)
    out.writerow(vals)
