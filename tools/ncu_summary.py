"""Summarise an ncu --set full report: per launch time, DRAM bytes, L2 hit, pipe use, top stalls.

    python tools/ncu_summary.py REPORT.ncu-rep > profiles/....txt
"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, data = rows[0], rows[1], rows[2:]
col = {n: i for i, n in enumerate(h)}
want = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr"),
        ("lts__t_sector_hit_rate.pct", "L2hit%"), ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM%"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64pipe%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps%"), ("launch__grid_size", "grid"),
        ("launch__block_size", "block"), ("launch__registers_per_thread", "regs")]
stalls = [x for x in h if x.startswith("smsp__pcsamp_warps_issue_stalled_") and not x.endswith("not_issued")]
print("# ncu --set full summary of", sys.argv[1].split("/")[-1])
print("# stalls = share of PC samples")
for r in data:
    name = r[col["Kernel Name"]].split("(")[0]
    vals = " ".join(f"{lab}={r[col[m]]}{units[col[m]].replace('%', '').replace(' ', '')}" for m, lab in want
                    if m in col)
    print(f"{name}: {vals}")
    tot = float(r[col["smsp__pcsamp_sample_count"]] or 1)
    st = sorted(((float(r[col[x]] or 0), x.replace("smsp__pcsamp_warps_issue_stalled_", "")) for x in stalls),
                reverse=True)[:5]
    print("    stalls: " + ", ".join(f"{n}={v / tot:.2f}" for v, n in st))
