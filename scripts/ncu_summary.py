"""Summarise an ncu --set full report: per kernel duration, DRAM bytes, throughput, occupancy, stalls.

    python scripts/ncu_summary.py <report.ncu-rep> [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
col = {h: i for i, h in enumerate(hdr)}


def val(r, name):
    i = col.get(name)
    if i is None or r[i] in ("", "n/a"):
        return None
    try:
        return float(r[i].replace(",", ""))
    except ValueError:
        return r[i]


out = {}
for r in data:
    name = r[col["Kernel Name"]]
    short = name.split("(")[0].replace("void ", "")
    dur_us = val(r, "gpu__time_duration.sum")
    unit = units[col["gpu__time_duration.sum"]]
    if unit == "nsecond":
        dur_us = dur_us / 1e3
    elif unit == "msecond":
        dur_us = dur_us * 1e3
    rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
    ur, uw = units[col["dram__bytes_read.sum"]], units[col["dram__bytes_write.sum"]]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = rd * scale.get(ur, 1) if rd is not None else None
    wr = wr * scale.get(uw, 1) if wr is not None else None
    stalls = {}
    for h, i in col.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
            v = val(r, h)
            if isinstance(v, float) and v > 0:
                stalls[h.split("stalled_")[-1]] = v
    tot = sum(stalls.values()) or 1.0
    top = sorted(stalls.items(), key=lambda t: -t[1])[:4]
    out.setdefault(short, []).append({
        "duration_us": dur_us,
        "dram_read_bytes": rd, "dram_write_bytes": wr,
        "dram_gbs": ((rd or 0) + (wr or 0)) / (dur_us * 1e-6) / 1e9 if dur_us else None,
        "dram_throughput_pct": val(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
        "sm_throughput_pct": val(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
        "warps_active_pct": val(r, "sm__warps_active.avg.pct_of_peak_sustained_active"),
        "registers": val(r, "launch__registers_per_thread"),
        "top_stalls_pct": {k: round(100 * v / tot, 1) for k, v in top},
    })
if "--json" in sys.argv:
    with open(sys.argv[sys.argv.index("--json") + 1], "w") as fh:
        json.dump(out, fh, indent=1)
for k, lst in out.items():
    for d in lst:
        print(f"{k[:60]:<60} {d['duration_us']:8.1f} us  DRAM {((d['dram_read_bytes'] or 0) + (d['dram_write_bytes'] or 0)) / 1e6:8.1f} MB "
              f"{d['dram_gbs'] or 0:7.0f} GB/s  regs {d['registers']}  warps {d['warps_active_pct']}%  {d['top_stalls_pct']}")
