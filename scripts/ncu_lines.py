"""Aggregate ncu source-page warp-stall samples by CUDA source line.

    python scripts/ncu_lines.py <report.ncu-rep> <kernel regex> [top]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file, items = None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        si = 4  # "Warp Stall Sampling (All Samples)" column in the cuda,sass layout
        continue
    if r[0] and r[0].isdigit() and len(r) > 4:
        try:
            v = float(r[4])
        except ValueError:
            continue
        items.append((v, f"{cur_file}:{r[0]}", r[1].strip()[:100]))
tot = sum(v for v, _, _ in items) or 1.0
items.sort(reverse=True)
for v, loc, src in items[:top]:
    print(f"{100 * v / tot:5.1f}%  {loc:<22} {src}")
