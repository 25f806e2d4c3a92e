"""Instructions executed per CUDA source line (ncu source page), top N.

    python scripts/ncu_inst_lines.py <report> <kernel regex> [top]
"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, hdr, items, total = None, None, {}, 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr and r[0].isdigit() and len(r) > 6:
        try:
            v = float(r[hdr["Instructions Executed"]])
        except (ValueError, KeyError):
            continue
        key = (cur, int(r[0]), r[1][:90])
        items[key] = items.get(key, 0) + v
        total += v
for (f, ln, src), v in sorted(items.items(), key=lambda t: -t[1])[:top]:
    print(f"{100 * v / total:5.1f}%  {f}:{ln:<5} {src}")
print("total warp instructions", total)
