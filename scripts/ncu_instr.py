"""Executed warp-instructions per CUDA source line (ncu source page)."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur, items, ie = None, [], None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        ie = r.index("Instructions Executed"); continue
    if r[0] and r[0].isdigit() and ie is not None and len(r) > ie:
        try:
            v = float(r[ie])
        except ValueError:
            continue
        items.append((v, f"{cur}:{r[0]}", r[1].strip()[:90]))
tot = sum(v for v, _, _ in items) or 1
items.sort(reverse=True)
print(f"total warp instructions {tot:.3e}")
for v, loc, src in items[:top]:
    print(f"{100 * v / tot:5.1f}%  {loc:<22} {src}")
