#!/usr/bin/env python3
"""Collect the round's final bench lines (gpurun_out/fin_*.json, written by
scripts/r02_final.sh) into profiles/r02_all_configs.json and print a
markdown table for DESIGN.md §8."""

import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def last_json(path):
    try:
        lines = [ln for ln in open(path).read().splitlines() if ln.strip().startswith("{")]
        return json.loads(lines[-1]) if lines else None
    except OSError:
        return None


def main():
    src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
    out = {}
    for p in sorted(glob.glob(os.path.join(src, "fin_*.json"))):
        d = last_json(p)
        if d:
            out[os.path.basename(p)[4:-5]] = d
    with open(os.path.join(ROOT, "profiles", "r02_all_configs.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    rows = []
    for name, d in out.items():
        if d.get("impl") == "reference":
            rows.append(f"| reference arm (C3, {d['cpu_baseline']['cores']} host cores) | f64 | "
                        f"{d['ms_per_step'] / 1e3:.1f} s | {d['value']:.4f} | — | — | — |")
            continue
        par = d.get("parity") or {}
        w = par.get("worst") or {}
        pi = (d.get("roofline") or {}).get("pcg_iteration") or {}
        rows.append(f"| {name} | {d['dtype']} | {d['ms_per_step']:.1f} ms | {d['value']:.1f} | "
                    f"{(d.get('e2e') or {}).get('value', float('nan')):.1f} | "
                    f"{pi.get('frac_from_step') or pi.get('frac') or float('nan'):.2f} | "
                    f"{w.get('u_rel', '—') if w else '—'} |")
        n = d.get("nested")
        if n:
            w2 = ((n.get("parity") or {}).get("worst") or {})
            pi2 = (n.get("roofline") or {}).get("pcg_iteration") or {}
            rows.append(f"| {name} (nested) | {n['dtype']} | {n['ms_per_step']:.1f} ms | {n['value']:.1f} | "
                        f"{(n.get('e2e') or {}).get('value', float('nan')):.1f} | "
                        f"{pi2.get('frac_from_step') or float('nan'):.2f} | F_rel {w2.get('F_rel', '—')} |")
    print("| run | dtype | per step | Mpixel/s (HBM) | Mpixel/s e2e | PCG-iteration roofline | parity |")
    print("|---|---|---|---|---|---|---|")
    print("\n".join(rows))


if __name__ == "__main__":
    main()
