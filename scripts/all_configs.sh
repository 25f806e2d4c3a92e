#!/bin/bash
# Bench every BASELINE config on one GPU; lines into gpurun_out/all_*.json
mkdir -p gpurun_out
run() { local tag=$1; shift; timeout 1200 python bench.py --no-cpu-baseline "$@" > gpurun_out/all_$tag.json 2> gpurun_out/all_$tag.err || tail -3 gpurun_out/all_$tag.err; }
run c1_fp32 --config c1 --steps 10 --warmup 3
run c2_fp32 --config c2 --steps 10 --warmup 3
run c2_fp64 --config c2 --dtype fp64 --steps 5 --warmup 3
run c3_fp32 --config c3 --steps 10 --warmup 3
run c3_fp64 --config c3 --dtype fp64 --steps 5 --warmup 3
run c4_fp32 --config c4 --steps 1 --warmup 3
run c5_fp32 --config c5 --steps 2 --warmup 3
run c3_rows_peer --config c3 --shard rows --peer --steps 3 --warmup 3
run c4_rows_peer --config c4 --shard rows --peer --steps 1 --warmup 3
python - <<'PY'
import json, glob
out = {}
for f in sorted(glob.glob("gpurun_out/all_*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        out[f] = str(e); continue
    it = d["roofline"].get("pcg_iteration", {})
    out[f.split("all_")[1][:-5]] = {"value_mpix_s": d["value"], "e2e_mpix_s": d["e2e"]["value"], "ms_per_step": d["ms_per_step"],
        "outer": d.get("outer_iters_per_step"), "pcg": d.get("pcg_iters_per_step"),
        "pcg_iter_ms_from_step": it.get("ms_from_step"), "pcg_iter_frac_from_step": it.get("frac_from_step"),
        "objective": d.get("objective"), "clocks": d.get("clocks")}
json.dump(out, open("gpurun_out/all_summary.json", "w"), indent=1)
for k, v in out.items():
    print(k, v if isinstance(v, str) else (round(v["value_mpix_s"], 2), round(v["e2e_mpix_s"], 2), round(v["ms_per_step"], 1), v["outer"], v["pcg"]))
PY
