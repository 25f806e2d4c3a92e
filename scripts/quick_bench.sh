#!/bin/bash
# quick C3 fp32 bench summary: value, step ms, per-kernel avg ms
cfg=${1:-c3}; dt=${2:-fp32}; steps=${3:-5}
timeout 900 python bench.py --no-cpu-baseline --config $cfg --dtype $dt --steps $steps --warmup 3 > gpurun_out/qb_$cfg.json 2> gpurun_out/qb_$cfg.err || tail -5 gpurun_out/qb_$cfg.err
python - <<PY
import json
d=json.load(open("gpurun_out/qb_$cfg.json"))
print("value", round(d["value"],2), "ms", round(d["ms_per_step"],2), "e2e", round(d["e2e"]["value"],2), "it_ms_step", round(d["roofline"]["pcg_iteration"]["ms_from_step"],4), "frac", round(d["roofline"]["pcg_iteration"]["frac_from_step"],3), "F", d["objective"])
print({k: round(v["avg_ms"],4) for k,v in d["kernels"].items()})
PY
