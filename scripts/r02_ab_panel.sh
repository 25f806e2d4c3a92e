#!/bin/bash
# A/B: K3 column panels of 2 columns (one packed sequence; PU_PANEL_COLS=2 build in _lib_p2) vs the default
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
P2=$PWD/paper_2401_09961_b200/_lib_p2/libpu_unwrap.so
for rep in 1 2; do
  for v in main p2; do
    if [ $v = p2 ]; then export PU_LIB_PATH=$P2; else unset PU_LIB_PATH; fi
    for cfg in c3 c2; do
    timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/pan_${v}_$cfg.json 2>> gpurun_out/pan.err
    python - $v $cfg >> gpurun_out/pan_ab.txt <<'PY'
import json, sys
v, cfg = sys.argv[1], sys.argv[2]
d = json.loads([l for l in open(f"gpurun_out/pan_{v}_{cfg}.json") if l.startswith("{")][-1])
n = d["nested"]
k = lambda x: {kk: round(vv["avg_ms"] * 1e3, 1) for kk, vv in x["kernels"].items() if kk.startswith("K")}
print(v, cfg, "f64", round(d["value"], 2), round(d["ms_per_step"], 2), k(d), "| f32", round(n["value"], 2), round(n["ms_per_step"], 2), k(n),
      "| parity", d["parity"]["worst"], d["config"]["plan"]["cols_per_cta"])
PY
    done
  done
done
unset PU_LIB_PATH
cat gpurun_out/pan_ab.txt
