#!/bin/bash
# C5 images-in-flight sweep (fp32 and fp64)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for dt in fp32 fp64; do
  for c in 2 4 8 12; do
    timeout 600 python bench.py --config c5 --dtype $dt --concurrency $c --steps 2 --warmup 3 --no-cpu-baseline --no-nested > gpurun_out/c5s_${dt}_$c.json 2> gpurun_out/c5s_${dt}_$c.err
    python - gpurun_out/c5s_${dt}_$c.json $dt $c <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
print(sys.argv[2], "concurrency", sys.argv[3], round(d["value"], 2), round(d["ms_per_step"], 1), "e2e", round(d["e2e"]["value"], 2))
PY
  done
done
