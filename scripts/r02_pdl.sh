#!/bin/bash
# A/B: programmatic dependent launch of the PCG-iteration kernels (PU_PDL=0/1/2), correctness then timing
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for m in 1 2; do
  PU_PDL=$m timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_unwrap.py tests/test_gpu_configs.py -k "fp64_matches or c1 or c2 or fused or many" > gpurun_out/pdl_tests_$m.log 2>&1; echo "rc=$?" >> gpurun_out/pdl_tests_$m.log
done
for rep in 1 2; do
  for m in 0 1 2; do
    for cfg in c1 c2 c3; do
      PU_PDL=$m timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-nested > gpurun_out/pdl_${cfg}_$m.json 2>> gpurun_out/pdl.err
      python - $cfg $m >> gpurun_out/pdl_ab.txt <<'PY'
import json, sys
cfg, m = sys.argv[1], sys.argv[2]
d = json.loads(open(f"gpurun_out/pdl_{cfg}_{m}.json").read().strip().splitlines()[-1])
print(cfg, "PU_PDL=" + m, round(d["value"], 2), "Mpix/s", round(d["ms_per_step"], 3), "ms/step", "pcg_iter_ms_from_step",
      round(d["roofline"]["pcg_iteration"]["ms_from_step"] * 1e3, 1), "us")
PY
    done
  done
done
tail -n 2 gpurun_out/pdl_tests_*.log; cat gpurun_out/pdl_ab.txt
