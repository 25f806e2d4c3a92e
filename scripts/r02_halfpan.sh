#!/bin/bash
# A/B: small-grid K3 half panels (default) vs full panels (PU_COL_NOBALANCE=1), C1 / C5 / C2
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_configs.py tests/test_gpu_unwrap.py > gpurun_out/hp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/hp_tests.log
tail -n 2 gpurun_out/hp_tests.log
for rep in 1 2; do
for cfg in c1 c5 c2; do
  for v in half full; do
    if [ $v = full ]; then export PU_COL_NOBALANCE=1; else unset PU_COL_NOBALANCE; fi
    st=10; [ $cfg = c5 ] && st=2
    timeout 600 python bench.py --config $cfg --steps $st --warmup 3 --no-cpu-baseline > gpurun_out/hp_${cfg}_$v.json 2> gpurun_out/hp_${cfg}_$v.err
    python - gpurun_out/hp_${cfg}_$v.json $cfg $v <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
n = d.get("nested") or {}
print(sys.argv[2], sys.argv[3], "f64", round(d["value"], 2), round(d["ms_per_step"], 2), "K3", round(d["kernels"]["K3_coldct_spectral"]["avg_ms"] * 1e3, 1),
      "f32", round(n.get("value", 0), 2), round(n.get("ms_per_step", 0), 2), "K3", round((n.get("kernels") or {}).get("K3_coldct_spectral", {}).get("avg_ms", 0) * 1e3, 1),
      "iter", (d["roofline"].get("pcg_iteration") or {}).get("frac_from_step"), "parity", (d.get("parity") or {}).get("worst"))
PY
  done
done
done
unset PU_COL_NOBALANCE
