#!/bin/bash
# A/B: fp64 32-byte vector loads/stores in the element-wise kernels (default build) vs 2 x 16 bytes (_lib_v128)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
V128=$PWD/paper_2401_09961_b200/_lib_v128/libpu_unwrap.so
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_configs.py tests/test_gpu_unwrap.py tests/test_gpu_kernels.py > gpurun_out/v256_tests.log 2>&1; echo "rc=$?" >> gpurun_out/v256_tests.log
tail -n 2 gpurun_out/v256_tests.log
for rep in 1 2; do
  for v in v256 v128; do
    if [ $v = v128 ]; then export PU_LIB_PATH=$V128; else unset PU_LIB_PATH; fi
    timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-nested > gpurun_out/v256_$v.json 2>> gpurun_out/v256.err
    python - $v >> gpurun_out/v256_ab.txt <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads([l for l in open(f"gpurun_out/v256_{v}.json") if l.startswith("{")][-1])
print(v, round(d["value"], 2), round(d["ms_per_step"], 2), {k: round(x["avg_ms"] * 1e3, 1) for k, x in d["kernels"].items()},
      "parity", d["parity"]["worst"], d["clocks"]["sm_mhz"])
PY
  done
done
unset PU_LIB_PATH
cat gpurun_out/v256_ab.txt
