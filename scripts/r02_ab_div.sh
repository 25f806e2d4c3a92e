#!/bin/bash
# A/B: fp64 slack division by reciprocal + Newton (PU_F64_SLACK_RCP build in _lib_div) vs IEEE division
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
DIV=$PWD/paper_2401_09961_b200/_lib_div/libpu_unwrap.so
PU_LIB_PATH=$DIV PU_PARITY_REPORT=gpurun_out/div_parity.jsonl timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_unwrap.py tests/test_gpu_configs.py tests/test_gpu_kernels.py -k "fp64 or pcg or c3" > gpurun_out/div_tests.log 2>&1; echo "rc=$?" >> gpurun_out/div_tests.log
for rep in 1 2; do
  for v in main div; do
    if [ $v = div ]; then export PU_LIB_PATH=$DIV; else unset PU_LIB_PATH; fi
    timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-nested > gpurun_out/div_$v.json 2>> gpurun_out/div.err
    python - $v >> gpurun_out/div_ab.txt <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/div_{v}.json").read().strip().splitlines()[-1])
print(v, round(d["value"], 2), round(d["ms_per_step"], 2), {k: round(x["avg_ms"] * 1e3, 1) for k, x in d["kernels"].items() if k.startswith("K")},
      "parity", d["parity"]["worst"])
PY
  done
done
unset PU_LIB_PATH
tail -n 2 gpurun_out/div_tests.log; cat gpurun_out/div_ab.txt
