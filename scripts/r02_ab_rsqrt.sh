#!/bin/bash
# A/B: fused acceptance fp64 weights via rsqrt (PU_F64_RSQRT_W=1 build in _lib_rsq) vs sqrt + reciprocal
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
RSQ=$PWD/paper_2401_09961_b200/_lib_rsq/libpu_unwrap.so
PU_LIB_PATH=$RSQ timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_configs.py > gpurun_out/rsq_tests.log 2>&1; echo "rc=$?" >> gpurun_out/rsq_tests.log
tail -n 2 gpurun_out/rsq_tests.log
for rep in 1 2; do
  for v in main rsq; do
    if [ $v = rsq ]; then export PU_LIB_PATH=$RSQ; else unset PU_LIB_PATH; fi
    timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-nested > gpurun_out/rsq_$v.json 2>> gpurun_out/rsq.err
    python - $v >> gpurun_out/rsq_ab.txt <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads([l for l in open(f"gpurun_out/rsq_{v}.json") if l.startswith("{")][-1])
print(v, round(d["value"], 2), round(d["ms_per_step"], 2), {k: round(x["avg_ms"] * 1e3, 1) for k, x in d["kernels"].items() if k in ("accept_center", "hpair_states")}, "parity", d["parity"]["worst"])
PY
  done
done
unset PU_LIB_PATH
cat gpurun_out/rsq_ab.txt
