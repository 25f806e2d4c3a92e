#!/bin/bash
# round-2 validation + measurement batch (after the C4 oracle call)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
GRP=$PWD/paper_2401_09961_b200/_lib_grp/libpu_unwrap.so
O1=$PWD/paper_2401_09961_b200/_lib_o1/libpu_unwrap.so
CHK=$PWD/paper_2401_09961_b200/_lib_chk/libpu_unwrap.so
# 1. K3 grouped barriers: correctness, then A/B
PU_LIB_PATH=$GRP timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_kernels.py tests/test_gpu_configs.py -k "sylvester or split or c3 or c2" > gpurun_out/post_grp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/post_grp_tests.log
PU_LIB_PATH=$O1 timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_unwrap.py tests/test_gpu_configs.py -k "fp64 or fused" > gpurun_out/post_o1_tests.log 2>&1; echo "rc=$?" >> gpurun_out/post_o1_tests.log
for v in main grp o1 main grp o1; do
  if [ $v = grp ]; then export PU_LIB_PATH=$GRP; elif [ $v = o1 ]; then export PU_LIB_PATH=$O1; else unset PU_LIB_PATH; fi
  for dt in fp64 fp32; do
    timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-nested --dtype $dt > gpurun_out/post_ab_${v}_${dt}.json 2>> gpurun_out/post_ab.err
    python - $v $dt >> gpurun_out/post_ab.txt <<'PY'
import json, sys
v, dt = sys.argv[1], sys.argv[2]
d = json.loads(open(f"gpurun_out/post_ab_{v}_{dt}.json").read().strip().splitlines()[-1])
print(v, dt, round(d["value"], 2), round(d["ms_per_step"], 2), {k: round(x["avg_ms"] * 1e3, 1) for k, x in d["kernels"].items()})
PY
  done
done
unset PU_LIB_PATH
# 2. debug-check build: sanitize cases + GPU suite
if [ -f $CHK ]; then
  PU_LIB_PATH=$CHK timeout 600 python scripts/sanitize_cases.py > gpurun_out/post_chk_cases.log 2>&1; echo "rc=$?" >> gpurun_out/post_chk_cases.log
  PU_LIB_PATH=$CHK timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_dist1.py > gpurun_out/post_chk_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/post_chk_pytest.log
fi
# 3. production build: full GPU suite with the parity report
PU_PARITY_REPORT=gpurun_out/post_parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/post_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/post_pytest.log
tail -n 3 gpurun_out/post_grp_tests.log gpurun_out/post_o1_tests.log gpurun_out/post_chk_cases.log gpurun_out/post_chk_pytest.log gpurun_out/post_pytest.log; cat gpurun_out/post_ab.txt
# 3b. row-sharded path through the bench (2 loopback bands, fp64) and C5 concurrency
timeout 600 python bench.py --bands 2 --steps 3 --warmup 3 > gpurun_out/post_bands2.json 2> gpurun_out/post_bands2.err
for c in 8 16; do
  for dt in fp32 fp64; do
    timeout 900 python bench.py --config c5 --concurrency $c --dtype $dt --steps 3 --warmup 3 --no-cpu-baseline --no-nested > gpurun_out/post_c5_${c}_${dt}.json 2>> gpurun_out/post_c5.err
  done
done
# 4. ncu: launch list of one fp64 C3 unwrap, and --set full of the PCG / outer kernels in fp64
CMD="python bench.py --profile-steps 1 --config c3 --dtype fp64"
$CMD > gpurun_out/post_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/post_launches_fp64.csv $CMD > gpurun_out/post_ncu_launches.log 2>&1
$CMD > gpurun_out/post_plain2.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:'k_pcg_(p|r)_v' \
    --launch-skip 20 --launch-count 4 -o gpurun_out/ncu_r02_pcg_fp64 -f $CMD > gpurun_out/post_ncu_full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:'k_(accept_start|hpair_states)_v' \
    --launch-skip 4 --launch-count 4 -o gpurun_out/ncu_r02_outer_fp64 -f $CMD > gpurun_out/post_ncu_full2.log 2>&1
echo "ncu rc=$?"
