#!/bin/bash
# A/B: fp64 transforms with radix-16 stages (PU_F64_EMAX=16 build in _lib_e16) vs the default build
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
E16=$PWD/paper_2401_09961_b200/_lib_e16/libpu_unwrap.so
PU_LIB_PATH=$E16 timeout 1200 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_kernels.py tests/test_gpu_unwrap.py -k "fp64 or sylvester or split or long" > gpurun_out/ab_e16_tests.log 2>&1; echo "rc=$?" >> gpurun_out/ab_e16_tests.log
PU_LIB_PATH=$E16 PU_PARITY_REPORT=gpurun_out/ab_e16_parity.jsonl timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_configs.py -k fp64 > gpurun_out/ab_e16_cfg.log 2>&1; echo "rc=$?" >> gpurun_out/ab_e16_cfg.log
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_capi.py tests/test_gpu_dist1.py > gpurun_out/capi_dist.log 2>&1; echo "rc=$?" >> gpurun_out/capi_dist.log
for v in main e16; do
  if [ $v = e16 ]; then export PU_LIB_PATH=$E16; else unset PU_LIB_PATH; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-nested > gpurun_out/ab_bench_$v.json 2> gpurun_out/ab_bench_$v.err
done
unset PU_LIB_PATH
tail -n 3 gpurun_out/ab_e16_tests.log gpurun_out/ab_e16_cfg.log gpurun_out/capi_dist.log
