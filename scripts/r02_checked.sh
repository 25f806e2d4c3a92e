#!/bin/bash
# GPU suite against the PU_DEBUG_CHECKS build (device asserts on shared/global
# indices; compute-sanitizer is closed on this pool), then the production
# build's full suite and the default bench line.
tag=${1:-chk}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CHK=$PWD/paper_2401_09961_b200/_lib_chk/libpu_unwrap.so
PU_LIB_PATH=$CHK timeout 600 python scripts/sanitize_cases.py > gpurun_out/${tag}_cases.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_cases.log
PU_LIB_PATH=$CHK timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_dist1.py \
   > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log
PU_PARITY_REPORT=gpurun_out/parity_${tag}.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider \
   > gpurun_out/${tag}_main_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_main_pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
tail -n 3 gpurun_out/${tag}_cases.log gpurun_out/${tag}_pytest.log gpurun_out/${tag}_main_pytest.log
