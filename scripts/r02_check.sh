#!/bin/bash
# GPU test suite + default bench line (tag in $1)
tag=${1:-x}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
PU_PARITY_REPORT=gpurun_out/parity_${tag}.jsonl timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_${tag}.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_${tag}.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
tail -3 gpurun_out/pytest_${tag}.log
