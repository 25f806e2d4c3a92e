#!/bin/bash
# round-2 first GPU call: host facts, GPU tests with the config parity report, fp64/fp32 C3 bench lines
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
(free -g; nproc; lscpu | head -20; nvidia-smi) > gpurun_out/host.txt 2>&1
PU_PARITY_REPORT=gpurun_out/parity.jsonl timeout 1800 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --dtype fp64 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_fp64.json 2> gpurun_out/bench_fp64.err
timeout 600 python bench.py --dtype fp32 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_fp32.json 2> gpurun_out/bench_fp32.err
tail -3 gpurun_out/pytest_gpu.log
