#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
PU_PARITY_REPORT=gpurun_out/c3k_parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/c3k_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/c3k_pytest.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/c3k_bench.json 2> gpurun_out/c3k_bench.err
for cfg in c2 c5; do timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c3k_$cfg.json 2>> gpurun_out/c3k_bench.err; done
tail -n 3 gpurun_out/c3k_pytest.log
