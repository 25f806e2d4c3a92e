#!/bin/bash
# one compute-sanitizer tool per gpurun call (B200_PROFILING.md): scripts/sanitize.sh <tool>
tool=${1:-memcheck}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python scripts/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1 && \
timeout 2400 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
    python scripts/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
echo "$tool rc=$?" | tee -a gpurun_out/sanitize_$tool.log
tail -n 5 gpurun_out/sanitize_$tool.log
