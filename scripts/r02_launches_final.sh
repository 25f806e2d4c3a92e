#!/bin/bash
# ncu launch list (gpu__time_duration.sum, recipe settings) of one C3 fp64 unwrap on the final build
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python scripts/one_unwrap.py c3 fp64 1 > gpurun_out/lf_plain.log 2>&1 || exit 1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/lf_launches.csv python scripts/one_unwrap.py c3 fp64 1 > gpurun_out/lf_ncu.log 2>&1
python scripts/launch_shares.py gpurun_out/lf_launches.csv > gpurun_out/lf_shares.txt
cat gpurun_out/lf_plain.log gpurun_out/lf_shares.txt
