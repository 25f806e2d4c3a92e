#!/bin/bash
# ncu launch list of one C1 fp64 unwrap (kernel durations vs the graph-replayed step)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python scripts/one_unwrap.py c1 fp64 2 > gpurun_out/c1l_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 6000 --csv --log-file gpurun_out/c1_launches.csv python scripts/one_unwrap.py c1 fp64 2 > gpurun_out/c1l_ncu.log 2>&1
python scripts/launch_shares.py gpurun_out/c1_launches.csv > gpurun_out/c1_launch_shares.txt
cat gpurun_out/c1l_plain.log gpurun_out/c1_launch_shares.txt
