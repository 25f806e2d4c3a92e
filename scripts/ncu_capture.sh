#!/bin/bash
# ncu --set full captures of the steady-state kernels of one C3 unwrap (run after a clean bench).
tag=${1:-r01}; cfg=${2:-c3}; dt=${3:-fp32}
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:'^k_' --launch-skip 400 --launch-count 10 \
    -o gpurun_out/ncu_${tag}_pcg -f python bench.py --profile-steps 1 --config $cfg --dtype $dt > gpurun_out/ncu_${tag}_pcg.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:'k_(pcg_start|hpair|accept|weights)' --launch-skip 8 --launch-count 4 \
    -o gpurun_out/ncu_${tag}_outer -f python bench.py --profile-steps 1 --config $cfg --dtype $dt > gpurun_out/ncu_${tag}_outer.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --profile-steps 1 --config $cfg --dtype $dt > gpurun_out/launches_${tag}.log 2>&1
ls -la gpurun_out/ | grep ncu_
