#!/bin/bash
# ncu --set full of the fp64 outer-iteration kernels (fused acceptance, H pair) on the final build
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
CMD="python bench.py --profile-steps 1 --config c3 --dtype fp64"
$CMD > gpurun_out/nof_plain.log 2>&1 || exit 1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:'k_(accept_start|hpair_states)_v' \
    --launch-skip 4 --launch-count 4 -o gpurun_out/ncu_r02_outer_fp64_final -f $CMD > gpurun_out/nof_ncu.log 2>&1
echo "ncu rc=$?"
