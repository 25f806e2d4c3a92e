#!/bin/bash
# ncu --set full of the transform kernels (K2b/K4 k_rows_pipe, K3 k_cols_spec) of one C3 unwrap, fp64 and fp32.
# usage: scripts/ncu_transforms.sh <tag> [extra regex]
tag=${1:-r02}; rx=${2:-'k_(cols_spec|rows_pipe|cols_split|rows_split)'}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for dt in fp64 fp32; do
  cmd="python bench.py --profile-steps 1 --config c3 --dtype $dt"
  $cmd > gpurun_out/plain_${tag}_${dt}.log 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:"$rx" --launch-skip 30 --launch-count 6 \
      -o gpurun_out/ncu_${tag}_xf_${dt} -f $cmd > gpurun_out/ncu_${tag}_xf_${dt}.log 2>&1
  echo "$dt rc=$?"
done
ls -la gpurun_out | grep ncu_
