#!/bin/bash
# tensor-core tile-DFT experiment: timings, then ncu --set full of the four kernels (one launch each)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 scripts/tc_tile_dft.cu -o scripts/tc_tile_dft
scripts/tc_tile_dft > gpurun_out/tc_tile_dft.jsonl 2> gpurun_out/tc_tile_dft.err && \
TC_PROFILE=1 scripts/tc_tile_dft > gpurun_out/tc_plain.log 2>&1 && \
TC_PROFILE=1 ncu --set full --import-source on --clock-control none -k regex:k_dft64 -c 4 -o gpurun_out/ncu_tc_tile_dft -f \
  scripts/tc_tile_dft > gpurun_out/ncu_tc_tile_dft.log 2>&1
echo rc=$?; cat gpurun_out/tc_tile_dft.jsonl
