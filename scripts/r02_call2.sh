#!/bin/bash
# round-2 call 2: split-transform tests, new unwrap tests, bench default line (fp64 headline + nested fp32)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_kernels.py -k "split or long or fp64_long" > gpurun_out/c2_split.log 2>&1; echo "rc=$?" >> gpurun_out/c2_split.log
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_gpu_unwrap.py -k "concurrent or survive or weight_shapes or held" tests/test_gpu_band.py -k "split or concurrent or survive or weight_shapes or held" > gpurun_out/c2_unwrap.log 2>&1; echo "rc=$?" >> gpurun_out/c2_unwrap.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c2_bench.json 2> gpurun_out/c2_bench.err
timeout 300 python bench.py --impl reference --config c1 --steps 3 --warmup 1 > gpurun_out/c2_ref_c1.json 2> gpurun_out/c2_ref_c1.err
tail -3 gpurun_out/c2_split.log gpurun_out/c2_unwrap.log
