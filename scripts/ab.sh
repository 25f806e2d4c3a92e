#!/bin/bash
# A/B: alternate the alternative library (alt/$1.so) and the in-tree build on one box.
alt=${1:-old}; cfg=${2:-c3}; dt=${3:-fp32}; reps=${4:-2}
for i in $(seq $reps); do
  for lib in alt cur; do
    if [ $lib = alt ]; then export PU_LIB_PATH=$PWD/paper_2401_09961_b200/_lib/alt/$alt.so; else unset PU_LIB_PATH; fi
    timeout 900 python bench.py --no-cpu-baseline --config $cfg --dtype $dt --steps 10 --warmup 3 > gpurun_out/ab_$lib.json 2>/dev/null
    python -c "
import json;d=json.load(open('gpurun_out/ab_$lib.json'))
print('$lib', round(d['value'],2), round(d['ms_per_step'],2), {k: round(v['avg_ms'],4) for k,v in d['kernels'].items() if k.startswith('K')})"
  done
done
