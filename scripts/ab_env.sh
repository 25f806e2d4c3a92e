#!/bin/bash
# A/B of an environment knob on one box: ab_env.sh VAR VAL_A VAL_B [cfg] [dtype] [reps]
var=$1; va=$2; vb=$3; cfg=${4:-c3}; dt=${5:-fp32}; reps=${6:-2}
for i in $(seq $reps); do
  for v in $va $vb; do
    env $var=$v timeout 900 python bench.py --no-cpu-baseline --config $cfg --dtype $dt --steps 10 --warmup 3 > gpurun_out/abe_$v.json 2>gpurun_out/abe_$v.err || tail -3 gpurun_out/abe_$v.err
    python -c "
import json;d=json.load(open('gpurun_out/abe_$v.json'))
print('$var=$v $cfg $dt', round(d['value'],2), round(d['ms_per_step'],2), 'e2e', round(d['e2e']['value'],2), 'F', d['objective']['F'] if d.get('objective') else None, {k: round(v['avg_ms'],4) for k,v in d['kernels'].items() if not k.startswith('K')})"
  done
done
