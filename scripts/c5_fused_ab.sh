for v in 0 1 0 1; do
  PU_FUSED_START=$v timeout 600 python bench.py --no-cpu-baseline --config c5 --steps 2 --warmup 3 > gpurun_out/c5_$v.json 2>gpurun_out/c5_$v.err || tail -3 gpurun_out/c5_$v.err
  python -c "import json;d=json.load(open('gpurun_out/c5_$v.json'));print('fused=$v', round(d['value'],2), round(d['ms_per_step'],1))"
done
