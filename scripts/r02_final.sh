#!/bin/bash
# round-2 final measurements: the driver's default bench line, the reference arm, every BASELINE config
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
PU_PARITY_REPORT=gpurun_out/fin_parity.jsonl timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/fin_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/fin_smoke.log
timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/fin_default.json 2> gpurun_out/fin_default.err
for cfg in c1 c2; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/fin_$cfg.json 2> gpurun_out/fin_$cfg.err
done
timeout 1500 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fin_c5.json 2> gpurun_out/fin_c5.err
timeout 1500 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-nested > gpurun_out/fin_c4_fp64.json 2> gpurun_out/fin_c4_fp64.err
timeout 1500 python bench.py --config c4 --dtype fp32 --steps 3 --warmup 3 --no-cpu-baseline --no-nested > gpurun_out/fin_c4_fp32.json 2> gpurun_out/fin_c4_fp32.err
timeout 900 python bench.py --bands 1 --steps 5 --warmup 3 > gpurun_out/fin_rows1.json 2> gpurun_out/fin_rows1.err
timeout 900 python bench.py --bands 1 --dtype fp32 --steps 5 --warmup 3 > gpurun_out/fin_rows1_fp32.json 2> gpurun_out/fin_rows1_fp32.err
timeout 900 python bench.py --bands 2 --steps 5 --warmup 3 > gpurun_out/fin_rows2.json 2> gpurun_out/fin_rows2.err
timeout 1700 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/fin_reference.json 2> gpurun_out/fin_reference.err
ls -la gpurun_out/fin_*
