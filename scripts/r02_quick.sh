cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest -q -x -p no:cacheprovider tests/test_gpu_configs.py tests/test_gpu_unwrap.py tests/test_gpu_kernels.py tests/test_gpu_band.py > gpurun_out/hy_tests.log 2>&1; echo "rc=$?" >> gpurun_out/hy_tests.log; tail -n 2 gpurun_out/hy_tests.log
for rep in 1 2; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/hy.json 2>> gpurun_out/hy.err
python - <<'PY'
import json
d = json.loads([l for l in open("gpurun_out/hy.json") if l.startswith("{")][-1])
n = d["nested"]
print(round(d["value"], 2), round(d["ms_per_step"], 2), {k: round(x["avg_ms"] * 1e3, 1) for k, x in d["kernels"].items()}, "f32", round(n["value"], 2), d["clocks"]["sm_mhz"])
PY
done
