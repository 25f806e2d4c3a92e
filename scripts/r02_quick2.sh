cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
bash scripts/r02_quick.sh
for cfg in c1 c2; do
timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-nested > gpurun_out/q2_$cfg.json 2>> gpurun_out/q2.err
python - $cfg <<'PY'
import json, sys
d = json.loads([l for l in open(f"gpurun_out/q2_{sys.argv[1]}.json") if l.startswith("{")][-1])
print(sys.argv[1], round(d["value"], 2), round(d["ms_per_step"], 3), {k: round(x["avg_ms"] * 1e3, 1) for k, x in d["kernels"].items()}, d["parity"]["worst"])
PY
done
