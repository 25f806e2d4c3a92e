#!/bin/bash
# full GPU suite, smoke, default bench line (the driver's round-end checks)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ver_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ver_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ver_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/ver_smoke.log
timeout 1200 python bench.py > gpurun_out/ver_default.json 2> gpurun_out/ver_default.err; echo "bench rc=$?"
tail -n 2 gpurun_out/ver_pytest.log; tail -n 2 gpurun_out/ver_smoke.log
python - <<'PY'
import json
d = json.loads([l for l in open("gpurun_out/ver_default.json") if l.startswith("{")][-1])
print(d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline"]["frac"], d["roofline"]["pcg_iteration"]["frac_from_step"], d["parity"]["worst"], d["clocks"], d["nested"]["value"], d["cpu_baseline"])
PY
