#!/bin/bash
# band path: speculative start-up, peer transpose by default, world-1 all-reduce elided
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest -q -p no:cacheprovider tests/test_gpu_band.py tests/test_gpu_dist1.py tests/test_gpu_ipc2.py > gpurun_out/band_tests.log 2>&1; echo "rc=$?" >> gpurun_out/band_tests.log
tail -n 3 gpurun_out/band_tests.log
run() {
  tag=$1; shift
  timeout 900 python bench.py "$@" --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/band_$tag.json 2> gpurun_out/band_$tag.err
  python - gpurun_out/band_$tag.json <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
print(sys.argv[1], d["dtype"], round(d["value"], 2), round(d["ms_per_step"], 2), "e2e", round(d["e2e"]["value"], 2),
      d["config"]["sharding"][-50:], {k: round(x["avg_ms"] * 1e3, 1) for k, x in d["kernels"].items()})
PY
}
for a in "$@"; do
  case $a in
    peer) run peer --bands 1 ;;
    nopeer) run nopeer --bands 1 --no-peer ;;
    peer32) run peer32 --bands 1 --dtype fp32 ;;
    b2) run b2 --bands 2 ;;
    b2nopeer) run b2nopeer --bands 2 --no-peer ;;
  esac
done
