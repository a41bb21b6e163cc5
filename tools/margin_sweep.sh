#!/bin/bash
# C5s / C3 ms per step against the wide margin (SPH_WIDE_MARGIN).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for W in C5s C3; do for m in ${MS:-0.1 0.2 0.3}; do
  SPH_WIDE_MARGIN=$m timeout 300 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/wm.json 2>/dev/null
  python - $W $m <<'PY'
import json, sys
d = json.loads(open("gpurun_out/wm.json").read().strip().splitlines()[-1])
print(sys.argv[1], "margin", sys.argv[2], round(d["ms_per_step"], 3), {k: round(v["ms_per_step"], 2) for k, v in d["kernels"].items()})
PY
done; done
