#!/bin/bash
# C4 per-kernel ms against the shared-memory carveout (SPH_CARVEOUT, percent; -1 = driver's choice).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for c in ${CS:--1 100 86 -1 100 86}; do
  SPH_CARVEOUT=$c timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/co.json 2>/dev/null
  python - $c <<'PY'
import json, sys
d = json.loads(open("gpurun_out/co.json").read().strip().splitlines()[-1])
print("carveout", sys.argv[1], round(d["ms_per_step"], 3), {k: round(v["ms_per_step"], 3) for k, v in d["kernels"].items()})
PY
done
