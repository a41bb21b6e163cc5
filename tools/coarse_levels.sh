#!/bin/bash
# C5s / C3 ms per step against the number of wide search grids (SPH_COARSE_LEVELS).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for W in C5s C3; do for L in ${LS:-1 2 3}; do
  SPH_COARSE_LEVELS=$L timeout 300 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cl.json 2>/dev/null
  python - $W $L <<'PY'
import json, sys
d = json.loads(open("gpurun_out/cl.json").read().strip().splitlines()[-1])
print(sys.argv[1], "levels", sys.argv[2], "ms/step", round(d["ms_per_step"], 3), {k: round(v["ms_per_step"], 2) for k, v in d["kernels"].items()})
PY
done; done
