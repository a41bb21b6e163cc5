#!/bin/bash
# C5s / C3 ms per step against the h quantile the wide search grid is sized from (SPH_COARSE_Q).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for W in C5s C3; do for q in ${QS:-0.99 0.9 0.75 0.5 0.3}; do
  SPH_COARSE_Q=$q timeout 300 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cq.json 2>/dev/null
  python - $W $q <<'PY'
import json, sys
d = json.loads(open("gpurun_out/cq.json").read().strip().splitlines()[-1])
print(sys.argv[1], "q", sys.argv[2], "ms/step", round(d["ms_per_step"], 3), {k: round(v["ms_per_step"], 2) for k, v in d["kernels"].items()})
PY
done; done
