#!/bin/bash
# C2 and e2e (host-latency-bound) with and without spin-wait host synchronisation.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for sp in 0 1 0 1; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --spin $sp > gpurun_out/sp.json 2>/dev/null
  timeout 300 python bench.py --workload C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --spin $sp > gpurun_out/sp2.json 2>/dev/null
  python - $sp <<'PY'
import json, sys
d = json.loads(open("gpurun_out/sp.json").read().strip().splitlines()[-1])
d2 = json.loads(open("gpurun_out/sp2.json").read().strip().splitlines()[-1])
print("spin", sys.argv[1], "C4", round(d["ms_per_step"], 3), "e2e", round(d["e2e"]["ms_per_step"], 3), "C2", round(d2["ms_per_step"], 3))
PY
done
