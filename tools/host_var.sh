#!/bin/bash
# Run-to-run variance of the host-latency-bound numbers (C2 ms per step, C4 e2e).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for k in 1 2 3; do
  timeout 300 python bench.py --workload C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/hv2.json 2>/dev/null
  timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/hv4.json 2>/dev/null
  python - <<'PY'
import json
d2 = json.loads(open("gpurun_out/hv2.json").read().strip().splitlines()[-1])
d4 = json.loads(open("gpurun_out/hv4.json").read().strip().splitlines()[-1])
print("C2", round(d2["ms_per_step"], 3), d2["clocks"], "C4", round(d4["ms_per_step"], 3), "e2e", round(d4["e2e"]["ms_per_step"], 3), d4["clocks"])
PY
done
