#!/bin/bash
# C2 (host-latency bound) against the nvidia-smi sampling interval (SPH_CLOCKS_MS).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for ms in ${MSS:-100 1000 100 1000 100 1000}; do
  SPH_CLOCKS_MS=$ms timeout 300 python bench.py --workload C2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/c2c.json 2>/dev/null
  python - $ms <<'PY'
import json, sys
d = json.loads(open("gpurun_out/c2c.json").read().strip().splitlines()[-1])
print("clocks_ms", sys.argv[1], round(d["ms_per_step"], 3), d["clocks"])
PY
done
