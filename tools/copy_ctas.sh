#!/bin/bash
# e2e ms per step against the CTA count of the pipelined host I/O's copy kernel (SPH_COPY_CTAS).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for n in ${NS:-32 64 148 296 592}; do
  SPH_COPY_CTAS=$n timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cc.json 2>/dev/null
  python - $n <<'PY'
import json, sys
d = json.loads(open("gpurun_out/cc.json").read().strip().splitlines()[-1])
print("ctas", sys.argv[1], round(d["ms_per_step"], 3), "e2e", round(d["e2e"]["ms_per_step"], 3), d["e2e"]["device_ms_per_step"])
PY
done
