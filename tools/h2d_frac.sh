#!/bin/bash
# e2e against the share of the upload on the copy engines (SPH_H2D_CE_FRAC), two runs each.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for f in ${FS:-0 0.3 0.5 0 0.3 0.5}; do
  SPH_H2D_CE_FRAC=$f timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/hf.json 2>/dev/null
  python - $f <<'PY'
import json, sys
d = json.loads(open("gpurun_out/hf.json").read().strip().splitlines()[-1])
print("ce_frac", sys.argv[1], round(d["ms_per_step"], 3), "e2e", round(d["e2e"]["ms_per_step"], 3), d["e2e"]["device_ms_per_step"])
PY
done
