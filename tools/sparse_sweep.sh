#!/bin/bash
# C5s / C3 ms per step against the sparse-block threshold (SPH_SPARSE_WIDE).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for W in C5s C3; do for t in ${TS:-16 32 64}; do
  SPH_SPARSE_WIDE=$t timeout 300 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sw.json 2>/dev/null
  python - $W $t <<'PY'
import json, sys
d = json.loads(open("gpurun_out/sw.json").read().strip().splitlines()[-1])
print(sys.argv[1], "sparse", sys.argv[2], round(d["ms_per_step"], 3), {k: round(v["ms_per_step"], 2) for k, v in d["kernels"].items()})
PY
done; done
